// ttl_fit.cu — the TTL fit: one HBM pass over duration samples.
//
// Kernel 1 (fit_hist): persistent CTAs stream tool-grouped (CSR) int32 samples with 16-B
// vector loads.  Every sample updates one packed u64 bin (count << 44 | sum) of its warp's
// private shared-memory histogram over the TTL grid buckets k = min(ceil(d / step), K), and the
// thread's register statistics (n, sum t~, sum t~^2 as 128-bit) of t~ = min(d, b) for the paper
// mode (reading R5).  At the end of a chunk the warp histograms are merged and
// flushed with integer atomics (order independent, hence deterministic).
// Kernel 2 (fit_scan): one warp per (tool row, turn bucket j): warp prefix scan of the bucket
// counts and sums, n U(k) in 128-bit integers (extension C-4), warp argmax with the smallest k on
// ties; the pooled row is the sum of the tool rows; tools with n_f < N take the pooled result;
// the j = 0 warp also evaluates CalcTTL on the row's statistics.
#include "ct_device.cuh"
#include "ct_internal.h"

namespace ct {

constexpr int FIT_THREADS = 256;
constexpr int FIT_WARPS = FIT_THREADS / 32;
constexpr uint64_t CNT_ONE = 1ull << 44;
constexpr uint64_t SUM_MASK = CNT_ONE - 1;

int fit_hist_threads() { return FIT_THREADS; }
int fit_hist_smem(int K) { return FIT_WARPS * (K + 1) * 8; }

struct Acc {
  uint64_t n, s1, lo, hi;
};

__device__ __forceinline__ void sample(uint64_t* __restrict__ h, int32_t d, int K, int64_t step,
                                       uint64_t magic, int64_t b_us, Acc& acc) {
  int b;
  uint64_t inc;
  if (d <= 0) {
    b = 0;
    inc = CNT_ONE;
  } else {
    uint64_t x = (uint64_t)(d - 1);
    uint64_t q = (x * magic) >> 32;
    if (q * (uint64_t)step > x) --q;
    b = q + 1 < (uint64_t)K ? (int)(q + 1) : K;
    inc = CNT_ONE | (b < K ? (uint64_t)d : 0ull);
  }
  atomicAdd((unsigned long long*)&h[b], (unsigned long long)inc);
  const uint64_t t = (uint64_t)min((int64_t)d, b_us);
  acc.n += 1;
  acc.s1 += t;
  const uint64_t t2 = t * t;
  acc.lo += t2;
  acc.hi += (acc.lo < t2);
}

__global__ void __launch_bounds__(FIT_THREADS) fit_hist_kernel(FitArgs a) {
  extern __shared__ __align__(16) unsigned long long hsm[];
  const int K = a.K;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t* h = (uint64_t*)hsm + warp * (K + 1);
  __shared__ unsigned long long red[FIT_WARPS][6];

  for (int64_t c = blockIdx.x; c < a.n_chunks; c += gridDim.x) {
    const FitChunk ch = a.chunks[c];
    for (int i = threadIdx.x; i < FIT_WARPS * (K + 1); i += FIT_THREADS) hsm[i] = 0;
    __syncthreads();
    Acc acc = {0, 0, 0, 0};
    // scalar head up to 16-B alignment, int4 body, scalar tail
    int64_t beg = ch.begin, end = ch.end;
    int64_t va = (beg + 3) & ~(int64_t)3;
    if (va > end) va = end;
    int64_t vb = va + ((end - va) & ~(int64_t)3);
    for (int64_t i = beg + threadIdx.x; i < va; i += FIT_THREADS)
      sample(h, __ldg(&a.dur[i]), K, a.step, a.step_magic, a.b_us, acc);
    const int4* v = (const int4*)(a.dur + va);
    const int64_t nv = (vb - va) >> 2;
    int64_t i = threadIdx.x;
    for (; i + 3 * FIT_THREADS < nv; i += 4 * FIT_THREADS) {
      int4 x0 = __ldcs(v + i);
      int4 x1 = __ldcs(v + i + FIT_THREADS);
      int4 x2 = __ldcs(v + i + 2 * FIT_THREADS);
      int4 x3 = __ldcs(v + i + 3 * FIT_THREADS);
      int4 xs[4] = {x0, x1, x2, x3};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        sample(h, xs[u].x, K, a.step, a.step_magic, a.b_us, acc);
        sample(h, xs[u].y, K, a.step, a.step_magic, a.b_us, acc);
        sample(h, xs[u].z, K, a.step, a.step_magic, a.b_us, acc);
        sample(h, xs[u].w, K, a.step, a.step_magic, a.b_us, acc);
      }
    }
    for (; i < nv; i += FIT_THREADS) {
      int4 x = __ldcs(v + i);
      sample(h, x.x, K, a.step, a.step_magic, a.b_us, acc);
      sample(h, x.y, K, a.step, a.step_magic, a.b_us, acc);
      sample(h, x.z, K, a.step, a.step_magic, a.b_us, acc);
      sample(h, x.w, K, a.step, a.step_magic, a.b_us, acc);
    }
    for (int64_t k = vb + threadIdx.x; k < end; k += FIT_THREADS)
      sample(h, __ldg(&a.dur[k]), K, a.step, a.step_magic, a.b_us, acc);

    // statistics: 128-bit sum of squares as four 32-bit limbs in 64-bit slots
    uint64_t l[6] = {acc.n, acc.s1, acc.lo & 0xffffffffull, acc.lo >> 32, acc.hi & 0xffffffffull,
                     acc.hi >> 32};
#pragma unroll
    for (int q = 0; q < 6; ++q) l[q] = warp_sum_u64(l[q]);
    if (lane == 0)
#pragma unroll
      for (int q = 0; q < 6; ++q) red[warp][q] = l[q];
    __syncthreads();
    if (threadIdx.x < 6) {
      uint64_t s = 0;
#pragma unroll
      for (int w = 0; w < FIT_WARPS; ++w) s += red[w][threadIdx.x];
      if (s) atomicAdd(&a.stat[ch.tool * 6 + threadIdx.x], (unsigned long long)s);
    }
    // merge the warp histograms and flush
    for (int b = threadIdx.x; b <= K; b += FIT_THREADS) {
      uint64_t cnt = 0, sum = 0;
#pragma unroll
      for (int w = 0; w < FIT_WARPS; ++w) {
        uint64_t x = hsm[w * (K + 1) + b];
        cnt += x >> 44;
        sum += x & SUM_MASK;
      }
      if (cnt) {
        atomicAdd(&a.hcnt[(int64_t)ch.tool * (K + 1) + b], (unsigned long long)cnt);
        if (sum) atomicAdd(&a.hsum[(int64_t)ch.tool * (K + 1) + b], (unsigned long long)sum);
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ void load_row(const ScanArgs& a, int row, int b, uint64_t& c,
                                         uint64_t& s) {
  const int K1 = a.K + 1;
  if (row < a.F) {
    c = a.hcnt[(int64_t)row * K1 + b];
    s = a.hsum[(int64_t)row * K1 + b];
  } else {
    c = 0;
    s = 0;
    for (int f = 0; f < a.F; ++f) {
      c += a.hcnt[(int64_t)f * K1 + b];
      s += a.hsum[(int64_t)f * K1 + b];
    }
  }
}

__device__ __forceinline__ Stat row_stat(const ScanArgs& a, int row) {
  uint64_t v[6] = {0, 0, 0, 0, 0, 0};
  for (int f = (row < a.F ? row : 0); f < (row < a.F ? row + 1 : a.F); ++f)
#pragma unroll
    for (int q = 0; q < 6; ++q) v[q] += a.stat[f * 6 + q];
  // renormalise the limbs: s2 = l0 + l1 2^32 + l2 2^64 + l3 2^96
  u128_t s2 = (u128_t)v[2] + ((u128_t)v[3] << 32) + ((u128_t)v[4] << 64) + ((u128_t)v[5] << 96);
  Stat s;
  s.n = (int64_t)v[0];
  s.s1 = (int64_t)v[1];
  s.s2lo = (uint64_t)s2;
  s.s2hi = (uint64_t)(s2 >> 64);
  return s;
}

// tau* for one row and turn bucket: warp scan over K bins + argmax (smallest k on ties).
__device__ int64_t argmax_row(const ScanArgs& a, int row, int j, int lane) {
  const int K = a.K;
  const ct_cost_params& cp = a.cost;
  const i128_t V = ((i128_t)cp.c_pf_ps * cp.ctx_tokens[j] *
                    ((i128_t)cp.a_den + (i128_t)cp.a_num * cp.turn_weight[j])) / cp.a_den;
  const i128_t C = (i128_t)cp.c_pin_ps * ceil_div_i64(cp.ctx_tokens[j], cp.bs);
  // n = all samples of the row, overflow bucket included
  uint64_t ntot = 0;
  for (int b = lane; b <= K; b += 32) {
    uint64_t c, s;
    load_row(a, row, b, c, s);
    ntot += c;
  }
  ntot = warp_sum_u64(ntot);
  // contiguous bins per lane for an ordered scan
  const int per = (K + 31) / 32;
  const int b0 = lane * per, b1 = min(b0 + per, K);
  uint64_t lc = 0, ls = 0;
  for (int b = b0; b < b1; ++b) {
    uint64_t c, s;
    load_row(a, row, b, c, s);
    lc += c;
    ls += s;
  }
  // exclusive scan across lanes
  uint64_t ic = lc, is = ls;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint64_t tc = __shfl_up_sync(FULL_MASK, ic, o);
    uint64_t ts = __shfl_up_sync(FULL_MASK, is, o);
    if (lane >= o) { ic += tc; is += ts; }
  }
  uint64_t cc = ic - lc, cs = is - ls;
  i128_t best = 0;  // U(0) = 0: TTL 0 = no pin
  int bk = 0;
  for (int b = b0; b < b1; ++b) {
    uint64_t c, s;
    load_row(a, row, b, c, s);
    cc += c;
    cs += s;
    if (b == 0) continue;
    const i128_t tau = (i128_t)b * a.cost.grid_step_us;
    const i128_t U = V * (i128_t)cc - C * ((i128_t)cs + tau * (i128_t)(ntot - cc));
    if (U > best) { best = U; bk = b; }
  }
  // argmax across lanes: larger U wins, ties -> smaller k
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    uint64_t lo = __shfl_xor_sync(FULL_MASK, (uint64_t)best, o);
    uint64_t hi = __shfl_xor_sync(FULL_MASK, (uint64_t)((u128_t)best >> 64), o);
    int ok = __shfl_xor_sync(FULL_MASK, bk, o);
    i128_t ob = (i128_t)(((u128_t)hi << 64) | lo);
    if (ob > best || (ob == best && ok < bk)) { best = ob; bk = ok; }
  }
  return (int64_t)bk * a.cost.grid_step_us;
}

__global__ void __launch_bounds__(128) fit_scan_kernel(ScanArgs a) {
  const int lane = threadIdx.x & 31;
  const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int J = a.J;
  if (w >= (a.F + 1) * J) return;
  const int row = w / J, j = w % J;
  const Stat g = row_stat(a, a.F);
  const Stat f = row_stat(a, row);
  // tools with fewer than N samples take the pooled row's result (PAPER.md:492-494 ladder)
  const int eff = (row < a.F && f.n < a.est.n_min) ? a.F : row;
  const int64_t tau = argmax_row(a, eff, j, lane);
  if (lane == 0) {
    a.ttl_argmax[(int64_t)row * J + j] = tau;
    if (j == 0) {
      a.ttl_paper[row] = calc_ttl(g, f, a.est, a.cost.avg_turns_den, a.cost.avg_turns_num);
      if (a.stats_out) {
        a.stats_out[row * 4 + 0] = f.n;
        a.stats_out[row * 4 + 1] = f.s1;
        a.stats_out[row * 4 + 2] = (int64_t)f.s2lo;
        a.stats_out[row * 4 + 3] = (int64_t)f.s2hi;
      }
    }
  }
}

cudaError_t launch_fit_hist(const FitArgs& a, int grid, cudaStream_t s) {
  int smem = fit_hist_smem(a.K);
  cudaError_t e = cudaFuncSetAttribute(fit_hist_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  fit_hist_kernel<<<grid, FIT_THREADS, smem, s>>>(a);
  return cudaGetLastError();
}

int fit_hist_occupancy(int smem) {
  if (cudaFuncSetAttribute(fit_hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) !=
      cudaSuccess)
    return 0;
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fit_hist_kernel, FIT_THREADS, smem);
  return nb;
}

cudaError_t launch_fit_scan(const ScanArgs& a, cudaStream_t s) {
  int warps = (a.F + 1) * a.J;
  int grid = (warps + 3) / 4;
  fit_scan_kernel<<<grid, 128, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace ct
