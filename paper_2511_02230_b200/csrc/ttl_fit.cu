// ttl_fit.cu — the TTL fit: one HBM pass over duration samples.
//
// Accumulator (fit_acc_words): per tool row f (row F pools every tool) the bucket counts and
// sums over the TTL grid, k = min(ceil(d / step), K) (a hit for tau_k iff d <= k step, reading
// R15), the paper-mode statistics (n, sum t~, sum t~^2 as 32-bit limb sums) of t~ = min(d, b)
// (reading R5), and the number of samples outside [0, 2^31).  Every field is
// a plain integer sum, so partial accumulators of disjoint sample sets add up exactly, in any
// order, on one GPU (atomics) or across ranks (an int64 all-reduce).
//
// fit_hist_kernel (phase 1): one CTA of 8 warps per resident slot streams one contiguous range
// of the tool-grouped (CSR) int32 samples with 16-B streaming loads (register double
// buffering, 8 int4 in flight per lane), cut into pieces at tool boundaries and at the 32-bit
// bin bound.  Every sample lands in the CTA's shared histogram as (count, sum of k step - d)
// with fire-and-forget 32-bit shared reductions; the histogram keeps one replica per lane index
// (32, or 16 when K is too large for shared memory), laid out [bucket][count x LR | remainder
// x LR] so that a warp instruction never hits one bank twice.  Each thread keeps the paper
// statistics in registers.  Pieces are merged and flushed with integer atomics.
// For ct_fit_ttl the same kernel also zeroes the other half of the context's double-buffered
// accumulator (the next call's), so no memset precedes it.
// fit_finish_kernel (phase 2), one warp per work item: (tool row, turn bucket j) -> the row's
// buckets prefix-summed by a warp scan (cnt_le(k), sum_le(k)), n U(k) in 128-bit integers
// (extension C-4), a warp argmax with the smallest k on ties; (row) -> the statistics and
// CalcTTL.  It is a programmatic dependent launch of the histogram pass
// (no launch gap), and runs alone in ct_fit_ttl_finish after a cross-rank all-reduce.
// fit_pairs_kernel is the fallback for the unsorted (dur_us, u8 tool) layout (PAPER.md:444's
// records S = {(f, t)} as they arrive): per-CTA shared bins per (tool, bucket), tool-keyed
// shared atomics; its accumulator is finished by fit_finish_kernel.
#include <algorithm>

#include "ct_device.cuh"
#include "ct_internal.h"

namespace ct {

constexpr int FW = 8;         // warps per CTA (histogram and finish phases)
constexpr int FT = 32 * FW;   // threads per CTA
constexpr int FU = 8;         // int4 loads per thread per double-buffer half
constexpr int SMEM_LIMIT = 232448 - 2048;  // B200 opt-in shared memory per block, minus static

int64_t fit_acc_words(int F, int K) {
  return 2 * (int64_t)(F + 1) * (K + 1) + 6 * (int64_t)(F + 1) + 1;
}

struct AccView {
  unsigned long long *hcnt, *hsum, *stat, *invalid;
};
__host__ __device__ __forceinline__ AccView acc_view(unsigned long long* base, int F, int K) {
  AccView v;
  const int64_t rows = (int64_t)(F + 1) * (K + 1);
  v.hcnt = base;
  v.hsum = base + rows;
  v.stat = base + 2 * rows;
  v.invalid = v.stat + 6 * (int64_t)(F + 1);
  return v;
}

FitPlan fit_plan(int K, int F, bool pairs) {
  FitPlan p;
  p.pairs = pairs;
  if (pairs) {
    p.lr = 0;
    p.smem = 8 * F * (K + 1) + 24 * F;
    p.ok = p.smem <= SMEM_LIMIT;
    return p;
  }
  p.lr = (K + 1) * 256 <= SMEM_LIMIT ? 32 : 16;
  p.smem = (K + 1) * 8 * p.lr;
  p.ok = p.smem <= SMEM_LIMIT && 16 * K <= p.smem;
  return p;
}

__device__ __forceinline__ void red_shared(uint32_t addr, uint32_t v) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

__device__ __forceinline__ void mad_wide(uint64_t& acc, uint32_t a, uint32_t b) {
  asm("mad.wide.u32 %0, %1, %2, %0;" : "+l"(acc) : "r"(a), "r"(b));
}

struct Lane {
  uint32_t base;                // shared address of this lane's count word of bucket 0
  uint32_t K, step, xoff, b_us;
  uint32_t dm, dsh, dadd;       // 32-bit Granlund-Montgomery divisor of step (step >= 2)
};

// One sample d.  Bucket k = min(ceil(d / step), K); the bins keep the count and the sum of
// r = k step - d in [0, step), so sum_k d = k step count_k - sum_k r is exact with 32-bit bins
// (bucket K keeps only the count).  ceil(d / step) = floor(x / step), x = d + step - 1 < 2^32,
// by the divisor's IMAD.HI plus shifts (DV: 0 identity for step 1, 1 multiply-high + shift,
// 2 the add variant; a compile-time choice, so no per-sample select).  The caller ORs the raw words
// of every int4 into neg: a negative sample (outside the documented [0, 2^31)) sets its sign
// bit, is then counted exactly and voids the outputs.
template <int DV, int LR, typename S1>
__device__ __forceinline__ void sample(const Lane& L, int32_t d, S1& s1, uint64_t& s2) {
  const uint32_t x = (uint32_t)d + L.xoff;
  uint32_t q;
  if (DV == 0) {  // step 1: the identity
    q = x;
  } else if (DV == 1) {  // multiply-high and shift
    q = __umulhi(x, L.dm) >> L.dsh;
  } else {  // the add variant of the divisor
    const uint32_t t = __umulhi(x, L.dm);
    q = (((x - t) >> 1) + t) >> L.dsh;
  }
  const uint32_t b = min(q, L.K);
  const uint32_t addr = L.base + b * (8 * LR);
  red_shared(addr, 1u);
  red_shared(addr + 4 * LR, b * L.step - (uint32_t)d);
  const uint32_t t = min((uint32_t)d, L.b_us);
  s1 += t;
  mad_wide(s2, t, t);
}

__device__ __forceinline__ Lane make_lane(const FitArgs& a, uint32_t* hsm, int lr) {
  Lane L;
  L.base = (uint32_t)__cvta_generic_to_shared(hsm) + 4 * (threadIdx.x & (lr - 1));
  L.K = (uint32_t)a.K;
  L.step = (uint32_t)a.step;
  L.xoff = L.step - 1;
  L.b_us = (uint32_t)a.b_us;
  L.dm = a.div_m;
  L.dsh = a.div_sh;
  L.dadd = a.div_add;
  return L;
}

// One work piece: samples [beg, end) of one tool -> zeroed CTA histogram -> flush into the
// tool's row and the pooled row F of the accumulator.
template <int DV, bool FAST32, int LR>
__device__ __forceinline__ void hist_piece(const FitArgs& a, const AccView& acc, const Lane& L,
                                           uint32_t* hsm, unsigned long long (*red)[3], int tool,
                                           int64_t beg, int64_t end) {
  const int K = a.K;
  const int tid = threadIdx.x, lane = tid & 31;
  const int words = (K + 1) * 2 * LR;
  for (int i = tid; i < words; i += FT) hsm[i] = 0;
  __syncthreads();
  uint64_t s1 = 0, s2 = 0;
  int32_t neg = 0;
  int64_t va = (beg + 3) & ~(int64_t)3;
  if (va > end) va = end;
  const int64_t vb = va + ((end - va) & ~(int64_t)3);
  if (tid < 32) {  // scalar head and tail (< 4 samples each)
    if (beg + lane < va) { const int32_t d = __ldg(&a.dur[beg + lane]); neg |= d; sample<DV, LR>(L, d, s1, s2); }
    if (vb + lane < end) { const int32_t d = __ldg(&a.dur[vb + lane]); neg |= d; sample<DV, LR>(L, d, s1, s2); }
  }
  const int4* v = (const int4*)(a.dur + va);
  const int64_t nv = (vb - va) >> 2;
  uint64_t q1 = 0, q2 = 0, q3 = 0;  // extra sum-of-squares accumulators (ILP)
  uint32_t s1w = 0;                  // 32-bit partial sum, flushed per 4 FU samples (b < 2^26)
  auto run4 = [&](const int4& x) {
    neg |= (x.x | x.y) | (x.z | x.w);
    if (FAST32) {
      sample<DV, LR>(L, x.x, s1w, s2);
      sample<DV, LR>(L, x.y, s1w, q1);
      sample<DV, LR>(L, x.z, s1w, q2);
      sample<DV, LR>(L, x.w, s1w, q3);
    } else {
      sample<DV, LR>(L, x.x, s1, s2);
      sample<DV, LR>(L, x.y, s1, q1);
      sample<DV, LR>(L, x.z, s1, q2);
      sample<DV, LR>(L, x.w, s1, q3);
    }
  };
  int64_t i = tid;
  int4 A[FU], B[FU];
  bool have_a = i + (FU - 1) * FT < nv;
  if (have_a) {
#pragma unroll
    for (int u = 0; u < FU; ++u) A[u] = __ldcs(v + i + u * FT);
  }
  while (have_a) {
    const int64_t ib = i + FU * FT;
    const bool have_b = ib + (FU - 1) * FT < nv;
    if (have_b) {
#pragma unroll
      for (int u = 0; u < FU; ++u) B[u] = __ldcs(v + ib + u * FT);
    }
#pragma unroll
    for (int u = 0; u < FU; ++u) run4(A[u]);
    if (FAST32) { s1 += s1w; s1w = 0; }
    i = ib;
    if (!have_b) break;
    const int64_t ia = ib + FU * FT;
    have_a = ia + (FU - 1) * FT < nv;
    if (have_a) {
#pragma unroll
      for (int u = 0; u < FU; ++u) A[u] = __ldcs(v + ia + u * FT);
    }
#pragma unroll
    for (int u = 0; u < FU; ++u) run4(B[u]);
    if (FAST32) { s1 += s1w; s1w = 0; }
    i = ia;
  }
  for (; i < nv; i += FT) {
    run4(__ldcs(v + i));
    if (FAST32) { s1 += s1w; s1w = 0; }
  }
  s2 += q1 + q2 + q3;
  const uint64_t w1 = warp_sum_u64(s1), w2 = warp_sum_u64(s2 & 0xffffffffull),
                 w3 = warp_sum_u64(s2 >> 32);
  if (lane == 0) { red[tid >> 5][0] = w1; red[tid >> 5][1] = w2; red[tid >> 5][2] = w3; }
  // a negative sample anywhere in the piece: count them exactly (rare path, invalid input)
  if (__syncthreads_or(neg < 0)) {
    unsigned long long c = 0;
    for (int64_t k = beg + tid; k < end; k += FT) c += a.dur[k] < 0;
    c = warp_sum_u64(c);
    if (lane == 0 && c) atomicAdd(acc.invalid, c);
  }
  if (tid < 6) {  // tid 0-2: the tool's row, 3-5: the pooled row F
    const int q = tid % 3;
    uint64_t sum = 0;
#pragma unroll
    for (int w = 0; w < FW; ++w) sum += red[w][q];
    unsigned long long* st = acc.stat + (tid < 3 ? tool : a.F) * 6;
    if (q == 0) atomicAdd(st, (unsigned long long)(end - beg));
    if (sum) atomicAdd(st + 1 + q, (unsigned long long)sum);
  }
  // merge the LR lane replicas of every bucket and flush (tool row + pooled row)
  for (int b = tid; b <= K; b += FT) {
    const uint4* pc = (const uint4*)(hsm + b * 2 * LR);
    uint64_t cn = 0, rr = 0;
#pragma unroll
    for (int q = 0; q < LR / 4; ++q) {
      const uint4 x = pc[q], y = pc[LR / 4 + q];
      cn += (uint64_t)x.x + x.y + x.z + x.w;
      rr += (uint64_t)y.x + y.y + y.z + y.w;
    }
    if (cn) {
      const uint64_t sm = b < K ? (uint64_t)b * L.step * cn - rr : 0;
#pragma unroll
      for (int row2 = 0; row2 < 2; ++row2) {
        const int64_t o = (int64_t)(row2 ? a.F : tool) * (K + 1) + b;
        atomicAdd(&acc.hcnt[o], (unsigned long long)cn);
        if (sm) atomicAdd(&acc.hsum[o], (unsigned long long)sm);
      }
    }
  }
  __syncthreads();
}

// Phase 1: CTA b streams virtual samples [bnd(b), bnd(b+1)) of the concatenated tool segments
// (segment f = physical samples [seg_lo[f], seg_hi[f]), virtual offset voff[f]); boundaries are
// 4-aligned in the virtual order (equal to the physical one for a whole CSR array, where only
// tool boundaries have scalar heads/tails).  A CTA zeroes and flushes its histogram about once.
template <int DV, bool FAST32, int LR>
__device__ __forceinline__ void hist_phase(const FitArgs& a, const AccView& acc, uint32_t* hsm,
                                           unsigned long long (*red)[3]) {
  const Lane L = make_lane(a, hsm, LR);
  const int64_t vtot = a.voff[a.F];
  const int64_t per = (vtot + gridDim.x - 1) / gridDim.x;
  auto bnd = [&](int64_t b) -> int64_t {
    if (b == 0) return 0;
    if (b >= (int64_t)gridDim.x) return vtot;
    return min(vtot, (b * per) & ~(int64_t)3);
  };
  int64_t lo = bnd(blockIdx.x);
  const int64_t hi = bnd((int64_t)blockIdx.x + 1);
  int tool = 0;
  while (lo < hi) {
    while (a.voff[tool + 1] <= lo) ++tool;
    const int64_t vend = min(hi, a.voff[tool + 1]);
    int64_t p0 = a.seg_lo[tool] + (lo - a.voff[tool]);
    const int64_t p1 = a.seg_lo[tool] + (vend - a.voff[tool]);
    while (p0 < p1) {
      const int64_t e = min(p1, p0 + a.ch);
      hist_piece<DV, FAST32, LR>(a, acc, L, hsm, red, tool, p0, e);
      p0 = e;
    }
    lo = vend;
  }
}

// ---------------------------------------------------------------------------------------------
// Phase 2: statistics row -> estimator Stat; argmax of n U(k) per (row, turn bucket); CalcTTL.
__device__ __forceinline__ Stat row_stat(const unsigned long long* stat, int row) {
  uint64_t v[6];
#pragma unroll
  for (int q = 0; q < 6; ++q) v[q] = stat[row * 6 + q];
  // renormalise the limbs: s2 = l0 + l1 2^32 + l2 2^64 + l3 2^96 (l2, l3 unused on this path)
  const u128_t s2 = (u128_t)v[2] + ((u128_t)v[3] << 32) + ((u128_t)v[4] << 64) + ((u128_t)v[5] << 96);
  Stat s;
  s.n = (int64_t)v[0];
  s.s1 = (int64_t)v[1];
  s.s2lo = (uint64_t)s2;
  s.s2hi = (uint64_t)(s2 >> 64);
  return s;
}

// V_j = floor(c_pf ctx_j (a_den + a_num w_j) / a_den) (prefill ps saved per hit, turn-weighted)
// and C_j = c_pin ceil(ctx_j / bs) (ps per µs pinned), extension C-4.
// (every factor is non-negative and a_den < 2^32, host-checked: an exact u128 / u64 quotient)
__device__ __forceinline__ void cost_vc(const ct_cost_params& cp, int j, i128_t& V, i128_t& C) {
  const u128_t num = (u128_t)(uint64_t)cp.c_pf_ps * (uint64_t)cp.ctx_tokens[j] *
                     ((u128_t)(uint64_t)cp.a_den + (u128_t)(uint64_t)cp.a_num * (uint64_t)cp.turn_weight[j]);
  V = (i128_t)div_u128_u64(num, (uint64_t)cp.a_den);
  C = (i128_t)cp.c_pin_ps * ceil_div_i64(cp.ctx_tokens[j], cp.bs);
}

// Phase 2, one CTA per (tool row, group of FW turn buckets), plus CTAs for the statistics and
// CalcTTL of every row (one thread per row).  In an argmax CTA warp w first
// prefix-sums bucket rounds w, w + FW, ... (round q = buckets 32 q .. 32 q + 31, coalesced
// loads, a warp scan each); the round totals through shared memory give every bucket's
// cnt_le(k), sum_le(k), kept in shared memory.  Then warp w takes turn bucket j = FW jg + w and
// evaluates n U(k) = V_j cnt_le(k) - C_j (sum_le(k) + tau_k (n - cnt_le(k))) in 128-bit
// integers over every k (lane-strided), keeps the smallest maximiser (U(0) = 0: no pin,
// PAPER.md:633), and one warp reduction gives tau*.  A tool with fewer than N samples takes the
// pooled row's argmax (PAPER.md:492-494 ladder).
constexpr int MAX_ROUNDS = (CT_MAX_K + 31) / 32;

__device__ __forceinline__ void argmax_cta(const ScanArgs& a, int row, int jg, unsigned long long* pre) {
  __shared__ unsigned long long tot[2][MAX_ROUNDS];
  const int K = a.K, F = a.F, J = a.J, K1 = K + 1;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const AccView acc = acc_view(const_cast<unsigned long long*>(a.acc), F, K);
  const unsigned long long n_bad = *acc.invalid;
  const uint64_t n_row = acc.stat[row * 6];
  const int src = (row != F && n_row < (uint64_t)a.est.n_min) ? F : row;
  const int j = jg * FW + warp;
  i128_t V = 0, C = 0;
  if (j < J) cost_vc(a.cost, j, V, C);
  const unsigned long long* hc = acc.hcnt + (int64_t)src * K1;
  const unsigned long long* hs = acc.hsum + (int64_t)src * K1;
  const int rounds = (K + 31) >> 5;
  constexpr int RW = MAX_ROUNDS / FW;  // rounds per warp at most
  uint64_t ic[RW], is[RW];
#pragma unroll
  for (int i = 0; i < RW; ++i) {  // loads of every round of this warp in flight together
    const int k = 32 * (warp + FW * i) + lane;
    ic[i] = k < K ? hc[k] : 0;
    is[i] = k < K ? hs[k] : 0;
  }
  const uint64_t over = hc[K];
#pragma unroll
  for (int i = 0; i < RW; ++i) {
    const int q = warp + FW * i;
    if (q < rounds) {
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint64_t tc = __shfl_up_sync(FULL_MASK, ic[i], o), ts = __shfl_up_sync(FULL_MASK, is[i], o);
        if (lane >= o) { ic[i] += tc; is[i] += ts; }
      }
      if (lane == 31) { tot[0][q] = ic[i]; tot[1][q] = is[i]; }
    }
  }
  __syncthreads();
  uint64_t carry_c = 0, carry_s = 0;
  int done = 0;
#pragma unroll
  for (int i = 0; i < RW; ++i) {
    const int q = warp + FW * i;
    if (q < rounds) {
      for (; done < q; ++done) { carry_c += tot[0][done]; carry_s += tot[1][done]; }
      const int k = 32 * q + lane;
      if (k < K) {
        pre[2 * k] = carry_c + ic[i];      // cnt_le(k)
        pre[2 * k + 1] = carry_s + is[i];  // sum_le(k)
      }
    }
  }
  uint64_t ntot = over;
  for (int q = 0; q < rounds; ++q) ntot += tot[0][q];
  __syncthreads();
  if (j >= J) return;
  const int64_t step = a.cost.grid_step_us;
  i128_t best = 0;
  int bk = 0;
  for (int k = lane; k < K; k += 32) {
    if (k == 0) continue;
    const uint64_t cc = pre[2 * k], cs = pre[2 * k + 1];
    const i128_t tau = (i128_t)k * step;
    const i128_t U = V * (i128_t)cc - C * ((i128_t)cs + tau * (i128_t)(ntot - cc));
    if (U > best) { best = U; bk = k; }  // k increases per lane: > keeps the smallest
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t lo = __shfl_xor_sync(FULL_MASK, (uint64_t)best, o);
    const uint64_t hi = __shfl_xor_sync(FULL_MASK, (uint64_t)((u128_t)best >> 64), o);
    const int ok = __shfl_xor_sync(FULL_MASK, bk, o);
    const i128_t ob = (i128_t)(((u128_t)hi << 64) | lo);
    if (ob > best || (ob == best && ok < bk)) { best = ob; bk = ok; }
  }
  if (lane == 0) a.ttl_argmax[(int64_t)row * J + j] = n_bad ? CT_TTL_INVALID : (int64_t)bk * step;
}

__device__ __forceinline__ void ttl_row(const ScanArgs& a, int row) {
  const AccView acc = acc_view(const_cast<unsigned long long*>(a.acc), a.F, a.K);
  const unsigned long long n_bad = *acc.invalid;
  if (n_bad) {  // samples outside [0, 2^31): no table (CT_TTL_INVALID everywhere)
    a.ttl_paper[row] = CT_TTL_INVALID;
    if (a.stats_out)
      for (int q = 0; q < 4; ++q) a.stats_out[row * 4 + q] = 0;
    if (row == 0 && a.n_invalid) *a.n_invalid = (int64_t)n_bad;
    return;
  }
  const Stat f = row_stat(acc.stat, row), g = row_stat(acc.stat, a.F);
  a.ttl_paper[row] = calc_ttl(g, f, a.est, a.cost.avg_turns_den, a.cost.avg_turns_num);
  if (a.stats_out) {
    a.stats_out[row * 4 + 0] = f.n;
    a.stats_out[row * 4 + 1] = f.s1;
    a.stats_out[row * 4 + 2] = (int64_t)f.s2lo;
    a.stats_out[row * 4 + 3] = (int64_t)f.s2hi;
  }
  if (row == 0 && a.n_invalid) *a.n_invalid = 0;
}

__host__ __device__ __forceinline__ int finish_argmax_ctas(int F, int J) { return (F + 1) * ((J + FW - 1) / FW); }

// ---------------------------------------------------------------------------------------------
// The histogram pass.  It first lets the finish kernel launch (programmatic dependent launch:
// the finish kernel's CTAs are scheduled while this grid streams and wait in
// griddepcontrol.wait for its completion, so no launch gap sits between the two), zeroes the
// other half of the context's double-buffered accumulator for the next call (no memset), then
// streams its range.
template <int DV, bool FAST32, int LR>
__global__ void __launch_bounds__(FT, 2) fit_hist_kernel(FitArgs a) {
  extern __shared__ __align__(16) uint32_t hsm[];
  __shared__ unsigned long long red[FW][3];
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int64_t nt = (int64_t)gridDim.x * FT;
  for (int64_t i = (int64_t)blockIdx.x * FT + threadIdx.x; i < a.zero_words; i += nt) a.zero[i] = 0;
  const AccView acc = acc_view(a.acc, a.F, a.K);
  hist_phase<DV, FAST32, LR>(a, acc, hsm, red);
}

__global__ void __launch_bounds__(FT) fit_finish_kernel(ScanArgs s) {
  extern __shared__ __align__(16) unsigned long long pre[];  // [K][2] cnt_le, sum_le
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the histogram grid is complete
  const int na = finish_argmax_ctas(s.F, s.J);
  if ((int)blockIdx.x < na) {
    const int jgs = (s.J + FW - 1) / FW;
    argmax_cta(s, blockIdx.x / jgs, blockIdx.x % jgs, pre);
  } else {
    const int row = ((int)blockIdx.x - na) * FT + threadIdx.x;
    if (row <= s.F) ttl_row(s, row);
  }
}

// ---------------------------------------------------------------------------------------------
// Unsorted pairs layout: dur_us int32[n] + tool uint8[n].  CTA b takes samples [bnd(b),
// bnd(b+1)) in pieces of <= ch; shared bins [F][K+1] x {count u32, remainder sum u32} and per
// tool {sum t~, sum lo32(t~^2), sum hi32(t~^2)} u64, updated with tool-keyed shared atomics.
__global__ void __launch_bounds__(FT) fit_pairs_kernel(FitArgs a) {
  extern __shared__ __align__(16) uint32_t psm[];
  const int F = a.F, K = a.K, K1 = K + 1;
  uint32_t* cnt = psm;                                       // [F][K+1]
  uint32_t* rem = psm + F * K1;                              // [F][K+1]
  unsigned long long* ts = (unsigned long long*)(psm + 2 * F * K1);  // [F][3]
  const AccView acc = acc_view(a.acc, F, K);
  const int tid = threadIdx.x, lane = tid & 31;
  const uint32_t step = (uint32_t)a.step, b_us = (uint32_t)a.b_us, xoff = step - 1;
  const int64_t n = a.n;
  const int64_t per = (((n + gridDim.x - 1) / gridDim.x) + 3) & ~(int64_t)3;
  const int64_t lo = min(n, (int64_t)blockIdx.x * per), hi = min(n, lo + per);
  for (int64_t beg = lo; beg < hi; beg += a.ch) {
    const int64_t end = min(hi, beg + a.ch);
    for (int i = tid; i < 2 * F * K1 + 6 * F; i += FT) psm[i] = 0;
    __syncthreads();
    unsigned long long bad = 0;
    auto one = [&](int32_t d, uint32_t f) {
      if (d < 0 || f >= (uint32_t)F) { ++bad; return; }
      const uint32_t x = (uint32_t)d + xoff;
      uint32_t q;
      if (step == 1) q = x;
      else {
        const uint32_t t = __umulhi(x, a.div_m);
        q = a.div_add ? ((((x - t) >> 1) + t) >> a.div_sh) : (t >> a.div_sh);
      }
      const uint32_t b = min(q, (uint32_t)K);
      atomicAdd(&cnt[f * K1 + b], 1u);
      if (b < (uint32_t)K) atomicAdd(&rem[f * K1 + b], b * step - (uint32_t)d);
      const uint64_t t = min((uint32_t)d, b_us), t2 = t * t;
      atomicAdd(&ts[f * 3 + 0], (unsigned long long)t);
      atomicAdd(&ts[f * 3 + 1], (unsigned long long)(t2 & 0xffffffffull));
      atomicAdd(&ts[f * 3 + 2], (unsigned long long)(t2 >> 32));
    };
    const int64_t va = min(end, (beg + 3) & ~(int64_t)3);
    const int64_t vb = va + ((end - va) & ~(int64_t)3);
    for (int64_t k = beg + tid; k < va; k += FT) one(a.dur[k], a.tool_u8[k]);
    for (int64_t k = vb + tid; k < end; k += FT) one(a.dur[k], a.tool_u8[k]);
    const int4* dv = (const int4*)(a.dur + va);
    const uint32_t* tv = (const uint32_t*)(a.tool_u8 + va);
    for (int64_t k = tid; k < (vb - va) >> 2; k += FT) {
      const int4 d = __ldcs(dv + k);
      const uint32_t t = __ldcs(tv + k);
      one(d.x, t & 0xff);
      one(d.y, (t >> 8) & 0xff);
      one(d.z, (t >> 16) & 0xff);
      one(d.w, t >> 24);
    }
    bad = warp_sum_u64(bad);
    if (lane == 0 && bad) atomicAdd(acc.invalid, bad);
    __syncthreads();
    // flush: tool rows, the pooled row F (bucket sums over tools), statistics
    for (int b = tid; b <= K; b += FT) {
      uint64_t pcn = 0, psum = 0;
      for (int f = 0; f < F; ++f) {
        const uint64_t cn = cnt[f * K1 + b];
        if (!cn) continue;
        const uint64_t sm = b < K ? (uint64_t)b * step * cn - rem[f * K1 + b] : 0;
        atomicAdd(&acc.hcnt[(int64_t)f * K1 + b], (unsigned long long)cn);
        if (sm) atomicAdd(&acc.hsum[(int64_t)f * K1 + b], (unsigned long long)sm);
        pcn += cn;
        psum += sm;
      }
      if (pcn) atomicAdd(&acc.hcnt[(int64_t)F * K1 + b], (unsigned long long)pcn);
      if (psum) atomicAdd(&acc.hsum[(int64_t)F * K1 + b], (unsigned long long)psum);
    }
    for (int f = tid >> 5; f < F; f += FW) {
      // n_f = sum of the tool's bucket counts; limbs of sum t~^2 = lo + hi 2^32
      uint64_t nf = 0;
      for (int b = lane; b <= K; b += 32) nf += cnt[f * K1 + b];
      nf = warp_sum_u64(nf);
      if (lane < 2 && nf) {
        unsigned long long* st = acc.stat + (lane ? F : f) * 6;
        const uint64_t s1 = ts[f * 3], lo = ts[f * 3 + 1], hi = ts[f * 3 + 2];
        atomicAdd(st + 0, (unsigned long long)nf);
        if (s1) atomicAdd(st + 1, (unsigned long long)s1);
        // lo = sum of 32-bit values, hi = sum of 32-bit values scaled by 2^32: split both into
        // 32-bit limb contributions l0 + l1 2^32 + l2 2^64
        if (lo & 0xffffffffull) atomicAdd(st + 2, (unsigned long long)(lo & 0xffffffffull));
        const uint64_t l1 = (lo >> 32) + (hi & 0xffffffffull);
        if (l1) atomicAdd(st + 3, (unsigned long long)l1);
        if (hi >> 32) atomicAdd(st + 4, (unsigned long long)(hi >> 32));
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------------------------
template <int DV>
static void* hist_fn_dv(bool fast32, int lr) {
  if (lr == 32) return fast32 ? (void*)fit_hist_kernel<DV, true, 32> : (void*)fit_hist_kernel<DV, false, 32>;
  return fast32 ? (void*)fit_hist_kernel<DV, true, 16> : (void*)fit_hist_kernel<DV, false, 16>;
}

static void* hist_fn(int dv, bool fast32, int lr) {
  return dv == 0 ? hist_fn_dv<0>(fast32, lr) : dv == 1 ? hist_fn_dv<1>(fast32, lr) : hist_fn_dv<2>(fast32, lr);
}

static void* pick_hist(const FitArgs& a, const FitPlan& p) {
  const int dv = a.step == 1 ? 0 : a.div_add ? 2 : 1;
  return p.pairs ? (void*)fit_pairs_kernel : hist_fn(dv, a.b_us < (1ll << 26), p.lr);
}

int fit_hist_occupancy(const FitArgs& a, const FitPlan& p) {
  void* k = pick_hist(a, p);
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, p.smem) != cudaSuccess) return 0;
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, FT, p.smem);
  return nb;
}

cudaError_t launch_fit_hist(const FitArgs& a, const FitPlan& p, int grid, cudaStream_t st) {
  void* args[] = {(void*)&a};
  return cudaLaunchKernel(pick_hist(a, p), dim3(grid), dim3(FT), args, p.smem, st);
}

// The finish kernel as a programmatic dependent launch of the histogram pass before it on the
// stream (its griddepcontrol.wait orders it after that grid's completion and memory flush).
cudaError_t launch_fit_finish(const ScanArgs& s, cudaStream_t st) {
  if (16 * s.K > 48 * 1024) {
    const cudaError_t e =
        cudaFuncSetAttribute(fit_finish_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * s.K);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(finish_argmax_ctas(s.F, s.J) + (s.F + 1 + FT - 1) / FT);
  cfg.blockDim = dim3(FT);
  cfg.dynamicSmemBytes = 16 * (size_t)s.K;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, fit_finish_kernel, s);
}

}  // namespace ct
