// synth.cu — on-device trace synthesis (NEXT-4): the integer-only generator
// of ctgen/synth.py (its docstring is the definition) evaluated in HBM, bit for bit.
//
// Three passes, one warp per seed in the per-seed passes:
//   1. synth_count: each lane takes programs p = lane + 32 k; the BFCL/SWE class is the rank of
//      the program's mix key among the seed's (keys staged in shared memory, O(P^2) compares),
//      the turn count is truncated at the context cap (R24) by regenerating new + decode per
//      turn; arrivals and turn offsets are warp prefix sums over program order.
//   2. scan_seeds: exclusive scan of the per-seed turn totals (block scan, block-total scan,
//      fix-up) -> every seed's first turn record.
//   3. synth_write: regenerates every turn record of every program at its final position.
#include "ct_device.cuh"
#include "ct_internal.h"

namespace ct {

namespace {

constexpr uint64_t KEY0 = 0x243F6A8885A308D3ull;
constexpr uint64_t MIX_KEY = 0xC1A55;

__device__ __forceinline__ uint64_t splitmix(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t key4(uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
  return splitmix(splitmix(splitmix(splitmix(KEY0 ^ a) ^ b) ^ c) ^ d);
}
__device__ __forceinline__ uint64_t key5(uint64_t a, uint64_t b, uint64_t c, uint64_t d, uint64_t e) {
  return splitmix(key4(a, b, c, d) ^ e);
}
// uniform(h, n) = (u(h) n) >> 32
__device__ __forceinline__ int64_t uni(uint64_t h, uint32_t n) {
  return (int64_t)(((h >> 32) * (uint64_t)n) >> 32);
}
// quantile(T, h) = T[i] + (((T[i+1] - T[i]) f) >> 16), i = u >> 22, f = (u >> 6) & 0xFFFF
__device__ __forceinline__ int64_t quant(const int64_t* T, uint64_t h) {
  const uint32_t u = (uint32_t)(h >> 32);
  const int i = (int)(u >> 22);
  const int64_t f = (int64_t)((u >> 6) & 0xFFFFu);
  const int64_t lo = __ldg(T + i), hi = __ldg(T + i + 1);
  return lo + (((hi - lo) * f) >> 16);
}

struct SynthArgs {
  uint64_t stream;
  int64_t ctx_cap;
  int max_turns, n_bfcl, F, P, n_seeds;
  int64_t seed0;
  const int64_t* tab;  // [turns_swe | obs SWE, BFCL | dec SWE, BFCL | exp | dur 0..F-1] x 1025
  const uint32_t* cdf;
  const int32_t* cls;
  ct_program* progs;
  ct_turn* turns;
  uint8_t* pcls;       // [S * P] class per program (pass 1 -> pass 3)
  int64_t* seed_tot;   // [S] turns per seed -> exclusive offsets
  int64_t* blk;        // [ceil(S / 1024)] block totals -> block offsets
};
constexpr int T_SWE = 0, T_OBS = CT_SYNTH_TABLE, T_DEC = 3 * CT_SYNTH_TABLE, T_EXP = 5 * CT_SYNTH_TABLE,
              T_DUR = 6 * CT_SYNTH_TABLE;

__device__ __forceinline__ int32_t gen_new(const SynthArgs& a, uint64_t s, uint64_t p, uint64_t t, int c) {
  if (t == 0) {
    const uint64_t h = key5(a.stream, s, p, 0, 10);
    return (int32_t)(c ? (2 * (1000 + uni(h, 2001))) / 5 : 1500 + uni(h, 2501));
  }
  return (int32_t)quant(a.tab + T_OBS + c * CT_SYNTH_TABLE, key5(a.stream, s, p, t, 11));
}
__device__ __forceinline__ int32_t gen_dec(const SynthArgs& a, uint64_t s, uint64_t p, uint64_t t, int c) {
  return (int32_t)quant(a.tab + T_DEC + c * CT_SYNTH_TABLE, key5(a.stream, s, p, t, 15));
}

constexpr int SW = 4;  // warps per block in the per-seed passes

__global__ void __launch_bounds__(32 * SW) synth_count_kernel(SynthArgs a) {
  __shared__ uint64_t keys[SW][CT_MAX_PROGRAMS];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int P = a.P;
  for (int64_t si = (int64_t)blockIdx.x * SW + w; si < a.n_seeds; si += (int64_t)gridDim.x * SW) {
    const uint64_t s = (uint64_t)(a.seed0 + si);
    for (int p = lane; p < P; p += 32) keys[w][p] = key4(a.stream, s, (uint64_t)p, MIX_KEY);
    __syncwarp();
    int64_t carry_arr = 0, carry_off = 0;
    for (int base = 0; base < P; base += 32) {
      const int p = base + lane;
      int64_t g = 0, nt2 = 0;
      if (p < P) {
        const uint64_t kp = keys[w][p];
        int rank = 0;
        for (int q = 0; q < P; ++q) {
          const uint64_t kq = keys[w][q];
          rank += kq < kp || (kq == kp && q < p);
        }
        const int c = rank < a.n_bfcl ? 1 : 0;
        a.pcls[si * P + p] = (uint8_t)c;
        int64_t nt = c ? 2 + uni(key4(a.stream, s, p, 3), 9) : quant(a.tab + T_SWE, key4(a.stream, s, p, 1));
        nt = min(nt, (int64_t)a.max_turns);
        int64_t cum = 0;
        for (int64_t t = 0; t < nt; ++t) {  // R24: leading turns whose cumulative tokens fit
          cum += gen_new(a, s, p, t, c) + gen_dec(a, s, p, t, c);
          if (cum > a.ctx_cap) break;
          ++nt2;
        }
        g = quant(a.tab + T_EXP, key4(a.stream, s, p, 30));
      }
      // inclusive prefix of the arrival gaps, exclusive prefix of the turn counts
      int64_t ig = g, io = nt2;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t xg = __shfl_up_sync(FULL_MASK, ig, o), xo = __shfl_up_sync(FULL_MASK, io, o);
        if (lane >= o) { ig += xg; io += xo; }
      }
      if (p < P) {
        ct_program pr;
        pr.arr_q = carry_arr + ig;
        pr.turn0 = (int32_t)(carry_off + io - nt2);  // offset inside the seed (pass 3 rebases)
        pr.nturns = (int32_t)nt2;
        a.progs[si * P + p] = pr;
      }
      carry_arr += __shfl_sync(FULL_MASK, ig, 31);
      carry_off += __shfl_sync(FULL_MASK, io, 31);
    }
    if (lane == 0) a.seed_tot[si] = carry_off;
    __syncwarp();
  }
}

// exclusive scan of v[0..n) in place within each 1024-element block; block totals -> blk
__global__ void __launch_bounds__(1024) scan_block_kernel(int64_t* v, int64_t n, int64_t* blk) {
  __shared__ int64_t ws[32];
  const int64_t i = (int64_t)blockIdx.x * 1024 + threadIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t x = i < n ? v[i] : 0;
  int64_t inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(FULL_MASK, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) ws[w] = inc;
  __syncthreads();
  if (w == 0) {
    int64_t t = ws[lane], ti = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(FULL_MASK, ti, o);
      if (lane >= o) ti += y;
    }
    ws[lane] = ti - t;  // exclusive over warps
    if (lane == 31) blk[blockIdx.x] = ti;
  }
  __syncthreads();
  if (i < n) v[i] = ws[w] + inc - x;
}

// exclusive scan of the block totals (one CTA, any count) -> blk; the grand total -> blk[nb]
__global__ void __launch_bounds__(1024) scan_totals_kernel(int64_t* blk, int64_t nb) {
  __shared__ int64_t ws[32];
  __shared__ int64_t carry;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < nb; base += 1024) {
    const int64_t i = base + threadIdx.x;
    const int64_t x = i < nb ? blk[i] : 0;
    int64_t inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(FULL_MASK, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) ws[w] = inc;
    __syncthreads();
    if (w == 0) {
      int64_t t = ws[lane], ti = t;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(FULL_MASK, ti, o);
        if (lane >= o) ti += y;
      }
      ws[lane] = ti - t;
    }
    __syncthreads();
    const int64_t c = carry;
    if (i < nb) blk[i] = c + ws[w] + inc - x;
    __syncthreads();
    if (threadIdx.x == 1023) carry = c + ws[w] + inc;
    __syncthreads();
  }
  if (threadIdx.x == 0) blk[nb] = carry;
}

__global__ void __launch_bounds__(32 * SW) synth_write_kernel(SynthArgs a) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int P = a.P;
  for (int64_t si = (int64_t)blockIdx.x * SW + w; si < a.n_seeds; si += (int64_t)gridDim.x * SW) {
    const uint64_t s = (uint64_t)(a.seed0 + si);
    const int64_t off = a.seed_tot[si] + a.blk[si >> 10];
    for (int p = lane; p < P; p += 32) {
      ct_program* pr = a.progs + si * P + p;
      const int64_t t0 = off + pr->turn0;
      const int nt2 = pr->nturns;
      pr->turn0 = (int32_t)t0;
      const int c = a.pcls[si * P + p];
      for (int t = 0; t < nt2; ++t) {
        ct_turn r;
        r.new_tokens = gen_new(a, s, p, t, c);
        r.decode_tokens = gen_dec(a, s, p, t, c);
        if (t == nt2 - 1) {
          r.tool = -1;
          r.dur_us = 0;
        } else {
          const uint32_t u = (uint32_t)(key5(a.stream, s, p, t, 20) >> 32);
          int tool = -1, lastc = -1;
          for (int f = 0; f < a.F; ++f) {
            if (__ldg(a.cls + f) != c) continue;
            lastc = f;
            if (tool < 0 && u < __ldg(a.cdf + f)) tool = f;
          }
          if (tool < 0) tool = lastc;
          r.tool = tool;
          r.dur_us = (int32_t)quant(a.tab + T_DUR + tool * CT_SYNTH_TABLE, key5(a.stream, s, p, t, 21));
        }
        a.turns[t0 + t] = r;
      }
    }
  }
}

}  // namespace

cudaError_t launch_synth(const SynthLaunch& L, int sm_count, cudaStream_t st, int64_t* total_host) {
  SynthArgs a;
  a.stream = (uint64_t)L.sp->stream;
  a.ctx_cap = L.sp->ctx_cap;
  a.max_turns = L.sp->max_turns;
  a.n_bfcl = L.sp->n_bfcl;
  a.F = L.sp->n_tools;
  a.P = L.P;
  a.n_seeds = L.n_seeds;
  a.seed0 = L.seed0;
  a.tab = L.tab;
  a.cdf = L.cdf;
  a.cls = L.cls;
  a.progs = L.progs;
  a.turns = L.turns;
  a.pcls = L.pcls;
  a.seed_tot = L.seed_tot;
  a.blk = L.blk;
  const int grid = (int)std::min<int64_t>((L.n_seeds + SW - 1) / SW, (int64_t)sm_count * 16);
  synth_count_kernel<<<grid, 32 * SW, 0, st>>>(a);
  const int64_t nb = (L.n_seeds + 1023) / 1024;
  scan_block_kernel<<<(unsigned)nb, 1024, 0, st>>>(a.seed_tot, L.n_seeds, a.blk);
  scan_totals_kernel<<<1, 1024, 0, st>>>(a.blk, nb);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  e = cudaMemcpyAsync(total_host, a.blk + nb, 8, cudaMemcpyDeviceToHost, st);
  if (e != cudaSuccess) return e;
  e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return e;
  if (*total_host > L.turns_cap) return cudaSuccess;  // the caller reports CT_EINVAL
  synth_write_kernel<<<grid, 32 * SW, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace ct
