// ttl_fit.cu — the TTL fit: one HBM pass over duration samples.
//
// Kernel 1 (fit_hist): one CTA of 8 warps per resident slot streams one contiguous range of the
// tool-grouped (CSR) int32 samples with 16-B streaming loads (register double buffering, 8 int4
// in flight per lane), cut into pieces at tool boundaries.
// Every sample lands in the CTA's histogram over the TTL grid buckets k = min(ceil(d / step), K)
// as (count, sum of k step - d) with fire-and-forget 32-bit shared reductions; the histogram has
// one replica per lane index shared by the CTA's warps, so a warp instruction never conflicts.
// Each thread keeps the paper-mode statistics (sum t~, sum t~^2) of t~ = min(d, b) in registers
// (reading R5).  After each chunk the replicas are merged and flushed with
// integer atomics (order independent, hence deterministic).  Older chunked variants remain
// selectable for measurement (CT_FIT_VARIANT).
// Kernel 2 (fit_scan): one CTA per tool row: block prefix scan of the bucket counts and sums in
// shared memory, then per turn bucket j n U(k) in 128-bit integers (extension C-4) and a warp
// argmax with the smallest k on ties; the pooled row sums the tool rows; tools with n_f < N take
// the pooled result; thread 0 also evaluates CalcTTL on the row's statistics.
#include <algorithm>
#include <cstdlib>

#include "ct_device.cuh"
#include "ct_internal.h"

namespace ct {

// TMA-staged variant (fit_hist_tma_kernel)
constexpr int TMA_THREADS = 1024;
constexpr int TMA_CW = 31;                     // consumer warps
constexpr int TMA_CT = 32 * TMA_CW;            // consumer threads
constexpr int TMA_U = 2;                       // int4 per consumer thread per stage
constexpr int TMA_STAGE = TMA_CT * 16 * TMA_U;  // bytes per stage (every consumer thread busy)
constexpr int TMA_MAX_STAGES = 8;
// per-warp TMA variant (fit_hist_wtma_kernel): warps, bytes per chunk, ring slots per warp
constexpr int WTMA_W = 20, WTMA_B = 2048, WTMA_S = 3;
constexpr int FIT_WARPS = 2;                 // warps per CTA; every warp is independent
constexpr int FIT_THREADS = 32 * FIT_WARPS;

// Histogram variants (replicas per warp, 16-bit packed counts).  A replica is shared by 32/REPL
// adjacent lanes; layout [bucket][replica] spreads one bucket over REPL banks.
struct FitVariant {
  int repl;
  bool pack;
  int u;  // int4 loads per lane per double-buffer half
};
static const FitVariant kVariants[] = {{16, false, 16}, {16, true, 16}, {8, false, 8},
                                       {8, true, 8},    {32, false, 16}, {16, true, 8},
                                       {8, true, 4},    {4, false, 8},   {4, false, 4},
                                       {8, false, 4},   {32, false, 4},   // 10: CTA-shared, U 4
                                       {32, false, 8},                    // 11: CTA-shared, U 8
                                       {32, false, 8},                    // 12: 11 + 32-bit sums
                                       {32, false, 4},                    // 13: 12 with U 4
                                       {32, false, 6},                    // 14: 12 with U 6
                                       {32, false, 8},                    // 15: 12, CTA ranges
                                       {32, false, 8},                    // 16: 11, CTA ranges
                                       {32, false, 0},                    // 17: 15, TMA-staged
                                       {32, false, 0},                    // 18: 16, TMA-staged
                                       {32, false, 0},                    // 19: 15, per-warp TMA
                                       {32, false, 0},                    // 20: 16, per-warp TMA
                                       {32, false, 0},                    // 21: cp.async 16 w x 4 x 1 KB
                                       {32, false, 0}};                   // 22: 21, no 32-bit sums
constexpr int N_VARIANTS = sizeof kVariants / sizeof kVariants[0];
static int g_variant = -1;  // default 15: measured best on B200 (DESIGN.md §8 variant table)

static int variant() {
  static_assert(N_VARIANTS == 23, "variant table / hist_fn mismatch");
  if (g_variant < 0) {
    const char* e = getenv("CT_FIT_VARIANT");
    int v = e ? atoi(e) : 15;
    g_variant = (v >= 0 && v < N_VARIANTS) ? v : 15;
  }
  return g_variant;
}

static int smem_words(int K, const FitVariant& fv) {
  return (K + 1) * (fv.repl + (fv.pack ? fv.repl / 2 : fv.repl));
}
constexpr int SMEM_LIMIT = 232448 - 2048;  // B200 opt-in per-block shared memory, minus static

// Variant choice for one call: the selected variant, its 32-bit-sum-free twin when b >= 2^26 µs,
// fewer TMA stages or the per-warp 4-replica kernel when the histogram does not fit.
FitPlan fit_plan(int K, int64_t b_us) {
  int v = variant();
  if (b_us >= (1ll << 26)) {  // 32-bit partial sums need b < 2^26 µs
    if (v == 12 || v == 13 || v == 14) v = 11;
    if (v == 15) v = 16;
    if (v == 17) v = 18;
    if (v == 19) v = 20;
    if (v == 21) v = 22;
  }
  FitPlan p;
  p.stages = 0;
  const int hist = (K + 1) * 64 * 4;
  const int aw = 16;  // cp.async variants: warps per CTA, 4 x 1 KB ring per warp
  if (v >= 21) {
    if (hist + aw * 4096 > SMEM_LIMIT) v = 8;
  } else if (v >= 19) {
    if (hist + WTMA_W * WTMA_S * (WTMA_B + 8) > SMEM_LIMIT) v = 8;
  } else if (v >= 17) {
    p.stages = std::min(TMA_MAX_STAGES, (SMEM_LIMIT - hist) / (TMA_STAGE + 16));
    if (p.stages < 2) v = 8;
  } else if (v >= 10 && hist > SMEM_LIMIT) {
    v = 8;
  }
  p.v = v;
  p.cta = v >= 10;
  p.ranges = v >= 15;
  p.repl = kVariants[v].repl;
  p.threads = v >= 21 ? 32 * aw : v >= 19 ? 32 * WTMA_W : v >= 17 ? TMA_THREADS : v >= 10 ? 256 : FIT_THREADS;
  p.smem = v >= 21   ? hist + aw * 4096
           : v >= 19 ? hist + WTMA_W * WTMA_S * (WTMA_B + 8)
           : v >= 17 ? hist + p.stages * (TMA_STAGE + 16)
                     : v >= 10 ? hist : FIT_WARPS * 4 * smem_words(K, kVariants[v]);
  return p;
}

__device__ __forceinline__ void red_shared(uint32_t addr, uint32_t v) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

__device__ __forceinline__ void mad_wide(uint64_t& acc, uint32_t a, uint32_t b) {
  asm("mad.wide.u32 %0, %1, %2, %0;" : "+l"(acc) : "r"(a), "r"(b));
}

struct Lane {
  uint32_t rs_base, cnt_base, cnt_inc;  // shared-window addresses of this lane's replica
  uint32_t K, step, mhi, mlo, xoff, b_us;
  uint32_t dm, dsh, dadd;  // 32-bit Granlund-Montgomery divisor (CTA-shared kernels)
};

// One sample d of the lane.  Bucket k = min(ceil(d / step), K) (a hit for tau_k iff d <= k step);
// the bins keep the count and the sum of r = k step - d in [0, step), so sum_k d =
// k step count_k - sum_k r is exact with 32-bit bins.  ceil(d / step) = floor(x / step) with
// x = d + step - 1 < 2^32 is the high word of x * M, M = ceil(2^64 / step) (error < 2^-32 cannot
// cross an integer for 32-bit x): one IMAD.HI + one IMAD.WIDE; step = 1 is the identity.
template <bool IDENT, int REPL, bool PACK>
__device__ __forceinline__ void sample(const Lane& L, int32_t d, uint64_t& s1, uint64_t& s2) {
  const uint32_t x = (uint32_t)d + L.xoff;
  uint32_t q;
  if (IDENT) {
    q = x;
  } else {
    uint64_t p = __umulhi(x, L.mlo);
    mad_wide(p, x, L.mhi);  // p = x * mhi + hi32(x * mlo)
    q = (uint32_t)(p >> 32);
  }
  const uint32_t b = min(q, L.K);
  const uint32_t r = b * L.step - (uint32_t)d;  // in [0, step) for b < K; ignored for b = K
  red_shared(L.cnt_base + b * ((PACK ? REPL / 2 : REPL) * 4), L.cnt_inc);
  red_shared(L.rs_base + b * (REPL * 4), r);
  const uint32_t t = min((uint32_t)d, L.b_us);
  s1 += t;
  mad_wide(s2, t, t);
}

template <bool IDENT, int REPL, bool PACK, int U>
__global__ void __launch_bounds__(FIT_THREADS) fit_hist_kernel(FitArgs a) {
  extern __shared__ __align__(16) uint32_t hsm[];
  constexpr int CW = PACK ? REPL / 2 : REPL;  // count words per bucket
  const int K = a.K;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int words = (K + 1) * (REPL + CW);
  uint32_t* rs = hsm + warp * words;
  uint32_t* cnt = rs + (K + 1) * REPL;
  const int rep = lane / (32 / REPL);
  Lane L;
  L.rs_base = (uint32_t)__cvta_generic_to_shared(rs) + 4 * rep;
  L.cnt_base = (uint32_t)__cvta_generic_to_shared(cnt) + 4 * (PACK ? rep >> 1 : rep);
  L.cnt_inc = PACK ? (1u << (16 * (rep & 1))) : 1u;
  L.K = (uint32_t)K;
  L.step = (uint32_t)a.step;
  L.mhi = (uint32_t)(a.step_magic >> 32);
  L.mlo = (uint32_t)a.step_magic;
  L.xoff = L.step - 1;
  L.b_us = (uint32_t)a.b_us;
  const int64_t gw = (int64_t)blockIdx.x * FIT_WARPS + warp, nw = (int64_t)gridDim.x * FIT_WARPS;

  for (int64_t c = gw; c < a.n_chunks; c += nw) {
    int tool = 0;
    while (a.chunk_off[tool + 1] <= c) ++tool;
    const int64_t beg = a.tool_off[tool] + (c - a.chunk_off[tool]) * a.ch;
    const int64_t end = min(beg + a.ch, a.tool_off[tool + 1]);
    for (int i = lane; i < words; i += 32) rs[i] = 0;
    __syncwarp();
    uint64_t s1 = 0, s2 = 0;
    int64_t va = (beg + 3) & ~(int64_t)3;
    if (va > end) va = end;
    const int64_t vb = va + ((end - va) & ~(int64_t)3);
    // scalar head and tail (< 4 samples each)
    if (beg + lane < va) sample<IDENT, REPL, PACK>(L, __ldg(&a.dur[beg + lane]), s1, s2);
    if (vb + lane < end) sample<IDENT, REPL, PACK>(L, __ldg(&a.dur[vb + lane]), s1, s2);
    const int4* v = (const int4*)(a.dur + va);
    const int64_t nv = (vb - va) >> 2;
    // register double buffering: U int4 per lane in flight while the previous U are binned
    int64_t i = lane;
    int4 A[U], B[U];
    bool have_a = i + (U - 1) * 32 < nv;
    if (have_a) {
#pragma unroll
      for (int u = 0; u < U; ++u) A[u] = __ldcs(v + i + u * 32);
    }
    while (have_a) {
      const int64_t ib = i + U * 32;
      const bool have_b = ib + (U - 1) * 32 < nv;
      if (have_b) {
#pragma unroll
        for (int u = 0; u < U; ++u) B[u] = __ldcs(v + ib + u * 32);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        sample<IDENT, REPL, PACK>(L, A[u].x, s1, s2);
        sample<IDENT, REPL, PACK>(L, A[u].y, s1, s2);
        sample<IDENT, REPL, PACK>(L, A[u].z, s1, s2);
        sample<IDENT, REPL, PACK>(L, A[u].w, s1, s2);
      }
      i = ib;
      if (!have_b) break;
      const int64_t ia = ib + U * 32;
      have_a = ia + (U - 1) * 32 < nv;
      if (have_a) {
#pragma unroll
        for (int u = 0; u < U; ++u) A[u] = __ldcs(v + ia + u * 32);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        sample<IDENT, REPL, PACK>(L, B[u].x, s1, s2);
        sample<IDENT, REPL, PACK>(L, B[u].y, s1, s2);
        sample<IDENT, REPL, PACK>(L, B[u].z, s1, s2);
        sample<IDENT, REPL, PACK>(L, B[u].w, s1, s2);
      }
      i = ia;
    }
    for (; i < nv; i += 32) {
      const int4 x = __ldcs(v + i);
      sample<IDENT, REPL, PACK>(L, x.x, s1, s2);
      sample<IDENT, REPL, PACK>(L, x.y, s1, s2);
      sample<IDENT, REPL, PACK>(L, x.z, s1, s2);
      sample<IDENT, REPL, PACK>(L, x.w, s1, s2);
    }
    // statistics: n is the chunk length; sum t~^2 split into 32-bit limb sums (fit_scan renormalises)
    const uint64_t w1 = warp_sum_u64(s1), w2 = warp_sum_u64(s2 & 0xffffffffull),
                   w3 = warp_sum_u64(s2 >> 32);
    if (lane < 2) {  // lane 0: the tool's row, lane 1: the pooled row F
      unsigned long long* st = a.stat + (lane == 0 ? tool : a.F) * 6;
      atomicAdd(st + 0, (unsigned long long)(end - beg));
      if (w1) atomicAdd(st + 1, (unsigned long long)w1);
      if (w2) atomicAdd(st + 2, (unsigned long long)w2);
      if (w3) atomicAdd(st + 3, (unsigned long long)w3);
    }
    __syncwarp();
    // merge the replicas and flush: sum_k d = k step count_k - sum_k r (k < K)
    for (int b = lane; b <= K; b += 32) {
      uint64_t cn = 0, rr = 0;
#pragma unroll
      for (int q = 0; q < REPL; ++q) rr += rs[b * REPL + q];
#pragma unroll
      for (int q = 0; q < CW; ++q) {
        const uint32_t w = cnt[b * CW + q];
        cn += PACK ? (uint64_t)(w & 0xffffu) + (w >> 16) : (uint64_t)w;
      }
      if (cn) {
        const uint64_t sm = b < K ? (uint64_t)b * L.step * cn - rr : 0;
#pragma unroll
        for (int row2 = 0; row2 < 2; ++row2) {  // the tool's row and the pooled row F
          const int64_t o = (int64_t)(row2 ? a.F : tool) * (K + 1) + b;
          atomicAdd(&a.hcnt[o], (unsigned long long)cn);
          if (sm) atomicAdd(&a.hsum[o], (unsigned long long)sm);
        }
      }
    }
    __syncwarp();
  }
}

// CTA-shared variant: the CTA's FW warps share one histogram with one replica per lane index,
// laid out [bucket][count x 32 | remainder x 32]: within a warp instruction the 32 lanes always
// hit 32 distinct banks (no conflicts, no same-address serialisation, even for a point mass),
// while the footprint per warp is 1/FW of a lane-private histogram.  Chunks are CTA-level.
constexpr int FW = 8;

// CTA-kernel sample: count at [base + 256 b], remainder at +128 (one address, immediate offset);
// the caller keeps 4 independent 64-bit sum-of-squares accumulators (ILP for the accumulate form
// of IMAD.WIDE) and, when b < 2^26, a 32-bit sum accumulator flushed every 32 samples.
//
// The quotient uses a 32-bit Granlund-Montgomery divisor (one IMAD.HI plus shifts and adds on
// the ALU pipe; FitArgs.div_*), exact for every 32-bit x: the fma pipe, which also carries the
// remainder and the sum of squares, is the kernel's busiest.
template <bool IDENT, typename S1>
__device__ __forceinline__ void sample_cta(const Lane& L, uint32_t base, int32_t d, S1& s1,
                                           uint64_t& s2) {
  const uint32_t x = (uint32_t)d + L.xoff;
  uint32_t q;
  if (IDENT) {
    q = x;
  } else {
    const uint32_t t = __umulhi(x, L.dm);
    q = L.dadd ? ((((x - t) >> 1) + t) >> L.dsh) : (t >> L.dsh);
  }
  const uint32_t b = min(q, L.K);
  const uint32_t addr = base + (b << 8);
  red_shared(addr, 1u);
  red_shared(addr + 128u, b * L.step - (uint32_t)d);
  const uint32_t t = min((uint32_t)d, L.b_us);
  s1 += t;
  mad_wide(s2, t, t);
}

__device__ __forceinline__ Lane cta_lane(const FitArgs& a, uint32_t* hsm) {
  Lane L;
  L.rs_base = (uint32_t)__cvta_generic_to_shared(hsm) + 4 * (threadIdx.x & 31) + 128;  // remainders
  L.cnt_base = L.rs_base - 128;                                                        // counts
  L.cnt_inc = 1u;
  L.K = (uint32_t)a.K;
  L.step = (uint32_t)a.step;
  L.mhi = (uint32_t)(a.step_magic >> 32);
  L.mlo = (uint32_t)a.step_magic;
  L.xoff = L.step - 1;
  L.b_us = (uint32_t)a.b_us;
  L.dm = a.div_m;
  L.dsh = a.div_sh;
  L.dadd = a.div_add;
  return L;
}

// One CTA work piece: samples [beg, end) of one tool -> zeroed CTA histogram -> flush.
template <bool IDENT, int U, bool FAST32>
__device__ __forceinline__ void cta_piece(const FitArgs& a, const Lane& L, uint32_t* hsm,
                                          unsigned long long (*red)[3], int tool, int64_t beg,
                                          int64_t end) {
  const int K = a.K;
  const int tid = threadIdx.x, lane = tid & 31;
  const int words = (K + 1) * 64;
  {
    for (int i = tid; i < words; i += 32 * FW) hsm[i] = 0;
    __syncthreads();
    uint64_t s1 = 0, s2 = 0;
    int64_t va = (beg + 3) & ~(int64_t)3;
    if (va > end) va = end;
    const int64_t vb = va + ((end - va) & ~(int64_t)3);
    if (tid < 32) {
      if (beg + lane < va) sample<IDENT, 64, false>(L, __ldg(&a.dur[beg + lane]), s1, s2);
      if (vb + lane < end) sample<IDENT, 64, false>(L, __ldg(&a.dur[vb + lane]), s1, s2);
    }
    const int4* v = (const int4*)(a.dur + va);
    const int64_t nv = (vb - va) >> 2;
    constexpr int T = 32 * FW;
    const uint32_t base = L.cnt_base;
    uint64_t q1 = 0, q2 = 0, q3 = 0;  // extra sum-of-squares accumulators (ILP)
    uint32_t s1w = 0;                  // 32-bit partial sum, flushed per 4U samples (b < 2^26)
    auto run4 = [&](const int4& x) {
      if (FAST32) {
        sample_cta<IDENT>(L, base, x.x, s1w, s2);
        sample_cta<IDENT>(L, base, x.y, s1w, q1);
        sample_cta<IDENT>(L, base, x.z, s1w, q2);
        sample_cta<IDENT>(L, base, x.w, s1w, q3);
      } else {
        sample_cta<IDENT>(L, base, x.x, s1, s2);
        sample_cta<IDENT>(L, base, x.y, s1, q1);
        sample_cta<IDENT>(L, base, x.z, s1, q2);
        sample_cta<IDENT>(L, base, x.w, s1, q3);
      }
    };
    int64_t i = tid;
    int4 A[U], B[U];
    bool have_a = i + (U - 1) * T < nv;
    if (have_a) {
#pragma unroll
      for (int u = 0; u < U; ++u) A[u] = __ldcs(v + i + u * T);
    }
    while (have_a) {
      const int64_t ib = i + U * T;
      const bool have_b = ib + (U - 1) * T < nv;
      if (have_b) {
#pragma unroll
        for (int u = 0; u < U; ++u) B[u] = __ldcs(v + ib + u * T);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) run4(A[u]);
      if (FAST32) { s1 += s1w; s1w = 0; }
      i = ib;
      if (!have_b) break;
      const int64_t ia = ib + U * T;
      have_a = ia + (U - 1) * T < nv;
      if (have_a) {
#pragma unroll
        for (int u = 0; u < U; ++u) A[u] = __ldcs(v + ia + u * T);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) run4(B[u]);
      if (FAST32) { s1 += s1w; s1w = 0; }
      i = ia;
    }
    for (; i < nv; i += T) {
      run4(__ldcs(v + i));
      if (FAST32) { s1 += s1w; s1w = 0; }
    }
    s2 += q1 + q2 + q3;
    const uint64_t w1 = warp_sum_u64(s1), w2 = warp_sum_u64(s2 & 0xffffffffull),
                   w3 = warp_sum_u64(s2 >> 32);
    if (lane == 0) { red[tid >> 5][0] = w1; red[tid >> 5][1] = w2; red[tid >> 5][2] = w3; }
    __syncthreads();
    if (tid < 6) {  // tid 0-2: the tool's row, 3-5: the pooled row F
      const int q = tid % 3;
      uint64_t sum = 0;
#pragma unroll
      for (int w = 0; w < FW; ++w) sum += red[w][q];
      unsigned long long* st = a.stat + (tid < 3 ? tool : a.F) * 6;
      if (q == 0) atomicAdd(st, (unsigned long long)(end - beg));
      if (sum) atomicAdd(st + 1 + q, (unsigned long long)sum);
    }
    // merge the 32 lane replicas of every bucket and flush (tool row + pooled row)
    for (int b = tid; b <= K; b += T) {
      const uint4* pc = (const uint4*)(hsm + b * 64);
      uint64_t cn = 0, rr = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint4 x = pc[q], y = pc[8 + q];
        cn += (uint64_t)x.x + x.y + x.z + x.w;
        rr += (uint64_t)y.x + y.y + y.z + y.w;
      }
      if (cn) {
        const uint64_t sm = b < K ? (uint64_t)b * L.step * cn - rr : 0;
#pragma unroll
        for (int row2 = 0; row2 < 2; ++row2) {
          const int64_t o = (int64_t)(row2 ? a.F : tool) * (K + 1) + b;
          atomicAdd(&a.hcnt[o], (unsigned long long)cn);
          if (sm) atomicAdd(&a.hsum[o], (unsigned long long)sm);
        }
      }
    }
    __syncthreads();
  }
}

template <bool IDENT, int U, bool FAST32>
__global__ void __launch_bounds__(32 * FW) fit_hist_cta_kernel(FitArgs a) {
  extern __shared__ __align__(16) uint32_t hsm[];
  __shared__ unsigned long long red[FW][3];
  const Lane L = cta_lane(a, hsm);
  for (int64_t c = blockIdx.x; c < a.n_chunks; c += gridDim.x) {
    int tool = 0;
    while (a.chunk_off[tool + 1] <= c) ++tool;
    const int64_t beg = a.tool_off[tool] + (c - a.chunk_off[tool]) * a.ch;
    const int64_t end = min(beg + a.ch, a.tool_off[tool + 1]);
    cta_piece<IDENT, U, FAST32>(a, L, hsm, red, tool, beg, end);
  }
}

// Contiguous-range variant: CTA b streams samples [bnd(b), bnd(b+1)) of the whole CSR array
// (boundaries 4-aligned, so only tool boundaries have scalar heads/tails), cut into pieces at
// tool boundaries and every ch samples (the 32-bit bin bound).  A CTA therefore zeroes and
// flushes its histogram ~once instead of once per 2^17-sample chunk.
template <bool IDENT, int U, bool FAST32>
__global__ void __launch_bounds__(32 * FW) fit_hist_seg_kernel(FitArgs a) {
  extern __shared__ __align__(16) uint32_t hsm[];
  __shared__ unsigned long long red[FW][3];
  const Lane L = cta_lane(a, hsm);
  const int64_t s0 = a.tool_off[0], s1 = a.tool_off[a.F];
  const int64_t per = (s1 - s0 + gridDim.x - 1) / gridDim.x;
  auto bnd = [&](int64_t b) -> int64_t {
    if (b == 0) return s0;
    if (b >= (int64_t)gridDim.x) return s1;
    return min(s1, max(s0, (s0 + b * per) & ~(int64_t)3));
  };
  int64_t lo = bnd(blockIdx.x);
  const int64_t hi = bnd((int64_t)blockIdx.x + 1);
  int tool = 0;
  while (lo < hi) {
    while (a.tool_off[tool + 1] <= lo) ++tool;
    const int64_t end = min(min(hi, a.tool_off[tool + 1]), lo + a.ch);
    cta_piece<IDENT, U, FAST32>(a, L, hsm, red, tool, lo, end);
    lo = end;
  }
}

// ---------------------------------------------------------------------------------------------
// TMA-staged variant: one CTA of 32 warps per SM.  Warp 31's elected lane streams the CTA's
// contiguous sample range into a ring of `stages` 31-KB shared-memory buffers with 1-D bulk
// copies (cp.async.bulk ... mbarrier::complete_tx), so up to stages x 31 KB per SM are in flight
// without holding registers; warps 0-30 consume each buffer (ld.shared.v4) into the same
// lane-indexed CTA histogram as the register-staged kernels and release it through an "empty"
// mbarrier.  Pieces (tool boundaries, the 32-bit bin bound) are cut exactly as in
// fit_hist_seg_kernel; producer and consumers walk the same piece/stage schedule.

__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(a), "r"(parity) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t a) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t a, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(mbar)
      : "memory");
}
__device__ __forceinline__ void consumer_bar() {  // named barrier over the consumer warps only
  asm volatile("bar.sync 1, %0;" ::"n"(TMA_CT) : "memory");
}

template <bool IDENT, bool FAST32>
__global__ void __launch_bounds__(TMA_THREADS, 1) fit_hist_tma_kernel(FitArgs a) {
  extern __shared__ __align__(128) uint32_t hsm[];
  __shared__ unsigned long long red[TMA_CW][3];
  const int K = a.K, S = a.stages;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int words = (K + 1) * 64;
  unsigned char* ring = (unsigned char*)(hsm + words);  // 16-B aligned: words is a multiple of 64
  const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(ring);
  const uint32_t full0 = ring_s + S * TMA_STAGE;  // S full barriers, then S empty barriers
  const uint32_t empty0 = full0 + 8 * S;
  if (tid == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(full0 + 8 * i, 1);
      mbar_init(empty0 + 8 * i, TMA_CW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const Lane L = cta_lane(a, hsm);
  const int64_t s0 = a.tool_off[0], s1e = a.tool_off[a.F];
  const int64_t per = (s1e - s0 + gridDim.x - 1) / gridDim.x;
  auto bnd = [&](int64_t b) -> int64_t {
    if (b == 0) return s0;
    if (b >= (int64_t)gridDim.x) return s1e;
    return min(s1e, max(s0, (s0 + b * per) & ~(int64_t)3));
  };
  const int64_t lo0 = bnd(blockIdx.x), hi = bnd((int64_t)blockIdx.x + 1);

  if (warp == TMA_CW) {  // ---- producer ----
    if (lane == 0) {
      int slot = 0;
      uint32_t ph = 0;
      int64_t issued = 0;
      int64_t lo = lo0;
      int tool = 0;
      while (lo < hi) {
        while (a.tool_off[tool + 1] <= lo) ++tool;
        const int64_t end = min(min(hi, a.tool_off[tool + 1]), lo + a.ch);
        int64_t va = (lo + 3) & ~(int64_t)3;
        if (va > end) va = end;
        const int64_t vb = va + ((end - va) & ~(int64_t)3);
        const unsigned char* src = (const unsigned char*)(a.dur + va);
        for (int64_t off = 0, nb = 4 * (vb - va); off < nb; off += TMA_STAGE) {
          const uint32_t bytes = (uint32_t)min((int64_t)TMA_STAGE, nb - off);
          if (issued >= S) mbar_wait(empty0 + 8 * slot, ph ^ 1u);
          mbar_expect_tx(full0 + 8 * slot, bytes);
          bulk_g2s(ring_s + slot * TMA_STAGE, src + off, bytes, full0 + 8 * slot);
          ++issued;
          if (++slot == S) { slot = 0; ph ^= 1u; }
        }
        lo = end;
      }
    }
    return;
  }

  // ---- consumers ----
  int slot = 0;
  uint32_t ph = 0;
  int64_t lo = lo0;
  int tool = 0;
  while (lo < hi) {
    while (a.tool_off[tool + 1] <= lo) ++tool;
    const int64_t beg = lo;
    const int64_t end = min(min(hi, a.tool_off[tool + 1]), lo + a.ch);
    lo = end;
    for (int i = tid; i < words; i += TMA_CT) hsm[i] = 0;
    consumer_bar();
    uint64_t s1 = 0, s2 = 0, q1 = 0, q2 = 0, q3 = 0;
    int64_t va = (beg + 3) & ~(int64_t)3;
    if (va > end) va = end;
    const int64_t vb = va + ((end - va) & ~(int64_t)3);
    if (tid < 32) {  // scalar head and tail (< 4 samples each)
      if (beg + lane < va) sample<IDENT, 64, false>(L, __ldg(&a.dur[beg + lane]), s1, s2);
      if (vb + lane < end) sample<IDENT, 64, false>(L, __ldg(&a.dur[vb + lane]), s1, s2);
    }
    const uint32_t base = L.cnt_base;
    for (int64_t off = 0, nb = 4 * (vb - va); off < nb; off += TMA_STAGE) {
      const int n4 = (int)(min((int64_t)TMA_STAGE, nb - off) >> 4);
      mbar_wait(full0 + 8 * slot, ph);
      const uint32_t buf = ring_s + slot * TMA_STAGE;
      uint32_t s1w = 0;
      for (int i = tid; i < n4; i += TMA_CT) {
        int4 x;
        asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(x.x), "=r"(x.y), "=r"(x.z), "=r"(x.w)
                     : "r"(buf + 16 * i));
        if (FAST32) {
          sample_cta<IDENT>(L, base, x.x, s1w, s2);
          sample_cta<IDENT>(L, base, x.y, s1w, q1);
          sample_cta<IDENT>(L, base, x.z, s1w, q2);
          sample_cta<IDENT>(L, base, x.w, s1w, q3);
        } else {
          sample_cta<IDENT>(L, base, x.x, s1, s2);
          sample_cta<IDENT>(L, base, x.y, s1, q1);
          sample_cta<IDENT>(L, base, x.z, s1, q2);
          sample_cta<IDENT>(L, base, x.w, s1, q3);
        }
      }
      if (FAST32) s1 += s1w;  // <= 4 TMA_U samples per thread per stage: < 2^29 when b < 2^26
      __syncwarp();
      if (lane == 0) mbar_arrive(empty0 + 8 * slot);
      if (++slot == S) { slot = 0; ph ^= 1u; }
    }
    s2 += q1 + q2 + q3;
    const uint64_t w1 = warp_sum_u64(s1), w2 = warp_sum_u64(s2 & 0xffffffffull),
                   w3 = warp_sum_u64(s2 >> 32);
    if (lane == 0) { red[warp][0] = w1; red[warp][1] = w2; red[warp][2] = w3; }
    consumer_bar();
    if (tid < 6) {  // tid 0-2: the tool's row, 3-5: the pooled row F
      const int q = tid % 3;
      uint64_t sum = 0;
      for (int w = 0; w < TMA_CW; ++w) sum += red[w][q];
      unsigned long long* st = a.stat + (tid < 3 ? tool : a.F) * 6;
      if (q == 0) atomicAdd(st, (unsigned long long)(end - beg));
      if (sum) atomicAdd(st + 1 + q, (unsigned long long)sum);
    }
    for (int b = tid; b <= K; b += TMA_CT) {  // merge the 32 lane replicas of every bucket
      const uint4* pc = (const uint4*)(hsm + b * 64);
      uint64_t cn = 0, rr = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint4 x = pc[q], y = pc[8 + q];
        cn += (uint64_t)x.x + x.y + x.z + x.w;
        rr += (uint64_t)y.x + y.y + y.z + y.w;
      }
      if (cn) {
        const uint64_t sm = b < K ? (uint64_t)b * L.step * cn - rr : 0;
#pragma unroll
        for (int row2 = 0; row2 < 2; ++row2) {
          const int64_t o = (int64_t)(row2 ? a.F : tool) * (K + 1) + b;
          atomicAdd(&a.hcnt[o], (unsigned long long)cn);
          if (sm) atomicAdd(&a.hsum[o], (unsigned long long)sm);
        }
      }
    }
    consumer_bar();
  }
}

// Per-warp TMA variant: no producer warp and no cross-warp stage barrier.  The body of each
// piece is cut into WB-byte chunks dealt round-robin to the CTA's WW warps; every warp keeps
// WS of its own chunks in flight in a private ring (lane 0 issues the 1-D bulk copy, the warp
// waits on that slot's mbarrier), so a warp stalls only on its own data.  The histogram and the
// piece schedule are those of fit_hist_tma_kernel.

// WW warps per CTA, WB bytes per chunk, WS ring slots per warp
template <bool IDENT, bool FAST32, int WW, int WB, int WS>
__global__ void __launch_bounds__(32 * WW, 1) fit_hist_wtma_kernel(FitArgs a) {
  extern __shared__ __align__(128) uint32_t hsm[];
  __shared__ unsigned long long red[WW][3];
  const int K = a.K;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int words = (K + 1) * 64;
  const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(hsm + words) + warp * (WS * WB);
  const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(hsm + words) + WW * WS * WB + warp * (8 * WS);
  if (lane == 0) {
    for (int i = 0; i < WS; ++i) mbar_init(bar0 + 8 * i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const Lane L = cta_lane(a, hsm);
  const int64_t s0 = a.tool_off[0], s1e = a.tool_off[a.F];
  const int64_t per = (s1e - s0 + gridDim.x - 1) / gridDim.x;
  auto bnd = [&](int64_t b) -> int64_t {
    if (b == 0) return s0;
    if (b >= (int64_t)gridDim.x) return s1e;
    return min(s1e, max(s0, (s0 + b * per) & ~(int64_t)3));
  };
  int64_t lo = bnd(blockIdx.x);
  const int64_t hi = bnd((int64_t)blockIdx.x + 1);
  uint32_t phase = 0;  // bit i: parity of this warp's slot i
  int tool = 0;
  const uint32_t base = L.cnt_base;
  while (lo < hi) {
    while (a.tool_off[tool + 1] <= lo) ++tool;
    const int64_t beg = lo;
    const int64_t end = min(min(hi, a.tool_off[tool + 1]), lo + a.ch);
    lo = end;
    int64_t va = (beg + 3) & ~(int64_t)3;
    if (va > end) va = end;
    const int64_t vb = va + ((end - va) & ~(int64_t)3);
    const unsigned char* src = (const unsigned char*)(a.dur + va);
    const int64_t nb = 4 * (vb - va);
    const int64_t nch = (nb + WB - 1) / WB;  // chunks of this piece; warp w takes w, w + WW, ...
    auto issue = [&](int64_t c, int slot) {
      const uint32_t bytes = (uint32_t)min((int64_t)WB, nb - c * WB);
      mbar_expect_tx(bar0 + 8 * slot, bytes);
      bulk_g2s(ring_s + slot * WB, src + c * WB, bytes, bar0 + 8 * slot);
    };
    if (lane == 0)  // prefetch before the histogram is zeroed: the copies overlap the barrier
      for (int k = 0; k < WS; ++k)
        if (warp + (int64_t)k * WW < nch) issue(warp + (int64_t)k * WW, k);
    for (int i = tid; i < words; i += 32 * WW) hsm[i] = 0;
    __syncthreads();
    uint64_t s1 = 0, s2 = 0, q1 = 0, q2 = 0, q3 = 0;
    if (tid < 32) {  // scalar head and tail (< 4 samples each)
      if (beg + lane < va) sample<IDENT, 64, false>(L, __ldg(&a.dur[beg + lane]), s1, s2);
      if (vb + lane < end) sample<IDENT, 64, false>(L, __ldg(&a.dur[vb + lane]), s1, s2);
    }
    int slot = 0;
    for (int64_t c = warp; c < nch; c += WW) {
      mbar_wait(bar0 + 8 * slot, (phase >> slot) & 1u);
      phase ^= 1u << slot;
      const int n4 = (int)(min((int64_t)WB, nb - c * WB) >> 4);
      const uint32_t buf = ring_s + slot * WB;
      uint32_t s1w = 0;
#pragma unroll
      for (int u = 0; u < WB / 512; ++u) {
        const int i = lane + 32 * u;
        if (i < n4) {
          int4 x;
          asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(x.x), "=r"(x.y), "=r"(x.z), "=r"(x.w)
                       : "r"(buf + 16 * i));
          if (FAST32) {
            sample_cta<IDENT>(L, base, x.x, s1w, s2);
            sample_cta<IDENT>(L, base, x.y, s1w, q1);
            sample_cta<IDENT>(L, base, x.z, s1w, q2);
            sample_cta<IDENT>(L, base, x.w, s1w, q3);
          } else {
            sample_cta<IDENT>(L, base, x.x, s1, s2);
            sample_cta<IDENT>(L, base, x.y, s1, q1);
            sample_cta<IDENT>(L, base, x.z, s1, q2);
            sample_cta<IDENT>(L, base, x.w, s1, q3);
          }
        }
      }
      if (FAST32) s1 += s1w;  // 4 WB/512 = 16 samples per lane per chunk: < 2^30 when b < 2^26
      __syncwarp();
      const int64_t cn = c + (int64_t)WS * WW;
      if (lane == 0 && cn < nch) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // our reads before the refill
        issue(cn, slot);
      }
      if (++slot == WS) slot = 0;
    }
    // warps that received fewer chunks left some slots' phases unused: keep them consistent
    s2 += q1 + q2 + q3;
    const uint64_t w1 = warp_sum_u64(s1), w2 = warp_sum_u64(s2 & 0xffffffffull),
                   w3 = warp_sum_u64(s2 >> 32);
    if (lane == 0) { red[warp][0] = w1; red[warp][1] = w2; red[warp][2] = w3; }
    __syncthreads();
    if (tid < 6) {  // tid 0-2: the tool's row, 3-5: the pooled row F
      const int q = tid % 3;
      uint64_t sum = 0;
      for (int w = 0; w < WW; ++w) sum += red[w][q];
      unsigned long long* st = a.stat + (tid < 3 ? tool : a.F) * 6;
      if (q == 0) atomicAdd(st, (unsigned long long)(end - beg));
      if (sum) atomicAdd(st + 1 + q, (unsigned long long)sum);
    }
    for (int b = tid; b <= K; b += 32 * WW) {  // merge the 32 lane replicas of every bucket
      const uint4* pc = (const uint4*)(hsm + b * 64);
      uint64_t cn = 0, rr = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint4 x = pc[q], y = pc[8 + q];
        cn += (uint64_t)x.x + x.y + x.z + x.w;
        rr += (uint64_t)y.x + y.y + y.z + y.w;
      }
      if (cn) {
        const uint64_t sm = b < K ? (uint64_t)b * L.step * cn - rr : 0;
#pragma unroll
        for (int row2 = 0; row2 < 2; ++row2) {
          const int64_t o = (int64_t)(row2 ? a.F : tool) * (K + 1) + b;
          atomicAdd(&a.hcnt[o], (unsigned long long)cn);
          if (sm) atomicAdd(&a.hsum[o], (unsigned long long)sm);
        }
      }
    }
    __syncthreads();
  }
}

// cp.async variant: the Ampere-style multistage pipeline.  Each lane copies its own 16-B pieces
// of the warp's chunks global -> shared with cp.async.cg (no register staging, so 32 warps fit
// in 64 registers), AD stages deep, and later reads back only what it copied itself: no warp
// or CTA synchronisation in the stream, only per-thread cp.async.wait_group.  Chunks of
// 32 AU int4 are dealt round-robin to the AW warps; histogram and pieces as fit_hist_seg_kernel.
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <bool IDENT, bool FAST32, int AW, int AD, int AU>
__global__ void __launch_bounds__(32 * AW, 1) fit_hist_async_kernel(FitArgs a) {
  extern __shared__ __align__(128) uint32_t hsm[];
  __shared__ unsigned long long red[AW][3];
  const int K = a.K;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int words = (K + 1) * 64;
  const uint32_t ring = (uint32_t)__cvta_generic_to_shared(hsm + words) + warp * (AD * AU * 512) + 16 * lane;
  const Lane L = cta_lane(a, hsm);
  const int64_t s0 = a.tool_off[0], s1e = a.tool_off[a.F];
  const int64_t per = (s1e - s0 + gridDim.x - 1) / gridDim.x;
  auto bnd = [&](int64_t b) -> int64_t {
    if (b == 0) return s0;
    if (b >= (int64_t)gridDim.x) return s1e;
    return min(s1e, max(s0, (s0 + b * per) & ~(int64_t)3));
  };
  int64_t lo = bnd(blockIdx.x);
  const int64_t hi = bnd((int64_t)blockIdx.x + 1);
  int tool = 0;
  const uint32_t base = L.cnt_base;
  while (lo < hi) {
    while (a.tool_off[tool + 1] <= lo) ++tool;
    const int64_t beg = lo;
    const int64_t end = min(min(hi, a.tool_off[tool + 1]), lo + a.ch);
    lo = end;
    int64_t va = (beg + 3) & ~(int64_t)3;
    if (va > end) va = end;
    const int64_t vb = va + ((end - va) & ~(int64_t)3);
    const int4* v = (const int4*)(a.dur + va);
    const int64_t n4 = (vb - va) >> 2;
    const int64_t nch = (n4 + 32 * AU - 1) / (32 * AU);
    auto issue = [&](int64_t c, int slot) {
      if (c < nch) {
#pragma unroll
        for (int u = 0; u < AU; ++u) {
          const int64_t idx = c * (32 * AU) + 32 * u + lane;
          if (idx < n4) cp_async16(ring + slot * (AU * 512) + u * 512, v + idx);
        }
      }
      cp_commit();  // one group per stage, empty or not: the wait counts stay uniform
    };
#pragma unroll
    for (int st = 0; st < AD; ++st) issue(warp + (int64_t)AW * st, st);
    for (int i = tid; i < words; i += 32 * AW) hsm[i] = 0;
    __syncthreads();
    uint64_t s1 = 0, s2 = 0, q1 = 0, q2 = 0, q3 = 0;
    if (tid < 32) {  // scalar head and tail (< 4 samples each)
      if (beg + lane < va) sample<IDENT, 64, false>(L, __ldg(&a.dur[beg + lane]), s1, s2);
      if (vb + lane < end) sample<IDENT, 64, false>(L, __ldg(&a.dur[vb + lane]), s1, s2);
    }
    int slot = 0;
    for (int64_t c = warp; c < nch; c += AW) {
      cp_wait<AD - 1>();
      uint32_t s1w = 0;
#pragma unroll
      for (int u = 0; u < AU; ++u) {
        const int64_t idx = c * (32 * AU) + 32 * u + lane;
        if (idx < n4) {
          int4 x;
          asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(x.x), "=r"(x.y), "=r"(x.z), "=r"(x.w)
                       : "r"(ring + slot * (AU * 512) + u * 512));
          if (FAST32) {
            sample_cta<IDENT>(L, base, x.x, s1w, s2);
            sample_cta<IDENT>(L, base, x.y, s1w, q1);
            sample_cta<IDENT>(L, base, x.z, s1w, q2);
            sample_cta<IDENT>(L, base, x.w, s1w, q3);
          } else {
            sample_cta<IDENT>(L, base, x.x, s1, s2);
            sample_cta<IDENT>(L, base, x.y, s1, q1);
            sample_cta<IDENT>(L, base, x.z, s1, q2);
            sample_cta<IDENT>(L, base, x.w, s1, q3);
          }
        }
      }
      if (FAST32) s1 += s1w;  // 4 AU samples per lane per chunk: < 2^29 when b < 2^26
      issue(c + (int64_t)AW * AD, slot);  // this lane's slot is free again: it read it itself
      if (++slot == AD) slot = 0;
    }
    cp_wait<0>();
    s2 += q1 + q2 + q3;
    const uint64_t w1 = warp_sum_u64(s1), w2 = warp_sum_u64(s2 & 0xffffffffull),
                   w3 = warp_sum_u64(s2 >> 32);
    if (lane == 0) { red[warp][0] = w1; red[warp][1] = w2; red[warp][2] = w3; }
    __syncthreads();
    if (tid < 6) {  // tid 0-2: the tool's row, 3-5: the pooled row F
      const int q = tid % 3;
      uint64_t sum = 0;
      for (int w = 0; w < AW; ++w) sum += red[w][q];
      unsigned long long* st = a.stat + (tid < 3 ? tool : a.F) * 6;
      if (q == 0) atomicAdd(st, (unsigned long long)(end - beg));
      if (sum) atomicAdd(st + 1 + q, (unsigned long long)sum);
    }
    for (int b = tid; b <= K; b += 32 * AW) {  // merge the 32 lane replicas of every bucket
      const uint4* pc = (const uint4*)(hsm + b * 64);
      uint64_t cn = 0, rr = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint4 x = pc[q], y = pc[8 + q];
        cn += (uint64_t)x.x + x.y + x.z + x.w;
        rr += (uint64_t)y.x + y.y + y.z + y.w;
      }
      if (cn) {
        const uint64_t sm = b < K ? (uint64_t)b * L.step * cn - rr : 0;
#pragma unroll
        for (int row2 = 0; row2 < 2; ++row2) {
          const int64_t o = (int64_t)(row2 ? a.F : tool) * (K + 1) + b;
          atomicAdd(&a.hcnt[o], (unsigned long long)cn);
          if (sm) atomicAdd(&a.hsum[o], (unsigned long long)sm);
        }
      }
    }
    __syncthreads();
  }
}

template <bool IDENT>
static void* hist_fn(int v) {
  switch (v) {
    case 0: return (void*)fit_hist_kernel<IDENT, 16, false, 16>;
    case 1: return (void*)fit_hist_kernel<IDENT, 16, true, 16>;
    case 2: return (void*)fit_hist_kernel<IDENT, 8, false, 8>;
    case 3: return (void*)fit_hist_kernel<IDENT, 8, true, 8>;
    case 4: return (void*)fit_hist_kernel<IDENT, 32, false, 16>;
    case 5: return (void*)fit_hist_kernel<IDENT, 16, true, 8>;
    case 6: return (void*)fit_hist_kernel<IDENT, 8, true, 4>;
    case 7: return (void*)fit_hist_kernel<IDENT, 4, false, 8>;
    case 8: return (void*)fit_hist_kernel<IDENT, 4, false, 4>;
    case 9: return (void*)fit_hist_kernel<IDENT, 8, false, 4>;
    case 10: return (void*)fit_hist_cta_kernel<IDENT, 4, false>;
    case 11: return (void*)fit_hist_cta_kernel<IDENT, 8, false>;
    case 12: return (void*)fit_hist_cta_kernel<IDENT, 8, true>;  // b < 2^26 fast sums
    case 13: return (void*)fit_hist_cta_kernel<IDENT, 4, true>;
    case 14: return (void*)fit_hist_cta_kernel<IDENT, 6, true>;
    case 15: return (void*)fit_hist_seg_kernel<IDENT, 8, true>;   // contiguous CTA ranges
    case 16: return (void*)fit_hist_seg_kernel<IDENT, 8, false>;
    case 17: return (void*)fit_hist_tma_kernel<IDENT, true>;      // TMA-staged ranges
    case 18: return (void*)fit_hist_tma_kernel<IDENT, false>;
    case 19: return (void*)fit_hist_wtma_kernel<IDENT, true, WTMA_W, WTMA_B, WTMA_S>;  // per-warp TMA
    case 20: return (void*)fit_hist_wtma_kernel<IDENT, false, WTMA_W, WTMA_B, WTMA_S>;
    case 21: return (void*)fit_hist_async_kernel<IDENT, true, 16, 4, 2>;  // cp.async pipeline
    default: return (void*)fit_hist_async_kernel<IDENT, false, 16, 4, 2>;
  }
}

// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ Stat row_stat(const ScanArgs& a, int row) {  // row F = pooled
  uint64_t v[6];
#pragma unroll
  for (int q = 0; q < 6; ++q) v[q] = a.stat[row * 6 + q];
  // renormalise the limbs: s2 = l0 + l1 2^32 + l2 2^64 + l3 2^96
  u128_t s2 = (u128_t)v[2] + ((u128_t)v[3] << 32) + ((u128_t)v[4] << 64) + ((u128_t)v[5] << 96);
  Stat s;
  s.n = (int64_t)v[0];
  s.s1 = (int64_t)v[1];
  s.s2lo = (uint64_t)s2;
  s.s2hi = (uint64_t)(s2 >> 64);
  return s;
}

constexpr int SCAN_THREADS = 256;

// One CTA per (tool row, group of 8 turn buckets) (row F = all samples pooled).  The row's bucket counts / sums are loaded
// once into shared memory and prefix-scanned (cnt_le(k), sum_le(k)); then each warp evaluates
// n U(k) = V_j cnt_le(k) - C_j (sum_le(k) + tau_k (n - cnt_le(k))) for its turn buckets j in
// 128-bit integers and keeps the smallest maximiser (U(0) = 0: no pin).
__global__ void __launch_bounds__(SCAN_THREADS) fit_scan_kernel(ScanArgs a) {
  extern __shared__ __align__(16) unsigned long long sh[];
  const int K = a.K, F = a.F, J = a.J;
  unsigned long long* pc = sh;          // [K] inclusive prefix of counts
  unsigned long long* ps = sh + K;      // [K] inclusive prefix of sums
  __shared__ unsigned long long wtot[2][SCAN_THREADS / 32];
  __shared__ unsigned long long carry[2], ntot_sh;
  const int row = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const Stat f = row_stat(a, row);
  // tools with fewer than N samples take the pooled row's result (PAPER.md:492-494 ladder)
  const int src = (row == F || f.n < a.est.n_min) ? F : row;
  if (tid == 0) { carry[0] = carry[1] = 0; ntot_sh = 0; }
  __syncthreads();
  const int K1 = K + 1;
  for (int base = 0; base < K; base += SCAN_THREADS) {
    const int b = base + tid;
    unsigned long long c = 0, s = 0;
    if (b < K) {
      c = a.hcnt[(int64_t)src * K1 + b];
      s = a.hsum[(int64_t)src * K1 + b];
    }
    unsigned long long ic = c, is = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      unsigned long long tc = __shfl_up_sync(FULL_MASK, ic, o), ts = __shfl_up_sync(FULL_MASK, is, o);
      if (lane >= o) { ic += tc; is += ts; }
    }
    if (lane == 31) { wtot[0][warp] = ic; wtot[1][warp] = is; }
    __syncthreads();
    unsigned long long oc = carry[0], os = carry[1];
    for (int w = 0; w < warp; ++w) { oc += wtot[0][w]; os += wtot[1][w]; }
    if (b < K) { pc[b] = ic + oc; ps[b] = is + os; }
    __syncthreads();
    if (tid == SCAN_THREADS - 1) { carry[0] = ic + oc; carry[1] = is + os; }
    __syncthreads();
  }
  if (tid == 0) {
    ntot_sh = carry[0] + a.hcnt[(int64_t)src * K1 + K];  // + overflow bucket
  }
  __syncthreads();
  const uint64_t ntot = ntot_sh;
  const ct_cost_params& cp = a.cost;
  for (int j = blockIdx.y * (SCAN_THREADS / 32) + warp; j < min(J, (int)(blockIdx.y + 1) * (SCAN_THREADS / 32));
       ++j) {
    const i128_t V = ((i128_t)cp.c_pf_ps * cp.ctx_tokens[j] *
                      ((i128_t)cp.a_den + (i128_t)cp.a_num * cp.turn_weight[j])) / cp.a_den;
    const i128_t C = (i128_t)cp.c_pin_ps * ceil_div_i64(cp.ctx_tokens[j], cp.bs);
    i128_t best = 0;
    int bk = 0;
    for (int k = 1 + lane; k < K; k += 32) {
      const uint64_t cc = pc[k], cs = ps[k];
      const i128_t tau = (i128_t)k * cp.grid_step_us;
      const i128_t U = V * (i128_t)cc - C * ((i128_t)cs + tau * (i128_t)(ntot - cc));
      if (U > best) { best = U; bk = k; }  // k increases: strict > keeps the smallest
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const uint64_t lo = __shfl_xor_sync(FULL_MASK, (uint64_t)best, o);
      const uint64_t hi = __shfl_xor_sync(FULL_MASK, (uint64_t)((u128_t)best >> 64), o);
      const int ok = __shfl_xor_sync(FULL_MASK, bk, o);
      const i128_t ob = (i128_t)(((u128_t)hi << 64) | lo);
      if (ob > best || (ob == best && ok < bk)) { best = ob; bk = ok; }
    }
    if (lane == 0) a.ttl_argmax[(int64_t)row * J + j] = (int64_t)bk * cp.grid_step_us;
  }
  if (tid == 0 && blockIdx.y == 0) {
    const Stat g = row_stat(a, F);
    a.ttl_paper[row] = calc_ttl(g, f, a.est, a.cost.avg_turns_den, a.cost.avg_turns_num);
    if (a.stats_out) {
      a.stats_out[row * 4 + 0] = f.n;
      a.stats_out[row * 4 + 1] = f.s1;
      a.stats_out[row * 4 + 2] = (int64_t)f.s2lo;
      a.stats_out[row * 4 + 3] = (int64_t)f.s2hi;
    }
  }
}

cudaError_t launch_fit_hist(const FitArgs& a, const FitPlan& p, int grid, cudaStream_t s) {
  void* k = a.step == 1 ? hist_fn<true>(p.v) : hist_fn<false>(p.v);
  void* args[] = {(void*)&a};
  return cudaLaunchKernel(k, dim3(grid), dim3(p.threads), args, p.smem, s);
}

int fit_hist_occupancy(const FitPlan& p) {
  for (void* k : {hist_fn<true>(p.v), hist_fn<false>(p.v)})
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, p.smem) != cudaSuccess)
      return 0;
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, hist_fn<false>(p.v), p.threads, p.smem);
  return nb;
}

cudaError_t launch_fit_scan(const ScanArgs& a, cudaStream_t s) {
  const int smem = 16 * a.K;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(fit_scan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
  }
  const dim3 grid(a.F + 1, (a.J + SCAN_THREADS / 32 - 1) / (SCAN_THREADS / 32));
  fit_scan_kernel<<<grid, SCAN_THREADS, smem, s>>>(a);
  return cudaGetLastError();
}

}  // namespace ct
