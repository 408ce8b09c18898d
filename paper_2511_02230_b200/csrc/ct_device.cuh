// ct_device.cuh — device helpers shared by libcontinuum's kernels (sm_100a only).
#pragma once
#include <stdint.h>

#include "continuum.h"

#define CT_INF64 ((int64_t)0x7fffffffffffffffLL)
#define FULL_MASK 0xffffffffu

typedef unsigned __int128 u128_t;
typedef __int128 i128_t;

namespace ct {

__device__ __forceinline__ int64_t warp_min64(int64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    int64_t w = __shfl_xor_sync(FULL_MASK, v, o);
    v = w < v ? w : v;
  }
  return v;
}

__device__ __forceinline__ int64_t warp_max64(int64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    int64_t w = __shfl_xor_sync(FULL_MASK, v, o);
    v = w > v ? w : v;
  }
  return v;
}

__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL_MASK, v, o);
  return v;
}

__device__ __forceinline__ int64_t ceil_div_i64(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Warp minimum of non-negative 64-bit values with two REDUX.MIN (hi word, then lo word of the
// lanes holding the minimal hi word).
__device__ __forceinline__ int64_t warp_min64_redux(int64_t v) {
  const uint32_t hi = (uint32_t)((uint64_t)v >> 32), lo = (uint32_t)v;
  const uint32_t mh = __reduce_min_sync(FULL_MASK, hi);
  const uint32_t ml = __reduce_min_sync(FULL_MASK, hi == mh ? lo : 0xffffffffu);
  return (int64_t)(((uint64_t)mh << 32) | ml);
}

// ceil(x / 1e6) for picosecond sums below 2^63 (constant divisor: multiply-high sequence).
__device__ __forceinline__ int64_t ceil_ps_to_us(uint64_t ps) {
  return (int64_t)((ps + 999999ull) / 1000000ull);
}

// ceil(x / d) for x < 2^31 and a runtime divisor d < 2^20 given by its magic M = ceil(2^64 / d):
// floor(y / d), y = x + d - 1 < 2^32, is the high word of y * M (exact for 32-bit y); d = 1 uses
// ident = 1, M = 0.
struct DivMagic {
  uint32_t mhi, mlo, dm1, ident;
};
__device__ __forceinline__ uint32_t ceil_div_magic(uint32_t x, const DivMagic& m) {
  const uint32_t y = x + m.dm1;
  uint64_t p = __umulhi(y, m.mlo);
  asm("mad.wide.u32 %0, %1, %2, %0;" : "+l"(p) : "r"(y), "r"(m.mhi));
  return (uint32_t)(p >> 32) + y * m.ident;
}

// The generic quotients (a 128-bit quotient of 2^50 or more, a 64-bit one of 2^50 or more) are
// cold paths.  OL = true (the 32 < P <= 256 kernels, whose estimator sits in a large loop)
// calls one out-of-line copy of each, keeping the long division sequences out of the hot
// instruction footprint (measured: cfg2 +3 %); the P <= 32 kernels keep them inline (a call
// there measured 2-5 % slower: register pressure around the call).
static __host__ __device__ __noinline__ u128_t div_u128_slow(u128_t num, u128_t den) { return num / den; }
static __host__ __device__ __noinline__ uint64_t div_u64_slow(uint64_t num, uint64_t den) { return num / den; }

// floor(sqrt(x)) exactly: double estimate, then integer correction.
// floor(sqrt(x)) for x < 2^128 exactly (the argument of the Bernstein square root can exceed
// 2^64 for small n, wide samples and a small delta): double estimate, integer correction.
__host__ __device__ __forceinline__ uint64_t isqrt_u128(u128_t x) {
  if ((x >> 64) == 0) {
    const uint64_t y = (uint64_t)x;
    uint64_t r = (uint64_t)sqrt((double)y);
    if (r > 0xffffffffull) r = 0xffffffffull;
    while (r * r > y) --r;
    while (r < 0xffffffffull && (r + 1) * (r + 1) <= y) ++r;
    return r;
  }
  const double dx = (double)(uint64_t)(x >> 64) * 18446744073709551616.0 + (double)(uint64_t)x;
  const double sq = sqrt(dx);  // relative error ~2^-54: within ~2^10 of the root (>= 2^32)
  uint64_t r = sq >= 18446744073709551615.0 ? 0xffffffffffffffffull : (uint64_t)sq;
  // one Newton step on the exact residual (x - r^2) / (2 r), in double: error below a few
  // units, then exact integer correction (no 128-bit division)
  const u128_t r2 = (u128_t)r * r;
  const double res = r2 > x ? -(double)(r2 - x) : (double)(x - r2);
  const double step = res / (2.0 * (double)r);
  if (step >= 0.0) {
    const uint64_t up = (uint64_t)step;
    r = up > 0xffffffffffffffffull - r ? 0xffffffffffffffffull : r + up;
  } else {
    const uint64_t dn = (uint64_t)(-step);
    r = dn > r ? 0 : r - dn;
  }
  while ((u128_t)r * r > x) --r;
  while (r < 0xffffffffffffffffull && (u128_t)(r + 1) * (r + 1) <= x) ++r;
  return r;
}

__host__ __device__ __forceinline__ uint64_t isqrt_u64(uint64_t x) {
  uint64_t r = (uint64_t)sqrt((double)x);
  if (r > 0xffffffffull) r = 0xffffffffull;
  while (r * r > x) --r;
  while (r < 0xffffffffull && (r + 1) * (r + 1) <= x) ++r;
  return r;
}

// floor(num / den) for 0 < den < 2^64, exact.  Fast path when the quotient is below 2^50: the
// double estimate has relative error < 2^-50.5 (three roundings), so it is within one of the
// quotient and a single integer correction against num - q den makes it exact.  Larger
// quotients take the generic 128-bit division.
// div_u128_r takes a precomputed reciprocal rden = 1.0 / (double)den, or its exact power-of-two
// scaling, so several quotients by one divisor share one double division.  rden then adds at
// most two roundings and the product one, for six in all: the relative error stays below
// 2^-50.4, and the estimate is still within one of any quotient below 2^50.
template <bool OL = false>
__host__ __device__ __forceinline__ u128_t div_u128_r(u128_t num, uint64_t den, double rden) {
  const double dn = (double)(uint64_t)(num >> 64) * 18446744073709551616.0 + (double)(uint64_t)num;
  const double est = dn * rden;
  if (est < 1125899906842624.0) {  // 2^50
    uint64_t q = (uint64_t)est;
    const u128_t prod = (u128_t)q * den;
    if (prod > num) q -= 1;
    else if (num - prod >= den) q += 1;
    return q;
  }
  return OL ? div_u128_slow(num, den) : num / den;
}

template <bool OL = false>
__host__ __device__ __forceinline__ u128_t div_u128_u64(u128_t num, uint64_t den) {
  const double dn = (double)(uint64_t)(num >> 64) * 18446744073709551616.0 + (double)(uint64_t)num;
  const double est = dn / (double)den;
  if (est < 1125899906842624.0) {  // 2^50
    uint64_t q = (uint64_t)est;
    const u128_t prod = (u128_t)q * den;
    if (prod > num) q -= 1;
    else if (num - prod >= den) q += 1;
    return q;
  }
  return OL ? div_u128_slow(num, den) : num / den;
}

struct Stat {  // one estimator row: n, sum t~, sum t~^2 (128-bit as lo/hi)
  int64_t n, s1;
  uint64_t s2lo, s2hi;
};

// Empirical Bernstein bound B(delta), fixed point (C-1):
// floor(s1/n) + isqrt(floor(2 v L_q / (n 2^32))) + floor(3 b L_q / (n 2^32)),
// v = floor((n s2 - s1^2) / (n (n-1))) for n >= 2, else 0.
// The three quotients by n and by n 2^32 share one reciprocal of n.
template <bool OL = false>
__host__ __device__ __forceinline__ int64_t bernstein(const Stat& s, uint64_t lq, int64_t b_us) {
  const int64_t n = s.n;
  const double rn = 1.0 / (double)n;           // n < 2^31 (validated): exact conversion
  const double rnsh = rn * 2.3283064365386963e-10;  // 2^-32: exact scaling
  // floor(s1 / n) with 64-bit operands (s1 < 2^63): double estimate, one 64-bit correction
  int64_t mu;
  {
    const uint64_t num = (uint64_t)s.s1, den = (uint64_t)n;
    const double est = (double)num * rn;
    if (est < 1125899906842624.0) {  // 2^50: the estimate is within one of the quotient
      uint64_t q = (uint64_t)est;
      const uint64_t prod = q * den;   // <= num + den < 2^64
      if (prod > num) q -= 1;
      else if (num - prod >= den) q += 1;
      mu = (int64_t)q;
    } else {
      mu = OL ? (int64_t)div_u64_slow(num, den) : (int64_t)(num / den);
    }
  }
  u128_t v = 0;
  if (n >= 2) {
    u128_t s2 = ((u128_t)s.s2hi << 64) | s.s2lo;
    u128_t num = (u128_t)(uint64_t)n * s2 - (u128_t)(uint64_t)s.s1 * (uint64_t)s.s1;
    uint64_t den = (uint64_t)n * (uint64_t)(n - 1);  // n < 2^31 (validated)
    v = div_u128_u64<OL>(num, den);
  }
  uint64_t nsh = (uint64_t)n << 32;
  u128_t a2 = div_u128_r<OL>((u128_t)2 * v * lq, nsh, rnsh);
  uint64_t t2 = isqrt_u128(a2);
  // floor(3 b L_q / (n 2^32)) = floor(floor(3 b L_q / 2^32) / n): a 64-bit numerator below
  // 3 2^48 (b, L_q < 2^40, host-checked), loop-invariant in the replay; its quotient by n as mu
  uint64_t t3;
  {
    const uint64_t num = (uint64_t)(((u128_t)3 * (uint64_t)b_us * lq) >> 32);
    const uint64_t den = (uint64_t)n;
    const double est = (double)num * rn;
    if (est < 1125899906842624.0) {  // 2^50
      uint64_t q = (uint64_t)est;
      const uint64_t prod = q * den;
      if (prod > num) q -= 1;
      else if (num - prod >= den) q += 1;
      t3 = q;
    } else {
      t3 = OL ? div_u64_slow(num, den) : num / den;
    }
  }
  return mu + (int64_t)t2 + (int64_t)t3;
}

#ifdef __CUDA_ARCH__
// A real upper bound of the fixed-point Bernstein bound B (C-1) of
// row s (n >= 1), in single precision with approximate reciprocal / square root: every rounding
// (at most ~2^-22 relative each) is covered by the margin M = 1 + 2^-12 applied after each
// step, and floor() only lowers the exact terms.  Uses the identities
// floor(s1/n) <= s1/n, v <= (s2/n - (s1/n)^2) n/(n-1), isqrt(floor(a)) <= sqrt(a).
__device__ __forceinline__ float bernstein_upper(const Stat& s, uint64_t lq, int64_t b_us) {
  constexpr float M = 1.000244140625f, Mi = 0.999755859375f;  // 1 +- 2^-12
  float rn, r;
  const float nf = (float)s.n;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rn) : "f"(nf));
  const float rn_up = rn * M, rn_lo = rn * Mi;
  const float s1 = (float)s.s1;
  const float mean_up = s1 * rn_up * M, mean_lo = s1 * rn_lo * Mi;
  float var_up = 0.0f;
  if (s.n >= 2) {
    const float s2 = (float)s.s2hi * 18446744073709551616.0f + (float)s.s2lo;
    float n1;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(n1) : "f"(nf - 1.0f));  // n - 1 >= 1 exact below 2^24
    var_up = fmaxf(s2 * M * rn_up * M - mean_lo * mean_lo * Mi, 0.0f) * (nf * n1 * M * M);
  }
  const float lqf = (float)lq * M;
  const float a_up = 2.0f * var_up * lqf * rn_up * 2.3283064365386963e-10f * M;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a_up));
  const float t3_up = 3.0f * (float)b_us * lqf * rn_up * 2.3283064365386963e-10f * M;
  return (mean_up + r * M + t3_up) * M + 2.0f;
}
#endif

// 𝓑(r,f) then CalcTTL offset, readings R7/R8/R36.
// QUICK (device): when an upper bound of 𝓑 already proves the offset at or above the clamp
// ttl_max (the common case once a tool row holds many samples), return the clamp without the
// exact 128-bit evaluation; the result is identical (the test is one-sided and rigorous).
template <bool OL = false, bool QUICK = false>
__host__ __device__ __forceinline__ int64_t calc_ttl(const Stat& g, const Stat& f,
                                            const ct_estimator_params& e, int64_t n_done,
                                            int64_t turns_done) {
#ifdef __CUDA_ARCH__
  if (QUICK && e.ttl_max_us > 0 && g.n >= e.n_min) {
    const Stat& q = f.n >= e.n_min ? f : g;
    const double bu = fmax((double)bernstein_upper(q, e.lq, e.b_us), 1.0);
    // floor(T^2 (D a_den + a_num turns) / (B D a_den)) >= ttl_max  <=  T^2 (D a_den + a_num
    // turns) >= ttl_max B_up D a_den; both sides in double with a 2^-40 relative margin
    const double t = (double)e.t_default_us;
    const double lhs = n_done > 0 ? t * t * ((double)n_done * (double)e.a_den +
                                             (double)e.a_num * (double)turns_done)
                                   : t * t;
    const double rhs = n_done > 0 ? (double)e.ttl_max_us * bu * (double)n_done * (double)e.a_den
                                  : (double)e.ttl_max_us * bu;
    if (lhs >= rhs * 1.0000000000009095) return e.ttl_max_us;  // ttl_max < CT_TTL_SAT
  }
#endif
  int64_t B;
  if (g.n < e.n_min) {
    B = e.t_default_us;
  } else {  // one inlined bound on the selected row (tool if |S_f| >= N, else global)
    const bool tool = f.n >= e.n_min;
    Stat s;
    s.n = tool ? f.n : g.n;
    s.s1 = tool ? f.s1 : g.s1;
    s.s2lo = tool ? f.s2lo : g.s2lo;
    s.s2hi = tool ? f.s2hi : g.s2hi;
    B = bernstein<OL>(s, e.lq, e.b_us);
  }
  if (B < 1) B = 1;
  const u128_t T2 = (u128_t)(uint64_t)e.t_default_us * (uint64_t)e.t_default_us;  // < 2^80
  u128_t ttl;
  if (n_done > 0) {
    u128_t num = T2 * ((u128_t)(uint64_t)n_done * (uint64_t)e.a_den +
                       (u128_t)(uint64_t)e.a_num * (uint64_t)turns_done);
    u128_t den = (u128_t)(uint64_t)B * (uint64_t)n_done * (uint64_t)e.a_den;
    ttl = (den >> 64) == 0 ? div_u128_u64<OL>(num, (uint64_t)den)
                           : OL ? div_u128_slow(num, den) : num / den;
  } else {
    ttl = div_u128_u64<OL>(T2, (uint64_t)B);
  }
  if (e.ttl_max_us > 0 && ttl > (u128_t)(uint64_t)e.ttl_max_us) ttl = (uint64_t)e.ttl_max_us;
  if (ttl >= (u128_t)CT_TTL_SAT) ttl = CT_TTL_SAT - 1;  // reading R36
  return (int64_t)(uint64_t)ttl;
}

// §4.5 simplified decision, reading R9.
__host__ __device__ __forceinline__ int64_t simplified_ttl(const Stat& g, const Stat& f,
                                                  const ct_estimator_params& e, int64_t t_pin,
                                                  int64_t t_thresh) {
  if (t_thresh == CT_ALWAYS) return t_pin;
  int64_t mu;
  if (f.n >= e.n_min) mu = f.s1 / f.n;
  else if (g.n >= 1) mu = g.s1 / g.n;
  else return 0;
  return mu < t_thresh ? t_pin : 0;
}

// InferCept: predicted tool time = mean of the tool when |S_f| >= N,
// else the global mean when |S| >= 1, else T_default.
__host__ __device__ __forceinline__ int64_t infercept_predict(const Stat& g, const Stat& f,
                                                     const ct_estimator_params& e) {
  if (f.n >= e.n_min) return f.s1 / f.n;
  if (g.n >= 1) return g.s1 / g.n;
  return e.t_default_us;
}

}  // namespace ct
