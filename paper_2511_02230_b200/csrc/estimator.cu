// estimator.cu — the estimator of PAPER.md §4.2-4.3 as batched device calls (include/continuum.h
// ct_bernstein, ct_calc_ttl_batch): one thread per row / query over the same fixed-point helpers
// (ct_device.cuh bernstein, calc_ttl) that the replay and the fit run, so the C ABI exposes the
// exact arithmetic of the hot path for checks against the paper's worked examples.
#include <algorithm>

#include "ct_device.cuh"
#include "ct_internal.h"

namespace ct {

__host__ __device__ __forceinline__ Stat to_stat(const ct_stat_row& r) {
  Stat s;
  s.n = r.n;
  s.s1 = r.s1;
  s.s2lo = r.s2_lo;
  s.s2hi = r.s2_hi;
  return s;
}

// the statistics of n < 2^31 samples in [0, b] (n = 0: all zero)
__host__ __device__ __forceinline__ bool row_ok(const ct_stat_row& r, int64_t b_us) {
  if (r.n < 0 || r.n >= (1ll << 31) || r.s1 < 0) return false;
  const u128_t s2 = ((u128_t)r.s2_hi << 64) | r.s2_lo;
  // s1 <= n b, s2 <= n b^2 and n s2 >= s1^2 (Cauchy-Schwarz: a non-negative variance)
  return (u128_t)(uint64_t)r.s1 <= (u128_t)(uint64_t)r.n * (uint64_t)b_us &&
         s2 <= (u128_t)(uint64_t)r.n * (uint64_t)b_us * (uint64_t)b_us &&
         (u128_t)(uint64_t)r.n * s2 >= (u128_t)(uint64_t)r.s1 * (uint64_t)r.s1;
}

int64_t bernstein_row(const ct_stat_row& r, const ct_estimator_params& e) {
  if (r.n < 1 || !row_ok(r, e.b_us)) return CT_TTL_INVALID;
  return bernstein(to_stat(r), e.lq, e.b_us);
}

int64_t calc_ttl_row(const ct_stat_row& g, const ct_stat_row& f, const ct_estimator_params& e,
                     int64_t n_done, int64_t turns_done) {
  if (!row_ok(g, e.b_us) || !row_ok(f, e.b_us) || n_done < 0 || n_done > CT_MAX_PROGRAMS ||
      turns_done < 0 || turns_done > (int64_t)CT_MAX_PROGRAMS * CT_MAX_TURNS)
    return CT_TTL_INVALID;
  return calc_ttl(to_stat(g), to_stat(f), e, n_done, turns_done);
}

__global__ void __launch_bounds__(256) bernstein_kernel(const ct_stat_row* rows, int64_t n,
                                                        ct_estimator_params e, int64_t* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const ct_stat_row r = rows[i];
    out[i] = (r.n < 1 || !row_ok(r, e.b_us)) ? CT_TTL_INVALID : bernstein(to_stat(r), e.lq, e.b_us);
  }
}

__global__ void __launch_bounds__(256) calc_ttl_kernel(const ct_stat_row* g, const ct_stat_row* f,
                                                       const int64_t* n_done,
                                                       const int64_t* turns_done, int64_t n,
                                                       ct_estimator_params e, int64_t* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const ct_stat_row gr = g[i], fr = f[i];
    const int64_t d = n_done[i], td = turns_done[i];
    const bool ok = row_ok(gr, e.b_us) && row_ok(fr, e.b_us) && d >= 0 && d <= CT_MAX_PROGRAMS &&
                    td >= 0 && td <= (int64_t)CT_MAX_PROGRAMS * CT_MAX_TURNS;
    // the replay's CalcTTL, including its clamp shortcut (identical results to the exact path)
    out[i] = ok ? calc_ttl<false, true>(to_stat(gr), to_stat(fr), e, d, td) : CT_TTL_INVALID;
  }
}

cudaError_t launch_bernstein(const ct_stat_row* rows, int64_t n, const ct_estimator_params& e,
                             int64_t* out, int sm_count, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const int grid = (int)std::min<int64_t>((n + 255) / 256, 8 * (int64_t)sm_count);
  bernstein_kernel<<<grid, 256, 0, s>>>(rows, n, e, out);
  return cudaGetLastError();
}

cudaError_t launch_calc_ttl(const ct_stat_row* g, const ct_stat_row* f, const int64_t* n_done,
                            const int64_t* turns_done, int64_t n, const ct_estimator_params& e,
                            int64_t* out, int sm_count, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const int grid = (int)std::min<int64_t>((n + 255) / 256, 8 * (int64_t)sm_count);
  calc_ttl_kernel<<<grid, 256, 0, s>>>(g, f, n_done, turns_done, n, e, out);
  return cudaGetLastError();
}

}  // namespace ct
