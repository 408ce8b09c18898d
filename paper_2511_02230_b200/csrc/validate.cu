// validate.cu — on-device check of a trace set before a replay (include/continuum.h,
// ct_simulate_batch preconditions).  Trace buffers live in HBM, so their records are checked
// where they are: one thread per program over the seeds the replica range touches, plus the
// FITTED table.  Violations set bits of err[0] and keep the first bad program in err[1] (as
// ~index, so a max works on a zeroed word); the replay kernel reads err[0] once per warp and
// reports every replica as CT_R_INVALID_INPUT instead of reading out of bounds.
#include <algorithm>

#include "ct_device.cuh"
#include "ct_internal.h"

namespace ct {

__global__ void __launch_bounds__(256) check_traces_kernel(CheckArgs a) {
  const int64_t nt = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t i = a.p_begin + t0; i < a.p_end; i += nt) {
    const ct_program p = a.progs[i];
    uint32_t bits = 0;
    if (p.nturns < 1 || p.nturns > CT_MAX_TURNS) bits |= CT_CHECK_NTURNS;
    if (p.turn0 < 0 || (int64_t)p.turn0 + p.nturns > a.n_turns) bits |= CT_CHECK_TURN_RANGE;
    if (p.arr_q < 0 || p.arr_q > a.arr_max) bits |= CT_CHECK_ARRIVAL;
    if (i % a.P && p.arr_q < a.progs[i - 1].arr_q) bits |= CT_CHECK_ARRIVAL;
    if (!(bits & (CT_CHECK_NTURNS | CT_CHECK_TURN_RANGE))) {
      int64_t ctx = 0;
      for (int t = 0; t < p.nturns; ++t) {
        const int4 u = __ldg(a.turns + p.turn0 + t);  // {new, decode, tool, dur}
        if (u.y < 1 || u.x < 0) bits |= CT_CHECK_TOKENS;
        if (t < p.nturns - 1 && (u.z < 0 || u.z >= a.F || u.w < 1)) bits |= CT_CHECK_TOOL;
        ctx += (int64_t)max(u.x, 0) + max(u.y, 0);
      }
      if (ctx > CT_MAX_CONTEXT) bits |= CT_CHECK_CONTEXT;
    }
    if (bits) {
      atomicOr((unsigned int*)a.err, bits);
      atomicMax(a.err + 1, ~(unsigned long long)i);
    }
  }
  for (int64_t i = t0; i < a.n_fitted; i += nt)
    if (a.fitted[i] < 0 || a.fitted[i] >= CT_TTL_SAT) atomicOr((unsigned int*)a.err, CT_CHECK_FITTED);
}

cudaError_t launch_check_traces(const CheckArgs& a, int sm_count, cudaStream_t s) {
  const int64_t work = std::max<int64_t>(a.p_end - a.p_begin, a.n_fitted);
  if (work <= 0) return cudaSuccess;
  const int grid = (int)std::min<int64_t>((work + 255) / 256, 4 * (int64_t)sm_count);
  check_traces_kernel<<<grid, 256, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace ct
