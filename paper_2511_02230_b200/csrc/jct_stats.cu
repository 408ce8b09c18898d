// jct_stats.cu — per sweep cell reduction of replica summaries.
// One warp per cell (rate, kv, policy); lanes stride over the cell's seeds.  Integer sums,
// so the result does not depend on the reduction order.
#include "ct_device.cuh"
#include "ct_internal.h"

namespace ct {

__global__ void __launch_bounds__(256) jct_stats_kernel(const ct_replica_summary* __restrict__ s,
                                                        int64_t n, int32_t n_cells,
                                                        ct_cell_stats* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t cell = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (cell >= n_cells) return;
  const int64_t seeds = n / n_cells;
  uint64_t ok = 0, bad = 0, done = 0, turns = 0, jsum = 0, bub = 0, mk = 0;
  int64_t jmax = 0;
  for (int64_t k = lane; k < seeds; k += 32) {
    const ct_replica_summary& r = s[k * n_cells + cell];
    if (r.status != CT_R_OK) { ++bad; continue; }
    ++ok;
    done += (uint64_t)r.n_done;
    turns += (uint64_t)r.turns_done;
    jsum += (uint64_t)r.sum_jct_us;
    jmax = max(jmax, r.max_jct_us);
    bub += (uint64_t)r.sum_bubble_us;
    mk += (uint64_t)r.makespan_us;
  }
  ok = warp_sum_u64(ok);
  bad = warp_sum_u64(bad);
  done = warp_sum_u64(done);
  turns = warp_sum_u64(turns);
  jsum = warp_sum_u64(jsum);
  bub = warp_sum_u64(bub);
  mk = warp_sum_u64(mk);
  jmax = warp_max64(jmax);
  if (lane == 0) {
    ct_cell_stats o;
    o.n_ok = (int64_t)ok;
    o.n_bad = (int64_t)bad;
    o.sum_done = (int64_t)done;
    o.sum_turns = (int64_t)turns;
    o.sum_jct_us = (int64_t)jsum;
    o.max_jct_us = jmax;
    o.sum_bubble_us = (int64_t)bub;
    o.sum_makespan_us = (int64_t)mk;
    out[cell] = o;
  }
}

cudaError_t launch_jct_stats(const ct_replica_summary* s, int64_t n, int32_t n_cells,
                             ct_cell_stats* out, cudaStream_t st) {
  const int wpb = 8;
  int grid = (int)((n_cells + wpb - 1) / wpb);
  jct_stats_kernel<<<grid, 32 * wpb, 0, st>>>(s, n, n_cells, out);
  return cudaGetLastError();
}

}  // namespace ct
