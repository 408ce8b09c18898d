// ct_internal.h — launch interfaces between libcontinuum's host runtime and its kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "continuum.h"

namespace ct {

struct ReplayArgs {
  const ct_program* progs;
  const int4* turns;
  int P, F;
  const int64_t* gap;
  const int64_t* kv;
  const ct_policy* pols;
  int n_rate, n_kv, n_pol;
  ct_estimator_params est;
  const int64_t* fitted;
  int J;
  ct_engine_params eng;
  int64_t r_begin, r_end;
  ct_replica_summary* out;
  int64_t* jct;
  int64_t* bubble;  // per-program waiting time [R * P] or NULL (NEXT-3)
  unsigned long long* counter;
  int smem_per_warp;
  uint64_t bs_magic;  // ceil(2^64 / bs) (0 when bs == 1)
  int d32;            // every no-prefill iteration is below 2^31 µs (32-bit macro-step division)
  int from_list;      // replay the replicas fb_list[0 .. *fb_count) instead of [r_begin, r_end)
  int64_t* fb_list;   // MODE 4: replicas handed to the 64-bit kernel (horizon, bubble output)
  unsigned long long* fb_count;
};

// The TTL-grid policy class, for which the P <= 32 replay has a specialised path: program
// FCFS; EVICT, or FIXED with T_thresh = CT_ALWAYS (pin for t_pin); no DRAM tier; eager expiry
// and the paper's victim rule (flags 0).
inline __host__ __device__ bool fast_policy(const ct_policy& p, const ct_engine_params& E) {
  return p.priority == CT_PRIO_PROG_FCFS && p.flags == 0 && (p.dram == 0 || E.dram_blocks <= 0) &&
         (p.pause == CT_PAUSE_EVICT || (p.pause == CT_PAUSE_FIXED && p.t_thresh_us == CT_ALWAYS));
}

// The program-FCFS class, for which the P > 32 replay has a specialised path: program FCFS; any
// pause action but InferCept; no DRAM tier; eager expiry and the paper's victim rule.
inline __host__ __device__ bool prog_policy(const ct_policy& p, const ct_engine_params& E) {
  return p.priority == CT_PRIO_PROG_FCFS && p.flags == 0 && (p.dram == 0 || E.dram_blocks <= 0) &&
         p.pause != CT_PAUSE_INFERCEPT;
}

// The simple class, for which the P <= 32 replay has a 32-bit-time path with the estimator:
// program or request FCFS; EVICT, FIXED, PAPER or FITTED; no DRAM tier; flags 0.
inline __host__ __device__ bool simple_policy(const ct_policy& p, const ct_engine_params& E) {
  return (p.priority == CT_PRIO_PROG_FCFS || p.priority == CT_PRIO_REQ_FCFS) && p.flags == 0 &&
         (p.dram == 0 || E.dram_blocks <= 0) && p.pause != CT_PAUSE_INFERCEPT;
}

// Bytes of shared memory one replica (one warp) needs for `ns` slots per lane and F tools.
// KV growth (NEXT-2) always runs the shared-memory path, also for P <= 32.
int replay_smem_per_warp(int ns, int F, bool growth, int mode);
// Same for the 32-bit program-FCFS kernel (MODE 4, ns >= 2).
int replay_ns32_smem_per_warp(int ns, int F);
// Launch the persistent replay kernel; returns the cudaError of the launch.
// mode (ns == 1, default engine): 0 generic, 1 all policies fast_policy(), 2 mixed.
cudaError_t launch_replay(const ReplayArgs& a, int ns, bool growth, int mode, int warps_per_block,
                          int grid, cudaStream_t s);
// Max resident blocks per SM for the given configuration.
int replay_occupancy(int ns, bool growth, int mode, int warps_per_block, int smem_per_block);

struct FitArgs {
  const int32_t* dur;
  int64_t n_chunks;              // work items: chunks of <= ch samples inside one tool segment
  int64_t ch;
  int64_t tool_off[CT_MAX_TOOLS + 1];
  int64_t chunk_off[CT_MAX_TOOLS + 1];  // first chunk index of each tool
  int F, K;
  int64_t step;          // grid step (µs)
  uint64_t step_magic;   // ceil(2^64 / step) for the bucket quotient (per-warp kernels)
  uint32_t div_m, div_sh, div_add;  // floor(x / step) for 32-bit x (CTA kernels, step >= 2)
  int64_t b_us;
  int stages;  // TMA ring depth (TMA-staged variant)
  unsigned long long* hcnt;  // [(F+1) * (K+1)] bucket counts, row F pooled over tools
  unsigned long long* hsum;  // [(F+1) * (K+1)] bucket sums (buckets < K)
  unsigned long long* stat;  // [(F+1) * 6]: n, s1, s2 limbs (32-bit limb sums in u64 slots)
};

struct ScanArgs {
  const unsigned long long* hcnt;
  const unsigned long long* hsum;
  const unsigned long long* stat;
  int F, K, J;
  ct_cost_params cost;
  ct_estimator_params est;
  int64_t* ttl_argmax;
  int64_t* ttl_paper;
  int64_t* stats_out;
};

// Kernel variant, launch shape and shared memory of the histogram pass for grid size K and
// clamp b (ttl_fit.cu: CT_FIT_VARIANT overrides the default for experiments).
struct FitPlan {
  int v, threads, smem, repl, stages;
  bool cta;     // CTA-shared lane-indexed histogram (work items are CTA-level)
  bool ranges;  // one contiguous sample range per CTA, pieces of <= ch samples
};
FitPlan fit_plan(int K, int64_t b_us);
int fit_hist_occupancy(const FitPlan& p);  // resident CTAs per SM
cudaError_t launch_fit_hist(const FitArgs& a, const FitPlan& p, int grid, cudaStream_t s);
cudaError_t launch_fit_scan(const ScanArgs& a, cudaStream_t s);

// On-device trace synthesis (synth.cu).  Device scratch is owned by the context.
struct SynthLaunch {
  const ct_synth_params* sp;
  int64_t seed0;
  int64_t n_seeds;
  int P;
  const int64_t* tab;   // [dev] (6 + F) x 1025 quantile tables
  const uint32_t* cdf;  // [dev] F
  const int32_t* cls;   // [dev] F
  ct_program* progs;
  ct_turn* turns;
  int64_t turns_cap;
  uint8_t* pcls;        // [dev] S * P
  int64_t* seed_tot;    // [dev] S
  int64_t* blk;         // [dev] ceil(S / 1024) + 1
};
// Runs the three passes; synchronises `st` after the count pass and skips the write pass when
// the total (returned in *total_host) exceeds turns_cap.
cudaError_t launch_synth(const SynthLaunch& L, int sm_count, cudaStream_t st, int64_t* total_host);

// Sets the thread-local message ct_last_error() returns (api.cu); host code in other files.
void set_last_error(const char* msg);

cudaError_t launch_jct_stats(const ct_replica_summary* s, int64_t n, int32_t n_cells,
                             ct_cell_stats* out, cudaStream_t st);

}  // namespace ct
