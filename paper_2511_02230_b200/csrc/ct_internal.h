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
  const unsigned long long* err;  // trace check result (validate.cu): err[0] != 0 = invalid input
  int kv32;            // c_kv bs max(kv) + 1e6 < 2^32: 32-bit iteration duration (iter_us_kv32)
  uint32_t kv_unit;    // c_kv bs (ps per resident block)
  uint32_t c0q, c0r;   // c0 = c0q 1e6 - c0r, 0 <= c0r < 1e6
  uint32_t pf_q, pf_r; // c_pf = pf_q 1e6 + pf_r, 0 <= pf_r < 1e6
  uint32_t pf32;       // prefills below pf32 tokens take the 32-bit path (pf_r pf + 1e6 < 2^32)
  const int* sel;      // policy subset of this launch (ascending indices) or NULL: every policy
  int n_sel;
  int64_t blk0;        // first block of n_pol replicas touched by [r_begin, r_end)
  int64_t sel_total;   // blocks x n_sel (< 2^31)
};

// Trace-set check (validate.cu).  Bits of err[0]:
#define CT_CHECK_NTURNS 1u      /* nturns outside [1, CT_MAX_TURNS] */
#define CT_CHECK_TURN_RANGE 2u  /* turn0 / turn0 + nturns outside the turn array */
#define CT_CHECK_ARRIVAL 4u     /* arr_q < 0, arr_q gap_max >= 2^62, or arrivals not sorted */
#define CT_CHECK_TOKENS 8u      /* decode < 1 or new < 0 */
#define CT_CHECK_TOOL 16u       /* a non-final turn's tool outside [0, F) or dur < 1 */
#define CT_CHECK_CONTEXT 32u    /* a program's total new + decode tokens > CT_MAX_CONTEXT */
#define CT_CHECK_FITTED 64u     /* a FITTED table entry outside [0, CT_TTL_SAT) */
struct CheckArgs {
  const ct_program* progs;
  const int4* turns;
  int64_t n_turns;
  int64_t p_begin, p_end;  // programs of the seeds the replica range touches
  int P, F;
  int64_t arr_max;         // largest arr_q with arr_q * max(gap) < 2^62
  const int64_t* fitted;
  int64_t n_fitted;
  unsigned long long* err;  // [2], zeroed by the caller
};
cudaError_t launch_check_traces(const CheckArgs& a, int sm_count, cudaStream_t s);

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

// The extended class, for which the P <= 32 replay has a 32-bit-time path with the DRAM tier,
// Autellix PLAS and InferCept (replay_one_t32<true, true>, MODE 6): any priority, any pause
// action, DRAM on or off; only the alternative readings (flags) are left to the generic path.
inline __host__ __device__ bool ext_policy(const ct_policy& p, const ct_engine_params& E) {
  (void)E;
  return p.flags == 0;
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
  const uint8_t* tool_u8;          // unsorted pairs layout: tool id per sample (else NULL)
  int64_t n;                       // pairs layout: sample count
  int64_t seg_lo[CT_MAX_TOOLS];    // CSR: physical sample range [seg_lo, seg_hi) of tool f
  int64_t seg_hi[CT_MAX_TOOLS];
  int64_t voff[CT_MAX_TOOLS + 1];  // CSR: prefix of the segment lengths (virtual order)
  int64_t ch;                      // max samples per histogram piece (32-bit bin bound)
  int F, K;
  int64_t step;                    // grid step (µs)
  uint32_t div_m, div_sh, div_add; // floor(x / step) for 32-bit x (step >= 2)
  int64_t b_us;
  unsigned long long* acc;         // accumulator, fit_acc_words(F, K) words
  unsigned long long* zero;        // zero this buffer first (the next call's accumulator) or NULL
  int64_t zero_words;
};

struct ScanArgs {
  const unsigned long long* acc;
  int F, K, J;
  ct_cost_params cost;
  ct_estimator_params est;
  int64_t* ttl_argmax;
  int64_t* ttl_paper;
  int64_t* stats_out;
  int64_t* n_invalid;
};

// Accumulator words: (F+1)(K+1) bucket counts | (F+1)(K+1) bucket sums | (F+1) x 6 statistic
// limbs {n, sum t~, l0..l3 of sum t~^2} | 1 count of samples outside [0, 2^31).
int64_t fit_acc_words(int F, int K);

// Shape of the histogram pass: lane replicas of the CTA histogram (32, or 16 when (K+1) x 256 B
// exceeds shared memory), dynamic shared memory; pairs = unsorted (dur, u8 tool) layout.
struct FitPlan {
  bool pairs, ok;
  int lr, smem;
};
FitPlan fit_plan(int K, int F, bool pairs);
int fit_hist_occupancy(const FitArgs& a, const FitPlan& p);  // CTAs per SM
cudaError_t launch_fit_hist(const FitArgs& a, const FitPlan& p, int grid, cudaStream_t st);
// programmatic dependent launch after the histogram pass on the same stream
cudaError_t launch_fit_finish(const ScanArgs& s, cudaStream_t st);

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

// Estimator calls (estimator.cu): device batches and the host references (same helpers).
cudaError_t launch_bernstein(const ct_stat_row* rows, int64_t n, const ct_estimator_params& e,
                             int64_t* out, int sm_count, cudaStream_t s);
cudaError_t launch_calc_ttl(const ct_stat_row* g, const ct_stat_row* f, const int64_t* n_done,
                            const int64_t* turns_done, int64_t n, const ct_estimator_params& e,
                            int64_t* out, int sm_count, cudaStream_t s);
int64_t bernstein_row(const ct_stat_row& r, const ct_estimator_params& e);
int64_t calc_ttl_row(const ct_stat_row& g, const ct_stat_row& f, const ct_estimator_params& e,
                     int64_t n_done, int64_t turns_done);

// Sets the thread-local message ct_last_error() returns (api.cu); host code in other files.
void set_last_error(const char* msg);

cudaError_t launch_jct_stats(const ct_replica_summary* s, int64_t n, int32_t n_cells,
                             ct_cell_stats* out, cudaStream_t st);

}  // namespace ct
