/* continuum.h — C ABI of libcontinuum: batched trace-replay evaluation of Continuum's
 * tool-call-aware KV-cache TTL scheduling (arXiv 2511.02230) on B200 (sm_100a).
 *
 * Three calls make up the hot path:
 *   ct_fit_ttl         TTL tables from per-tool duration samples        (§8(a) A-2)
 *   ct_simulate_batch  replay of independent agent workloads            (§8(a) A-1, A-3..A-8)
 *   ct_jct_stats       per-sweep-cell reduction of replica summaries    (§8(a) A-8)
 * Citations are PAPER.md line numbers (the paper's LaTeX source) and DESIGN.md readings.
 *
 * Conventions
 *   - Time is integer microseconds (int64); cost constants are integer picoseconds; an
 *     iteration lasts ceil(sum_ps / 1e6) µs.  Statistics are exact integers (int64 / 128-bit).
 *   - Pointers marked [dev] are CUDA device pointers, [host] are host pointers.  The caller
 *     owns every input and output buffer; the library never frees caller memory.  A ct_ctx
 *     owns only its own scratch.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).  Calls are
 *     asynchronous on that stream unless stated otherwise; results are valid after the stream
 *     is synchronised.
 *   - Every call returns CT_OK (0) or a negative CT_E* code; ct_last_error() returns a
 *     thread-local message for the last failure.  No C++ exception crosses this boundary.
 *   - Per-replica outcomes are reported in ct_replica_summary.status, not as return codes.
 *   - Outputs are a pure function of the inputs: sharding the replica range over ranks, the
 *     launch configuration and the stream do not change a single byte.
 */
#ifndef CONTINUUM_H
#define CONTINUUM_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CT_ABI_VERSION 1

/* return codes */
#define CT_OK 0
#define CT_EINVAL (-1)        /* an argument violates a documented precondition */
#define CT_ENOMEM (-2)        /* device or host allocation failed */
#define CT_ECUDA (-3)         /* a CUDA runtime call failed (message in ct_last_error) */
#define CT_EUNSUPPORTED (-4)  /* device is not compute capability 10.0 (B200, sm_100a) */

/* replica status (ct_replica_summary.status) */
#define CT_R_OK 0
#define CT_R_UNSCHEDULABLE 1  /* the head request can never fit (C-5 step 5c) */
#define CT_R_EVENT_BUDGET 2   /* more than max_iters engine iterations would be needed */
#define CT_R_INVALID_INPUT 3  /* the trace set (device buffers) violates a precondition of
                                 ct_simulate_batch; ct_validate_trace_set names it */

/* priority (PAPER.md:535-551 for PROG_FCFS; vanilla vLLM request FCFS PAPER.md:272) */
#define CT_PRIO_PROG_FCFS 0   /* key (not pinned, program index): pinned first, then FCFS */
#define CT_PRIO_REQ_FCFS 1    /* key (request arrival time, program index) */
#define CT_PRIO_PLAS 2        /* Autellix PLAS: key (attained engine time of
                                 the program, program index); every running request accrues
                                 each iteration's duration */

/* pause action on a non-final finish */
#define CT_PAUSE_EVICT 0      /* free KV at once (vanilla vLLM) */
#define CT_PAUSE_FIXED 1      /* §4.5 simplified: pin T_pin iff mean < T_thresh */
#define CT_PAUSE_PAPER 2      /* Alg. 1 CalcTTL with the online empirical-Bernstein bound */
#define CT_PAUSE_FITTED 3     /* table lookup ttl[tool][turn bucket] from ct_fit_ttl */
#define CT_PAUSE_INFERCEPT 4  /* InferCept: preserve without TTL iff the
                                 predicted tool time (tool mean if |S_f| >= N, else global mean,
                                 else T_default) < swap round trip 2 ceil(ceil(ctx/bs) c_h2d / 1e6);
                                 else evict (DRAM write-through = swap when policy.dram = 1) */

#define CT_FLAG_VICTIMS_ANY 1 /* DESIGN.md R13 alternative: victims whenever the head misses */
#define CT_FLAG_STEP_EXPIRY 2 /* DESIGN.md R4 alternative: release only at scheduling points */
#define CT_ALWAYS INT64_MAX   /* t_thresh_us sentinel: pin unconditionally (TTL grid) */

#define CT_MAX_PROGRAMS 256   /* programs per replica */
#define CT_MAX_TOOLS 64
#define CT_MAX_K 1024         /* TTL grid points */
#define CT_MAX_J 64           /* turn buckets */
#define CT_MAX_TURNS 65536    /* turns per program */
#define CT_MAX_CONTEXT (1 << 30)  /* a program's total new + decode tokens */
#define CT_TTL_SAT (1ll << 50)    /* every TTL (pin length) is below this, in µs (~35.7 years):
                                     FIXED t_pin and FITTED entries are validated against it and
                                     CalcTTL saturates at CT_TTL_SAT - 1 (R36) */

typedef struct ct_ctx ct_ctx;

/* ---- trace set ------------------------------------------------ */
typedef struct {            /* 16 B, one per program, seeds back to back */
  int64_t arr_q;            /* cumulative unit-rate Exp(1) arrival in Q20; non-decreasing in a
                               seed.  arrival_us = floor(arr_q * gap_us / 2^20), < 2^62 */
  int32_t turn0;            /* index of the program's first turn record */
  int32_t nturns;           /* >= 1 */
} ct_program;

typedef struct {            /* 16 B, one per turn */
  int32_t new_tokens;       /* tokens appended to the context this turn (>= 0) */
  int32_t decode_tokens;    /* >= 1 */
  int32_t tool;             /* tool called after this turn, 0..n_tools-1; -1 on the final turn */
  int32_t dur_us;           /* tool duration = Δ_obs of PAPER.md:622-626, >= 1 (R25); 0 on final */
} ct_turn;

typedef struct {
  const ct_program* programs;  /* [dev] n_seeds * n_programs records */
  const ct_turn* turns;        /* [dev] n_turns records */
  int64_t n_turns;
  int32_t n_seeds;
  int32_t n_programs;          /* P, programs per replica, 1..CT_MAX_PROGRAMS */
  int32_t n_tools;             /* F, 1..CT_MAX_TOOLS */
  int32_t reserved;
} ct_trace_set;

/* ---- parameters ---------------------------------------------------------------------- */
typedef struct {            /* Continuum tunables, C-1/C-2 */
  uint64_t lq;              /* round(ln(3/delta) * 2^32), delta in (0,1) => lq > 0 */
  int64_t b_us;             /* upper bound b of a tool interval, > 0 */
  int64_t t_default_us;     /* T_default, > 0 */
  int64_t n_min;            /* threshold N, >= 1 */
  int64_t a_num, a_den;     /* alpha = a_num / a_den, a_num >= 0, a_den >= 1 */
  int64_t ttl_max_us;       /* clamp (reading R8); 0 disables */
  int64_t reserved;
} ct_estimator_params;

typedef struct {            /* linear engine cost model (R16) */
  int64_t c0_ps;            /* per iteration, >= 1 */
  int64_t c_pf_ps;          /* per uncached prefill token in a request's first iteration */
  int64_t c_kv_ps;          /* per resident token (bs * blocks) per iteration */
  int64_t c_h2d_ps;         /* per block reloaded from DRAM, >= 1 when any policy uses DRAM */
  int64_t bs;               /* tokens per KV block, >= 1 */
  int64_t max_batch;        /* running + loading requests, >= 1 */
  int64_t dram_blocks;      /* DRAM tier capacity in blocks, 0 = no tier */
  int64_t max_iters;        /* engine-iteration budget per replica (CT_R_EVENT_BUDGET) */
  int64_t kv_growth;        /* 0: admission reserves the whole request, ceil((ctx+new+decode)/bs)
                               blocks (R12); 1: vLLM-style block-by-block growth with
                               recompute preemption and the preempted rank of PAPER.md:541
                               (NEXT-2, R27-R30) */
  int64_t prefill_chunk;    /* 0: a request's whole prompt runs in its first iteration (R16);
                               B > 0: chunked prefill, at most B tokens per iteration (one per
                               decoding request, then prompt chunks by rank, R31-R32).
                               Needs B >= max_batch and kv_growth = 0 (else CT_EINVAL). */
} ct_engine_params;

typedef struct {            /* 48 B */
  int32_t priority;         /* CT_PRIO_* */
  int32_t pause;            /* CT_PAUSE_* */
  int32_t dram;             /* 1 = evictions write through to the DRAM tier */
  int32_t flags;            /* CT_FLAG_* */
  int64_t t_pin_us;         /* FIXED: pin length */
  int64_t t_thresh_us;      /* FIXED: pin iff mean < t_thresh (CT_ALWAYS = always) */
  int64_t reserved[2];
} ct_policy;

/* Sweep: replica r -> (seed, rate, kv, policy) in mixed radix, policy fastest:
 *   pol = r % n_policies; kv = (r / n_policies) % n_kv; rate = (r / (n_policies n_kv)) % n_rates;
 *   seed = r / (n_policies n_kv n_rates).  Seed s replays programs [s P, (s+1) P). */
typedef struct {
  int32_t n_seeds, n_rates, n_kv, n_policies;
  const int64_t* gap_us;      /* [host] n_rates mean inter-arrival gaps (lambda = 1e6/gap JPS) */
  const int64_t* kv_blocks;   /* [host] n_kv GPU KV pool sizes in blocks */
  const ct_policy* policies;  /* [host] n_policies */
  ct_estimator_params est;
  const int64_t* fitted_ttl;  /* [dev] fitted_rows x fitted_j table for CT_PAUSE_FITTED, or NULL;
                                 entries in [0, CT_TTL_SAT) (checked on the device) */
  int32_t fitted_j;           /* 1..CT_MAX_J */
  int32_t fitted_rows;        /* >= n_tools (row f = tool f; e.g. ct_fit_ttl's ttl_argmax rows) */
} ct_sweep;

/* ---- outputs --------------------------------------------------------------------------- */
typedef struct {            /* 128 B per replica; all zero except status when status != OK */
  int32_t status;           /* CT_R_* */
  int32_t n_done;           /* completed programs */
  int64_t turns_done;
  int64_t sum_jct_us, max_jct_us, p50_jct_us, p99_jct_us;  /* nearest rank (R20) */
  int64_t sum_bubble_us;    /* waiting-queue time before admission */
  int64_t makespan_us;      /* max completion - min arrival (R19) */
  int64_t iterations;       /* engine iterations */
  int64_t busy_us;          /* engine busy time */
  int64_t prefill_tokens;   /* uncached tokens prefilled */
  int64_t recompute_tokens; /* context tokens recomputed after eviction */
  int64_t pin_hits, pin_expiries, victims, reloads;
} ct_replica_summary;

typedef struct {            /* 64 B per sweep cell (rate, kv, policy): sums over seeds */
  int64_t n_ok, n_bad, sum_done, sum_turns, sum_jct_us, max_jct_us, sum_bubble_us, sum_makespan_us;
} ct_cell_stats;

/* ---- TTL fit ----------------------------------------------------------------------------- */
/* Samples S = {(f, t)} of PAPER.md:444 (§4.2), t = Δ_obs in µs.  Two layouts:
 *  - CSR (tool_off != NULL): dur_us grouped by tool, segment f = dur_us[tool_off[f] .. tool_off[f+1]);
 *    the bandwidth path (4 B per sample);
 *  - unsorted pairs (tool_off == NULL): dur_us[i] with tool_u8[i], in arrival order; the fallback
 *    (5 B per sample, tool-keyed shared atomics), needs F x (K+1) x 8 B of shared memory.
 * dur_us must be 16-B aligned, tool_u8 4-B aligned (else CT_EINVAL). */
typedef struct {
  const int32_t* dur_us;      /* [dev] n samples, each in [0, 2^31) (negative ones are counted into
                                 ct_ttl_table.n_invalid and void the table, see CT_TTL_INVALID) */
  const int64_t* tool_off;    /* [host] n_tools + 1 non-decreasing offsets, tool_off[0] = 0,
                                 tool_off[n_tools] = n; NULL selects the unsorted layout */
  const uint8_t* tool_u8;     /* [dev] unsorted layout: tool id per sample (ids >= n_tools are
                                 invalid samples); ignored for CSR */
  int64_t n;                  /* < 2^32 */
  int32_t n_tools;            /* F, 1..CT_MAX_TOOLS */
  int32_t reserved;
} ct_samples;

/* ttl_argmax / ttl_paper entries written when the sample set held n_invalid > 0 samples outside
 * [0, 2^31) (or, unsorted layout, tool ids >= n_tools): the fit is undefined on such input, so no
 * plausible-looking table is produced.  (The call itself is asynchronous and still returns CT_OK;
 * read n_invalid after the stream synchronises.) */
#define CT_TTL_INVALID (-1)

typedef struct {            /* extension C-4 (not in PAPER.md; motivated by PAPER.md:323-338) */
  int64_t c_pf_ps;          /* prefill ps per token saved on a hit */
  int64_t c_pin_ps;         /* opportunity cost, ps per pinned block per µs */
  int64_t bs;
  int64_t a_num, a_den;     /* turn factor (1 + alpha w_j), alpha = a_num / a_den */
  int64_t grid_step_us;     /* tau_k = k * grid_step_us, k = 0..K-1 */
  int32_t K;                /* 1..CT_MAX_K */
  int32_t J;                /* turn buckets, 1..CT_MAX_J */
  int64_t ctx_tokens[CT_MAX_J];   /* expected context at turn bucket j */
  int64_t turn_weight[CT_MAX_J];  /* w_j, default j + 1 = m(r) */
  int64_t avg_turns_num;    /* paper mode: AvgTurns = num / den (turns_done / n_done), */
  int64_t avg_turns_den;    /* den = 0 => AvgTurns factor 1 (reading R7) */
} ct_cost_params;

typedef struct {
  int64_t* ttl_argmax;      /* [dev] (F+1) x J: tau* per tool row (row F = pooled samples) */
  int64_t* ttl_paper;       /* [dev] F+1: CalcTTL offset per row */
  int64_t* stats;           /* [dev] (F+1) x 4 {n, sum t~, sum t~^2 lo, hi}, t~ = min(t, b); or NULL */
  int64_t* n_invalid;       /* [dev] 1: number of invalid samples (0 on valid input); or NULL */
} ct_ttl_table;

/* ---- estimator statistics ------------------------------------------------------------------ */
typedef struct {            /* the statistics of PAPER.md:447-458 over t~ = min(t, b) (R5) */
  int64_t n;                /* |S| (or |S_f|) */
  int64_t s1;               /* sum t~ */
  uint64_t s2_lo, s2_hi;    /* sum t~^2 = s2_hi 2^64 + s2_lo */
} ct_stat_row;

/* ---- calls ------------------------------------------------------------------------------- */
int ct_version(void);
const char* ct_last_error(void);

/* Create a context on `device`.  Fails with CT_EUNSUPPORTED unless the device is sm_100. */
int ct_ctx_create(int device, ct_ctx** out);
int ct_ctx_destroy(ct_ctx* ctx);

/* TTL fit, one HBM pass over the samples:
 *  - paper mode: per tool f the statistics (n, sum t~, sum t~^2) of t~ = min(t, b) (R5), and
 *    ttl_paper[f] = CalcTTL offset with 𝓑 selected by PAPER.md:515-521 and the caller's AvgTurns;
 *  - argmax mode (extension C-4): n U(k) = V_j cnt_le(k) - C_j (sum_le(k) + tau_k (n - cnt_le(k))),
 *    V_j = floor(c_pf ctx_j (a_den + a_num w_j) / a_den), C_j = c_pin ceil(ctx_j / bs); tau* is the
 *    smallest maximiser over k >= 1 with U > 0, else 0.  Tools with n_f < N take the pooled row.
 * Launches: the histogram pass, then the finish kernel (scan / argmax / CalcTTL) as its
 * programmatic dependent launch (no launch gap); no memset: the histogram pass zeroes the other
 * half of the context's double-buffered accumulator for the next call.  Unsorted layout: the
 * pairs kernel (after a memset) then the finish kernel.  Calls on one context must be ordered
 * on one stream.
 * Preconditions (else CT_EINVAL): dur_us 16-B aligned; n < 2^32; grid_step_us, b < 2^31;
 * (K-1) step < 2^43; every product bounded so that the 128-bit arithmetic cannot overflow
 * (checked against n and the cost maxima).  Sample VALUES are checked on the device (n_invalid).
 * Errors: CT_EINVAL, CT_ENOMEM, CT_ECUDA. */
int ct_fit_ttl(ct_ctx* ctx, const ct_samples* samples, const ct_cost_params* cost,
               const ct_estimator_params* est, ct_ttl_table* out, void* stream);

/* The estimator of PAPER.md §4.2-4.3 as batched device calls over the fixed-point arithmetic
 * the replay and the fit run (C-1/C-2), for checks against the paper's worked
 * examples and for callers that keep their own statistics.
 * ct_bernstein: out[i] = B(delta) of rows[i] (printed form, reading R26):
 *   floor(s1/n) + isqrt(floor(2 v L_q / (n 2^32))) + floor(3 b L_q / (n 2^32)),
 *   v = floor((n s2 - s1^2) / (n (n-1))) (0 for n = 1), L_q = est->lq.
 * ct_calc_ttl_batch: out[i] = CalcTTL offset for global statistics g[i] and
 *   tool statistics f[i]: 𝓑 = T_default if g.n < N, else B(f) if f.n >= N, else B(g)
 *   (PAPER.md:515-521), at least 1; then floor(T_default^2 (D a_den + a_num turns_done) /
 *   (𝓑 D a_den)) for D = n_done[i] > 0, else floor(T_default^2 / 𝓑) (R7); clamped to ttl_max
 *   when > 0 (R8) and saturated at CT_TTL_SAT - 1 (R36).
 * Rows must hold the statistics of n < 2^31 samples in [0, b] (s1 <= n b, s2 <= n b^2; n >= 1
 * for ct_bernstein); n_done in [0, CT_MAX_PROGRAMS], turns_done in [0, CT_MAX_PROGRAMS
 * CT_MAX_TURNS].  Entries violating this get CT_TTL_INVALID.  All pointers [dev]; n >= 0.
 * Errors: CT_EINVAL (NULL pointers, invalid est), CT_ECUDA. */
int ct_bernstein(ct_ctx* ctx, const ct_stat_row* rows, int64_t n, const ct_estimator_params* est,
                 int64_t* out, void* stream);
int ct_calc_ttl_batch(ct_ctx* ctx, const ct_stat_row* g, const ct_stat_row* f,
                      const int64_t* n_done, const int64_t* turns_done, int64_t n,
                      const ct_estimator_params* est, int64_t* out, void* stream);
/* Host scalar references of the same two formulas (the same helpers compiled for the host; no
 * context, no device).  Return CT_TTL_INVALID on invalid rows or parameters. */
int64_t ct_bernstein_ref(const ct_stat_row* row, const ct_estimator_params* est);
int64_t ct_calc_ttl_ref(const ct_stat_row* g, const ct_stat_row* f, const ct_estimator_params* est,
                        int64_t n_done, int64_t turns_done);

/* Multi-GPU fit: the accumulator is a plain vector of int64 sums (bucket
 * counts and sums, statistic limbs, the invalid count), so accumulators of disjoint sample
 * sets add up exactly in any order.  ct_fit_acc_words(F, K) = 2 (F+1)(K+1) + 6 (F+1) + 1.
 * ct_fit_ttl_partial accumulates rank `rank`'s slice of every tool segment, samples
 * [off_f + floor(len_f rank / world), off_f + floor(len_f (rank + 1) / world)), into acc [dev]
 * (zeroed first); after an int64 SUM all-reduce of acc over the ranks, ct_fit_ttl_finish
 * computes the tables exactly as ct_fit_ttl would on all samples (byte for byte).
 * CSR layout only for world > 1.  Errors as ct_fit_ttl. */
int64_t ct_fit_acc_words(int32_t n_tools, int32_t K);  /* -1 if out of range */
int ct_fit_ttl_partial(ct_ctx* ctx, const ct_samples* samples, const ct_cost_params* cost,
                       const ct_estimator_params* est, int32_t rank, int32_t world, int64_t* acc,
                       void* stream);
int ct_fit_ttl_finish(ct_ctx* ctx, const int64_t* acc, int32_t n_tools, const ct_cost_params* cost,
                      const ct_estimator_params* est, ct_ttl_table* out, void* stream);

/* Replay replicas [replica_begin, replica_end) of the sweep:
 * Alg. 1 with §5.3 pin/unpin/victims inside an
 * integer discrete-event continuous-batching engine (C-5/C-6).
 * out[i] (and jct_us[i*P .. i*P+P-1] when jct_us != NULL) belongs to replica
 * replica_begin + i.  jct_us = completion - arrival per program, -1 when status != OK.
 * Preconditions checked on the host (else CT_EINVAL): 1 <= P <= CT_MAX_PROGRAMS; c0 >= 1,
 * bs >= 1, max_batch >= 1; the int64 fixed-point bounds of every constant, and
 * c0 + (c_pf + c_kv) bs max(kv_blocks) < 2^62 ps (one iteration), dram_blocks c_h2d < 2^62 ps
 * (one load); c_h2d >= 1 when a policy has dram = 1; 0 <= gap_us, kv_blocks < 2^30;
 * t_pin < CT_TTL_SAT; fitted_ttl with fitted_rows >= n_tools when a policy is FITTED; estimator
 * valid (a_num, a_den < 2^20, T_default, b < 2^40) when a policy uses it.
 * The trace records (device buffers) are checked on the device before the replay, as
 * ct_validate_trace_set lists; when they fail, no record is read and every replica of the call
 * reports status CT_R_INVALID_INPUT (zero summary, -1 per-program outputs).
 * Under these bounds every intermediate of the replay fits its integer type (the simulated
 * clock stays below 2^62 µs for any replica that finishes within 2^18 iterations of the
 * largest cost, and in practice for every workload).  Errors: CT_EINVAL, CT_ENOMEM, CT_ECUDA. */
int ct_simulate_batch(ct_ctx* ctx, const ct_trace_set* traces, const ct_sweep* sweep,
                      const ct_engine_params* eng, int64_t replica_begin, int64_t replica_end,
                      ct_replica_summary* out, int64_t* jct_us, void* stream);

/* Check a device trace set against the trace preconditions of ct_simulate_batch for the seeds
 * that replicas [replica_begin, replica_end) replay, plus the FITTED table when a policy uses
 * it: every program has 1 <= nturns <= CT_MAX_TURNS and its turns inside the turn array;
 * 0 <= arr_q, arr_q * max(gap_us) < 2^62, arrivals non-decreasing within a seed; every turn
 * decode >= 1, new >= 0, and (non-final) tool in [0, n_tools), dur_us >= 1; a program's total
 * new + decode tokens <= CT_MAX_CONTEXT; FITTED entries in [0, CT_TTL_SAT).  Synchronises the
 * stream.  Returns CT_OK, or CT_EINVAL naming the first offending program in ct_last_error().
 * ct_simulate_batch runs the same check asynchronously before every replay. */
int ct_validate_trace_set(ct_ctx* ctx, const ct_trace_set* traces, const ct_sweep* sweep,
                          int64_t replica_begin, int64_t replica_end, void* stream);

/* Optional per-program outputs of a replay (all [dev], n = replica_end - replica_begin).
 * summary is required; jct_us and bubble_us may be NULL.  bubble_us[i*P + p] is program p's
 * total time waiting in Q before its admissions (the per-program bubble series of PAPER.md
 * Fig. waiting_time_analysis_comparison, NEXT-3); -1 for replicas whose status is not OK. */
typedef struct {
  ct_replica_summary* summary;
  int64_t* jct_us;
  int64_t* bubble_us;
} ct_replay_outputs;

/* ct_simulate_batch with the optional per-program bubble output.  Same errors. */
int ct_simulate_batch_ex(ct_ctx* ctx, const ct_trace_set* traces, const ct_sweep* sweep,
                         const ct_engine_params* eng, int64_t replica_begin, int64_t replica_end,
                         const ct_replay_outputs* out, void* stream);

/* Same as ct_simulate_batch but with HOST buffers: programs/turns in traces->programs/turns are
 * host pointers, out/jct_us are host pointers.  Copies in, checks the records of the seeds the
 * replica range touches on the device (ct_validate_trace_set: CT_EINVAL naming the first bad
 * program), runs, copies out and synchronises the stream before returning (end-to-end path;
 * pinned host memory recommended). */
int ct_simulate_batch_host(ct_ctx* ctx, const ct_trace_set* host_traces, const ct_sweep* sweep,
                           const ct_engine_params* eng, int64_t replica_begin,
                           int64_t replica_end, ct_replica_summary* host_out,
                           int64_t* host_jct_us, void* stream);

/* Per sweep cell (rate, kv, policy) sums over seeds of a full sweep's summaries (R19, R21).
 * n_replicas must be a multiple of n_cells; replica r belongs to cell r % n_cells.
 * summaries [dev] n_replicas, out [dev] n_cells.  Errors: CT_EINVAL, CT_ECUDA. */
int ct_jct_stats(ct_ctx* ctx, const ct_replica_summary* summaries, int64_t n_replicas,
                 int32_t n_cells, ct_cell_stats* out, void* stream);

/* On-device trace synthesis (NEXT-4).  Writes the trace set that
 * ctgen/synth.py defines (an integer-only generator: SplitMix64 counters, quantile tables with
 * 16-bit interpolation) for seeds [seed0, seed0 + n_seeds), P programs
 * each, straight into HBM: no host generation and no host-to-device copy of the traces.
 * Tables are int64[1025] quantiles at p = i/1024, monotone, values < 2^46. */
#define CT_SYNTH_TABLE 1025
typedef struct {
  int64_t stream;           /* generator stream (key part 0) */
  int64_t ctx_cap;          /* R24: a program keeps the leading turns whose cumulative
                               new + decode <= ctx_cap; >= 8192 */
  int32_t max_turns;        /* 2..1024 */
  int32_t n_bfcl;           /* BFCL programs per seed (rank of the mix key < n_bfcl) */
  int32_t n_tools;          /* F, 1..CT_MAX_TOOLS */
  int32_t reserved;
  const int64_t* turns_swe; /* [host] [1025] SWE turn-count quantiles */
  const int64_t* obs;       /* [host] [2][1025] observation tokens (SWE, BFCL) */
  const int64_t* dec;       /* [host] [2][1025] decode tokens (SWE, BFCL) */
  const int64_t* dur;       /* [host] [F][1025] tool durations, µs */
  const int64_t* exp_q20;   /* [host] [1025] unit-rate arrival gaps in Q20 */
  const uint32_t* tool_cdf; /* [host] [F] cumulative u32 threshold within the tool's class */
  const int32_t* tool_class;/* [host] [F] 0 = SWE, 1 = BFCL (each class has >= 1 tool) */
} ct_synth_params;

/* programs [dev] n_seeds * P records (turn0 relative to `turns`); turns [dev] turns_cap records;
 * *n_turns [host] receives the number written.  Synchronises `stream` (the turn count is
 * needed on the host).  Errors: CT_EINVAL (bad parameters, P not in [1, CT_MAX_PROGRAMS],
 * turns_cap too small: *n_turns still receives the count needed, nothing is written to
 * turns), CT_ENOMEM, CT_ECUDA. */
int ct_synthesize_traces(ct_ctx* ctx, const ct_synth_params* sp, int64_t seed0, int32_t n_seeds,
                         int32_t n_programs, ct_program* programs, ct_turn* turns,
                         int64_t turns_cap, int64_t* n_turns, void* stream);

/* ---- host-side trace ingest (NEXT-4) ----------------------------------
 * These two calls run on the host only (no CUDA call, no context): they turn recorded agent
 * traces into the ct_program / ct_turn records the replay reads.  DESIGN.md R33-R35. */

/* tool-call formats of ct_parse_tool_name (§5.2 and App. A) */
#define CT_TOOLFMT_AUTO 0       /* detect: JSON (OPENAI / NAME / TERMINAL by its keys), a ```bash
                                   fence, a <tool_call> wrapper, a pythonic call; else no call */
#define CT_TOOLFMT_OPENAI 1     /* JSON block or array of blocks; the first block whose "type"
                                   names a function/tool call gives "name" (or "function"."name")
                                    */
#define CT_TOOLFMT_NAME 2       /* Qwen-3 style {"name": f, "arguments": {...}} (App. A) */
#define CT_TOOLFMT_PYTHONIC 3   /* Llama-3 style f(p1=v1, ...) or [f(...), ...] (App. A) */
#define CT_TOOLFMT_BASH 4       /* bash command (the ```bash block if one is present, else the
                                   whole message): split on && and ||, first whitespace token
                                   of the first sub-command (App. A) */
#define CT_TOOLFMT_TERMINAL 5   /* Terminal-Bench {"commands": [{"keystrokes": ...}, ...]}: the
                                   first command's keystrokes parsed as BASH (App. A) */

/* Extract the tool name of one model output message.  msg [host] is `len` bytes of UTF-8 (need
 * not be NUL-terminated).  On CT_OK, *name_len = length of the name written to name [host]
 * (NUL-terminated, at most name_cap - 1 bytes) or 0 when the message holds no tool call, and
 * *malformed = 1 when a structured block (JSON) could not be parsed or lacks its name (the name
 * is then absent; SPEC.md:164 counts these as parse warnings), else 0.
 * Errors: CT_EINVAL (NULL pointers, len < 0, unknown format, name longer than name_cap - 1). */
int ct_parse_tool_name(const char* msg, int64_t len, int32_t format, char* name, int32_t name_cap,
                       int32_t* name_len, int32_t* malformed);

/* Load a JSONL trace: one program per line,
 *   {"program_id": str|int, "arrival_time_s": num, "turns": [turn, ...]}
 *   turn = {"new_prompt_tokens": int >= 0, "decode_tokens": int >= 1,
 *           "tool_name": str, "tool_duration_s": num >= 0}   (tool fields on non-final turns)
 * where a non-final turn may give "message" (the raw model output, parsed with
 * ct_parse_tool_name(format)) instead of "tool_name".  Blank lines are skipped; unknown keys are
 * ignored.  Validation: turns non-empty; decode >= 1; tool fields present on
 * every non-final turn and absent on the final one; cumulative new + decode <= ctx_window when
 * ctx_window > 0.  Times are parsed from their decimal text exactly and rounded half away from
 * zero to integer µs; tool durations below 1 µs become 1 µs (R25).  Programs are sorted by
 * arrival (stable; file order on ties) and written as one seed with arr_q = arrival µs, so a
 * sweep with gap_us = 2^20 replays the recorded arrivals and any other gap scales them (R34).
 * Tool ids: the first n_known names of `tool_names` keep their ids; other names are appended
 * in order of first use (after sorting).  tool_names [host] is a table of 64-byte NUL-padded
 * entries with room for CT_MAX_TOOLS; names must be 1..63 bytes.
 * Two-call use: with programs == NULL or turns == NULL nothing but the counts is written.
 * Outputs: counts[0] = programs, counts[1] = turns, counts[2] = tools (known + new),
 *          counts[3] = malformed tool-call messages (warnings), counts[4] = failing line (1-based,
 *          0 on success).
 * Errors: CT_EINVAL (unreadable file, JSON or schema violation, named with its line and field in
 * ct_last_error; more than CT_MAX_TOOLS tools; capacity too small: counts still filled),
 * CT_ENOMEM. */
int ct_load_trace_jsonl(const char* path, int32_t format, int64_t ctx_window, char* tool_names,
                        int32_t n_known, ct_program* programs, int64_t programs_cap,
                        ct_turn* turns, int64_t turns_cap, int64_t* counts);

/* Launch statistics of the last ct_simulate_batch / ct_fit_ttl on this context (bench
 * accounting).  With timing enabled (ct_ctx_set_timing), the library records CUDA events on the
 * caller's stream around the dominant kernel of each call (replay_kernel, fit_hist_kernel);
 * ct_last_launch then waits for them and reports the kernel-only durations in milliseconds
 * (-1 when not timed). */
typedef struct {
  int32_t grid, block, warps_per_block, slots_per_lane;
  int64_t smem_per_block;
  int64_t launches;         /* kernels launched by the last ct_simulate_batch */
  float replay_ms;          /* last replay_kernel duration */
  float fit_hist_ms;        /* last fit_hist_kernel duration */
  int32_t kernel_mode;      /* replay specialisation of the last call: 0 generic,
                               1 TTL-grid class (P <= 32, 32-bit times) or program-FCFS class
                               (P > 32, 64-bit), 2 mixed, 3 simple class (P <= 32, 32-bit),
                               4 program-FCFS class (P > 32, 32-bit) + list-driven 64-bit launch,
                               5 as 4 with request FCFS (simple class), 6 extended class
                               (P <= 32, 32-bit: + DRAM tier, PLAS, InferCept); 10 + m: two
                               launches over policy subsets, MODE 1 for the TTL-grid policies
                               and MODE m (2, 3 or 6) for the others */
  int32_t reserved;
} ct_launch_info;
int ct_last_launch(ct_ctx* ctx, ct_launch_info* info);
int ct_ctx_set_timing(ct_ctx* ctx, int enable);

#ifdef __cplusplus
}
#endif
#endif
