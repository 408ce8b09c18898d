/* ct_oracle.h — CPU ORACLE FOR TESTS ONLY.
 *
 * TEST INFRASTRUCTURE: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2511_02230_b200/, libcontinuum) never includes, links or calls it, and
 * this file includes nothing from the product (no shared headers or helpers).
 *
 * A plain, slow, single-threaded-per-replica implementation of what Continuum
 * (arXiv 2511.02230) computes, written from PAPER.md step by step:
 *   - or_bernstein / or_select_bound / or_calc_ttl / or_simplified : §4.2-4.5
 *     (PAPER.md:440-562), fixed-point readings C-1..C-3 of DESIGN.md.
 *   - or_fit : the north-star TTL fit (extension C-4), computed from its plain
 *     definition over raw samples, O(n*K), no bucketing.
 *   - or_simulate : Alg. 1 + §5.3 inside a
 *     per-ITERATION discrete-event model of a continuous-batching engine
 *     (readings R1-R26 of DESIGN.md), no macro-stepping.
 *
 * Flat int64 parameter vectors (indices documented in ct_oracle.cpp) keep this
 * ABI independent of include/continuum.h.
 */
#ifndef CT_ORACLE_H
#define CT_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

uint64_t or_isqrt(uint64_t lo, uint64_t hi);  /* floor(sqrt(hi 2^64 + lo)) */
/* B(delta) of PAPER.md:469-474 in integer µs; s2 = s2_hi*2^64 + s2_lo. */
int64_t or_bernstein(int64_t n, int64_t s1, uint64_t s2_lo, uint64_t s2_hi,
                     uint64_t lq, int64_t b_us);
/* 𝓑(r,f) of PAPER.md:515-521. stats rows: {n, s1, s2_lo, s2_hi}. */
int64_t or_select_bound(const int64_t* g, const int64_t* f, const int64_t* est);
/* CalcTTL offset with AvgTurns = turns_done / n_done. */
int64_t or_calc_ttl(const int64_t* g, const int64_t* f, const int64_t* est,
                    int64_t n_done, int64_t turns_done);
/* §4.5 simplified decision: returns T_pin or 0. */
int64_t or_simplified(const int64_t* g, const int64_t* f, const int64_t* est,
                      int64_t t_pin, int64_t t_thresh);

/* InferCept baseline (NEXT-1): predicted tool time and swap round trip (µs). */
int64_t or_infercept_predict(const int64_t* g, const int64_t* f, const int64_t* est);
int64_t or_infercept_swap_us(int64_t ctx, int64_t bs, int64_t c_h2d_ps);

/* TTL fit (extension C-4 + paper-mode C-2 per tool).
 * dur[n] grouped by tool, tool_off[F+1]; cost = {c_pf, c_pin, bs, a_num, a_den,
 * delta_us, K, J}; ctx_j[J], w_j[J]; est = estimator vector; avg = {turns_done, n_done}.
 * out: ttl_argmax[(F+1)*J], ttl_paper[F+1], stats[(F+1)*4]. */
int or_fit(const int32_t* dur, const int64_t* tool_off, int F,
           const int64_t* cost, const int64_t* ctx_j, const int64_t* w_j,
           const int64_t* est, const int64_t* avg,
           int64_t* ttl_argmax, int64_t* ttl_paper, int64_t* stats);

/* Replay replicas [r_begin, r_end) of a sweep.
 * progs: 16-B records {i64 arr_q, i32 turn0, i32 nturns} [S*P]; turns: i32[T][4].
 * summary: int64[16] per replica; jct, bubble: int64[P] per replica (or NULL); bubble is
 * each program's total waiting time before admissions (NEXT-3 per-program bubble series).
 * Returns 0, or a negative value on invalid input. */
int or_simulate(const void* progs, const int32_t* turns, int64_t n_turns,
                int S, int P, int F,
                const int64_t* gap_us, int n_rate, const int64_t* kv_blocks, int n_kv,
                const int64_t* policies, int n_pol, const int64_t* est,
                const int64_t* eng, const int64_t* fitted, int J,
                int64_t r_begin, int64_t r_end, int n_threads,
                int64_t* summary, int64_t* jct, int64_t* bubble);

/* One replica with the per-decision audit log of SPEC.md:433 (pin / unpin with the reason
 * hit | expiry | victim / evict / admit / done, each with its µs timestamp) as JSON lines in buf.
 * Returns 0, 1 if cap < *len (the log is truncated; *len is its full size), <0 on bad input. */
int or_simulate_audit(const void* progs, const int32_t* turns, int64_t n_turns, int S, int P, int F,
                      const int64_t* gap_us, int n_rate, const int64_t* kv_blocks, int n_kv,
                      const int64_t* policies, int n_pol, const int64_t* est, const int64_t* eng,
                      const int64_t* fitted, int J, int64_t replica, char* buf, int64_t cap,
                      int64_t* len, int64_t* summary);

/* Per sweep cell sums over seeds (cells = rate x kv x policy). out: int64[8] per cell. */
int or_jct_stats(const int64_t* summary, int64_t n_replicas, int n_cells, int64_t* out);

#ifdef __cplusplus
}
#endif
#endif
