// ct_oracle.cpp — CPU ORACLE FOR TESTS ONLY (see ct_oracle.h).
//
// TEST INFRASTRUCTURE: loaded only by tests/, __graft_entry__.smoke() and the
// cpu_baseline / --impl reference legs of bench.py.  Shares no code with the
// CUDA path.  Plain, slow, obviously correct: linear scans over programs, one
// loop turn per engine iteration, 128-bit integers written out.
//
// Parameter vectors (int64):
//   est  = {L_q, b_us, T_default_us, N, a_num, a_den, ttl_max_us, 0}
//   eng  = {c0_ps, c_pf_ps, c_kv_ps, c_h2d_ps, bs, max_batch, dram_blocks, max_iters,
//           kv_growth, prefill_chunk}
//   pol  = {priority, pause, dram, flags, t_pin_us, t_thresh_us, 0, 0}
//   cost = {c_pf_ps, c_pin_ps, bs, a_num, a_den, grid_step_us, K, J}
// Summary (int64[16]) per replica:
//   0 status | n_done<<32, 1 turns_done, 2 sum_jct, 3 max_jct, 4 p50_jct, 5 p99_jct,
//   6 sum_bubble, 7 makespan, 8 iterations, 9 busy_us, 10 prefill_tokens,
//   11 recompute_tokens, 12 pin_hits, 13 pin_expiries, 14 victims, 15 reloads.
#include "ct_oracle.h"

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

typedef __int128 i128;
typedef unsigned __int128 u128;

static const int64_t INF = INT64_MAX;
static const int64_t ALWAYS = INT64_MAX;

static int64_t ceil_div(i128 a, i128 b) { return (int64_t)((a + b - 1) / b); }  // a >= 0, b > 0

// ---------------------------------------------------------------------------
// §4.2 estimator, fixed point (C-1).
// ---------------------------------------------------------------------------

// floor(sqrt(x)) of x = hi 2^64 + lo, bit by bit (the result has at most 64 bits).
uint64_t or_isqrt(uint64_t lo, uint64_t hi) {
  const u128 x = ((u128)hi << 64) | lo;
  uint64_t r = 0;
  for (int bit = 63; bit >= 0; --bit) {
    uint64_t c = r | (1ull << bit);
    if ((u128)c * c <= x) r = c;
  }
  return r;
}

// B(delta) = mu + sqrt(2 sigma^2 ln(3/delta) / n) + 3 b ln(3/delta) / n
// mu = floor(s1/n); sigma^2 = floor((n s2 - s1^2) / (n (n-1))), 0 when n = 1;
// ln(3/delta) = L_q / 2^32; each term floored.
int64_t or_bernstein(int64_t n, int64_t s1, uint64_t s2_lo, uint64_t s2_hi, uint64_t lq,
                     int64_t b_us) {
  if (n < 1) return -1;
  u128 s2 = ((u128)s2_hi << 64) | s2_lo;
  int64_t mu = s1 / n;
  u128 var = 0;
  if (n >= 2) {
    u128 num = (u128)n * s2 - (u128)s1 * (u128)s1;
    var = num / ((u128)n * (u128)(n - 1));
  }
  u128 arg2 = ((u128)2 * var * (u128)lq) / ((u128)n << 32);
  uint64_t term2 = or_isqrt((uint64_t)arg2, (uint64_t)(arg2 >> 64));  // sqrt of all 128 bits
  u128 term3 = ((u128)3 * (u128)b_us * (u128)lq) / ((u128)n << 32);
  return mu + (int64_t)term2 + (int64_t)term3;
}

static int64_t bern_row(const int64_t* st, const int64_t* est) {
  return or_bernstein(st[0], st[1], (uint64_t)st[2], (uint64_t)st[3], (uint64_t)est[0], est[1]);
}

// 𝓑(r,f) = T_default if |S| < N; B_f if |S_f| >= N; B otherwise; >= 1.
int64_t or_select_bound(const int64_t* g, const int64_t* f, const int64_t* est) {
  const int64_t N = est[3], T_def = est[2];
  int64_t B;
  if (g[0] < N) B = T_def;
  else if (f[0] >= N) B = bern_row(f, est);
  else B = bern_row(g, est);
  return B < 1 ? 1 : B;
}

// CalcTTL - now = T_default^2 / 𝓑 * (1 + alpha * AvgTurns)
// alpha = a_num/a_den, AvgTurns = turns_done / n_done (0 before any completion, R7);
// clamp to ttl_max when > 0 (R8); saturate at 2^50 - 1 (R36).
int64_t or_calc_ttl(const int64_t* g, const int64_t* f, const int64_t* est, int64_t n_done,
                    int64_t turns_done) {
  const int64_t T = est[2], a_num = est[4], a_den = est[5], ttl_max = est[6];
  int64_t B = or_select_bound(g, f, est);
  u128 ttl;
  if (n_done > 0) {
    u128 num = (u128)T * (u128)T * ((u128)n_done * a_den + (u128)a_num * turns_done);
    u128 den = (u128)B * (u128)n_done * (u128)a_den;
    ttl = num / den;
  } else {
    ttl = ((u128)T * (u128)T) / (u128)B;
  }
  if (ttl_max > 0 && ttl > (u128)ttl_max) ttl = ttl_max;
  // R36: a pin length is a µs count below 2^50 (~35.7 years, beyond any replay horizon);
  // without a clamp the formula can exceed int64 (T_default^2 / 𝓑 with T_default < 2^40)
  if (ttl >= ((u128)1 << 50)) ttl = ((u128)1 << 50) - 1;
  return (int64_t)ttl;
}

// §4.5: pin for T_pin iff historical mean < T_thresh.  Mean of the
// tool when |S_f| >= N, else global when |S| >= 1, else none (no pin) (R9).
int64_t or_simplified(const int64_t* g, const int64_t* f, const int64_t* est, int64_t t_pin,
                      int64_t t_thresh) {
  if (t_thresh == ALWAYS) return t_pin;
  const int64_t N = est[3];
  int64_t mu;
  if (f[0] >= N) mu = f[1] / f[0];
  else if (g[0] >= 1) mu = g[1] / g[0];
  else return 0;
  return mu < t_thresh ? t_pin : 0;
}

// InferCept: predicted tool time = mean of the tool
// when |S_f| >= N, else the global mean when |S| >= 1, else T_default.
int64_t or_infercept_predict(const int64_t* g, const int64_t* f, const int64_t* est) {
  if (f[0] >= est[3]) return f[1] / f[0];
  if (g[0] >= 1) return g[1] / g[0];
  return est[2];
}

// Swap round trip of a context: out + in, each ceil(blocks * c_h2d / 1e6) µs, blocks = ceil(ctx/bs).
int64_t or_infercept_swap_us(int64_t ctx, int64_t bs, int64_t c_h2d_ps) {
  int64_t blocks = ceil_div(ctx, bs);
  return 2 * ceil_div((i128)blocks * c_h2d_ps, 1000000);
}

// ---------------------------------------------------------------------------
// TTL fit (extension C-4): plain definition over raw samples.
// ---------------------------------------------------------------------------
int or_fit(const int32_t* dur, const int64_t* tool_off, int F, const int64_t* cost,
           const int64_t* ctx_j, const int64_t* w_j, const int64_t* est, const int64_t* avg,
           int64_t* ttl_argmax, int64_t* ttl_paper, int64_t* stats) {
  const int64_t c_pf = cost[0], c_pin = cost[1], bs = cost[2], a_num = cost[3], a_den = cost[4];
  const int64_t step = cost[5], K = cost[6], J = cost[7];
  const int64_t b_us = est[1], N = est[3];
  if (F < 1 || K < 1 || J < 1 || step < 1 || bs < 1 || a_den < 1) return -1;
  std::vector<int64_t> arg((size_t)(F + 1) * J, 0);
  std::vector<int64_t> st((size_t)(F + 1) * 4, 0);
  for (int row = 0; row <= F; ++row) {
    int64_t lo = row < F ? tool_off[row] : tool_off[0];
    int64_t hi = row < F ? tool_off[row + 1] : tool_off[F];
    int64_t n = hi - lo;
    // paper-mode statistics over t~ = min(t, b)  (R5)
    int64_t s1 = 0;
    u128 s2 = 0;
    for (int64_t i = lo; i < hi; ++i) {
      int64_t t = dur[i] < b_us ? dur[i] : b_us;
      s1 += t;
      s2 += (u128)t * (u128)t;
    }
    st[row * 4 + 0] = n;
    st[row * 4 + 1] = s1;
    st[row * 4 + 2] = (int64_t)(uint64_t)s2;
    st[row * 4 + 3] = (int64_t)(uint64_t)(s2 >> 64);
    // cnt_le(k) = #{d <= tau_k}, sum_le(k) = sum_{d <= tau_k} d, tau_k = k * step
    std::vector<int64_t> cnt(K, 0), sum(K, 0);
    for (int64_t k = 0; k < K; ++k) {
      int64_t tau = k * step;
      for (int64_t i = lo; i < hi; ++i)
        if (dur[i] <= tau) { cnt[k] += 1; sum[k] += dur[i]; }
    }
    for (int64_t j = 0; j < J; ++j) {
      // V_j = c_pf ctx_j (1 + alpha w_j) [ps saved], C_j = c_pin ceil(ctx_j / bs) [ps per µs pinned]
      i128 V = ((i128)c_pf * ctx_j[j] * ((i128)a_den + (i128)a_num * w_j[j])) / a_den;
      i128 C = (i128)c_pin * ceil_div(ctx_j[j], bs);
      i128 best = 0;  // U(0) = 0: TTL 0 means no pin
      int64_t best_k = 0;
      for (int64_t k = 1; k < K; ++k) {
        i128 tau = (i128)k * step;
        i128 U = V * cnt[k] - C * ((i128)sum[k] + tau * (n - cnt[k]));
        if (U > best) { best = U; best_k = k; }
      }
      arg[row * J + j] = best_k * step;
    }
  }
  // tools with n_f < N fall back to the pooled row (mirrors PAPER.md:492-494)
  for (int f = 0; f < F; ++f)
    if (st[f * 4] < N)
      for (int64_t j = 0; j < J; ++j) arg[f * J + j] = arg[(size_t)F * J + j];
  for (int row = 0; row <= F; ++row) {
    const int64_t* g = &st[(size_t)F * 4];
    const int64_t* f = &st[(size_t)row * 4];
    ttl_paper[row] = or_calc_ttl(g, f, est, avg[1], avg[0]);
  }
  std::memcpy(ttl_argmax, arg.data(), arg.size() * 8);
  std::memcpy(stats, st.data(), st.size() * 8);
  return 0;
}

// ---------------------------------------------------------------------------
// Replay: Alg. 1 inside a per-iteration engine model (C-5/C-6).
// ---------------------------------------------------------------------------
namespace {

enum { NOT_ARRIVED = 0, QUEUED = 1, RUNNING = 2, LOADING = 3, READY = 4, TOOL = 5, DONE = 6 };
enum { PRIO_PROG_FCFS = 0, PRIO_REQ_FCFS = 1, PRIO_PLAS = 2 };
enum { PAUSE_EVICT = 0, PAUSE_FIXED = 1, PAUSE_PAPER = 2, PAUSE_FITTED = 3, PAUSE_INFERCEPT = 4 };
enum { FLAG_VICTIMS_ANY = 1, FLAG_STEP_EXPIRY = 2 };
enum { ST_OK = 0, ST_UNSCHED = 1, ST_BUDGET = 2, ST_INVARIANT = -1 };

struct Prog {
  int st = NOT_ARRIVED;
  int turn = 0;
  int64_t ctx = 0, gblk = 0, dblk = 0;
  bool pinned = false;
  int64_t expiry = 0, req_arr = 0, t_ret = 0, load_done = 0, emitted = 0;
  int64_t arrival = 0, completion = -1;
  int64_t service = 0;  // attained engine time (Autellix PLAS)
  int64_t bubble = 0;   // this program's waiting time before admissions (NEXT-3 series)
  int64_t prem = 0;     // prefill tokens of the current request not yet computed
  int64_t chunk = 0;    // prefill tokens computed in the iteration in flight
  bool emit = false;    // emits a token at the end of the iteration in flight
  bool preempted = false;  // recompute-preempted, back in Q (NEXT-2, R28)
  // JCT accounting: time spent in each lifecycle state, accumulated at every
  // state change, and the tool time the trace prescribes
  int64_t since = 0;
  int64_t in_state[7] = {0, 0, 0, 0, 0, 0, 0};
  int64_t tool_us = 0;
};

struct Row { int64_t n = 0, s1 = 0; u128 s2 = 0; };

struct Sim {
  // inputs
  const uint8_t* progs;
  const int32_t* turns;
  int P, F, J;
  int64_t gap, kv;
  const int64_t* pol;
  const int64_t* est;
  const int64_t* eng;
  const int64_t* fitted;
  int seed;
  // state
  std::vector<Prog> p;
  std::vector<Row> tool;
  Row glob;
  int64_t now = 0, free_blk = 0, dram_free = 0, chan_free = 0;
  int64_t D = 0, turns_done = 0;
  bool in_flight = false;
  int64_t iter_end = 0;
  int next_arr = 0;
  int status = ST_OK;
  int64_t pins_created = 0;
  std::string* audit = nullptr;  // per-decision log, JSON lines, or NULL

  void log(const char* ev, int i, const char* extra = "") {
    if (!audit) return;
    char b[256];
    snprintf(b, sizeof b, "{\"t\":%lld,\"ev\":\"%s\",\"p\":%d%s}\n", (long long)now, ev, i, extra);
    *audit += b;
  }
  // counters
  int64_t iterations = 0, busy = 0, bubble = 0, prefill = 0, recompute = 0;
  int64_t hits = 0, expiries = 0, victims = 0, reloads = 0;

  int64_t prog_arr_q(int i) const { int64_t v; std::memcpy(&v, progs + 16 * (size_t)(seed * P + i), 8); return v; }
  int32_t prog_turn0(int i) const { int32_t v; std::memcpy(&v, progs + 16 * (size_t)(seed * P + i) + 8, 4); return v; }
  int32_t prog_nturns(int i) const { int32_t v; std::memcpy(&v, progs + 16 * (size_t)(seed * P + i) + 12, 4); return v; }
  const int32_t* turn_rec(int i, int t) const { return turns + 4 * ((int64_t)prog_turn0(i) + t); }
  int64_t arrival_time(int i) const { return (int64_t)(((i128)prog_arr_q(i) * gap) >> 20); }

  // every lifecycle transition goes through here, so in_state[] partitions [arrival, completion]
  void set_state(int i, int st) {
    p[i].in_state[p[i].st] += now - p[i].since;
    p[i].since = now;
    p[i].st = st;
  }

  bool dram_on() const { return pol[2] != 0 && eng[6] > 0; }
  bool growth() const { return eng[8] != 0; }  // NEXT-2 block-by-block KV growth (R27)
  int64_t budget() const { return eng[9]; }     // NEXT-2 chunked prefill token budget (R31), 0 = off

  // R31/R32: token budget left after the running requests: one token per decoding request,
  // then the prefilling ones in rank order (R28) take min(remaining prefill, budget left).
  // Sets chunk for every running request; returns the budget left for admissions.
  int64_t assign_running() {
    int64_t left = budget();
    for (int i = 0; i < P; ++i)
      if (p[i].st == RUNNING && p[i].prem == 0) left -= 1;
    std::vector<int> order;
    for (int i = 0; i < P; ++i)
      if (p[i].st == RUNNING) { p[i].chunk = 0; if (p[i].prem > 0) order.push_back(i); }
    std::sort(order.begin(), order.end(), [&](int a, int b) { return run_before(a, b); });
    for (int i : order) {
      p[i].chunk = std::min(p[i].prem, std::max<int64_t>(left, 0));
      left -= p[i].chunk;
    }
    return left;
  }
  bool eager() const { return (pol[3] & FLAG_STEP_EXPIRY) == 0; }

  // evict(v): free GPU blocks; DRAM write-through when the tier is on (R18).
  void evict(int v) {
    free_blk += p[v].gblk;
    p[v].gblk = 0;
    if (dram_on()) {
      dram_free += p[v].dblk;
      p[v].dblk = 0;
      int64_t nb = ceil_div(p[v].ctx, eng[4]);
      if (nb > 0 && nb <= dram_free) { p[v].dblk = nb; dram_free -= nb; }
    }
  }

  void record(int f, int64_t d) {  // Alg. 1 line 7: update global and per-tool stats
    int64_t t = d < est[1] ? d : est[1];
    Row* rows[2] = {&glob, &tool[f]};
    for (Row* r : rows) { r->n += 1; r->s1 += t; r->s2 += (u128)t * (u128)t; }
  }

  int64_t ttl_for(int i) {  // pause action on a non-final finish
    const int32_t* tr = turn_rec(i, p[i].turn);
    int f = tr[2];
    int64_t g[4] = {glob.n, glob.s1, (int64_t)(uint64_t)glob.s2, (int64_t)(uint64_t)(glob.s2 >> 64)};
    const Row& r = tool[f];
    int64_t fr[4] = {r.n, r.s1, (int64_t)(uint64_t)r.s2, (int64_t)(uint64_t)(r.s2 >> 64)};
    switch (pol[1]) {
      case PAUSE_EVICT: return 0;
      case PAUSE_FIXED: return or_simplified(g, fr, est, pol[4], pol[5]);
      case PAUSE_PAPER: return or_calc_ttl(g, fr, est, D, turns_done);
      case PAUSE_FITTED: {
        int j = p[i].turn < J - 1 ? p[i].turn : J - 1;
        return fitted[(int64_t)f * J + j];
      }
      case PAUSE_INFERCEPT: {  // preserve (no TTL) iff predicted tool time < swap round trip
        int64_t pred = or_infercept_predict(g, fr, est);
        int64_t swap = or_infercept_swap_us(p[i].ctx, eng[4], eng[3]);
        return pred < swap ? INF : 0;
      }
    }
    return 0;
  }

  void finish(int i) {  // OnRequestFinish
    const int32_t* tr = turn_rec(i, p[i].turn);
    p[i].ctx += tr[0] + tr[1];
    if (p[i].turn == prog_nturns(i) - 1) {  // last request: free KV, program completes
      free_blk += p[i].gblk; p[i].gblk = 0;
      dram_free += p[i].dblk; p[i].dblk = 0;
      p[i].completion = now; set_state(i, DONE);
      log("done", i);
      D += 1; turns_done += prog_nturns(i);
      return;
    }
    int64_t ttl = ttl_for(i);
    if (ttl > 0) {  // pin_request(request, TTL) only if TTL != 0
      p[i].pinned = true; p[i].expiry = ttl == INF ? INF : now + ttl; pins_created++;
      if (audit) {
        char x[64];
        if (ttl == INF) snprintf(x, sizeof x, ",\"ttl\":null");
        else snprintf(x, sizeof x, ",\"ttl\":%lld", (long long)ttl);
        log("pin", i, x);
      }
    } else {
      evict(i);
      log("evict", i);
    }
    p[i].t_ret = now + tr[3];
    p[i].tool_us += tr[3];
    set_state(i, TOOL);
  }

  int head() {  // argmax priority over Q
    // preempted requests first (reading R29); they exist only with KV growth
    bool any_pre = false;
    for (int i = 0; i < P; ++i) any_pre |= p[i].st == QUEUED && p[i].preempted;
    auto cand = [&](int i) { return p[i].st == QUEUED && (!any_pre || p[i].preempted); };
    int best = -1;
    if (pol[0] == PRIO_PROG_FCFS) {
      if (!any_pre)
        for (int i = 0; i < P; ++i) if (cand(i) && p[i].pinned) return i;
      for (int i = 0; i < P; ++i) if (cand(i)) return i;
    } else if (pol[0] == PRIO_REQ_FCFS) {
      for (int i = 0; i < P; ++i)
        if (cand(i) && (best < 0 || p[i].req_arr < p[best].req_arr)) best = i;
    } else {  // PLAS: least attained service first, ties by program arrival
      for (int i = 0; i < P; ++i)
        if (cand(i) && (best < 0 || p[i].service < p[best].service)) best = i;
    }
    return best;
  }

  // Priority among RUNNING requests (reading R28): true iff a ranks above b.
  bool run_before(int a, int b) const {
    if (pol[0] == PRIO_REQ_FCFS && p[a].req_arr != p[b].req_arr) return p[a].req_arr < p[b].req_arr;
    if (pol[0] == PRIO_PLAS && p[a].service != p[b].service) return p[a].service < p[b].service;
    return a < b;
  }

  // vLLM recompute preemption (R28): drop the GPU KV, back to Q marked preempted.
  void preempt(int v) {
    free_blk += p[v].gblk;
    p[v].gblk = 0;
    set_state(v, QUEUED);
    p[v].preempted = true;
    p[v].req_arr = now;
  }

  // Growth step (R27/R28): every running request needs a slot for its next token, i.e.
  // ceil((ctx + new + emitted + 1) / bs) blocks; served in priority order; when no block is
  // free the lowest-priority running request (possibly itself) is preempted.
  void grow_running() {
    const int64_t bs = eng[4];
    std::vector<int> order;
    for (int i = 0; i < P; ++i) if (p[i].st == RUNNING) order.push_back(i);
    std::sort(order.begin(), order.end(), [&](int a, int b) { return run_before(a, b); });
    for (int i : order) {
      if (p[i].st != RUNNING) continue;  // preempted earlier in this pass
      const int32_t* tr = turn_rec(i, p[i].turn);
      const int64_t need = ceil_div(p[i].ctx + tr[0] + p[i].emitted + 1, bs) - p[i].gblk;
      while (need > free_blk) {
        int v = -1;
        for (int j = 0; j < P; ++j)
          if (p[j].st == RUNNING && (v < 0 || run_before(v, j))) v = j;
        preempt(v);
        if (v == i) break;
      }
      if (p[i].st == RUNNING && need > 0) { free_blk -= need; p[i].gblk += need; }
    }
  }

  bool schedule() {  // returns false when the replica stops (unschedulable / budget)
    const int64_t bs = eng[4];
    // (a) release expired pins of programs not in Q
    for (int i = 0; i < P; ++i)
      if (p[i].pinned && p[i].st != QUEUED && now > p[i].expiry) {
        evict(i); p[i].pinned = false; expiries++;
        log("unpin", i, ",\"why\":\"expiry\"");
      }
    // (a2) KV growth of the running requests (NEXT-2, R27/R28)
    if (growth()) grow_running();
    // (b) loaded requests join the batch
    for (int i = 0; i < P; ++i)
      if (p[i].st == READY) { set_state(i, RUNNING); p[i].prem = unc[i]; }
    // chunked prefill (R31/R32): the running requests take their share of the budget first
    int64_t left = budget() > 0 ? assign_running() : 1;
    // (c) admit loop (victims PAPER.md:645-655)
    int admitted = 0;
    for (;;) {
      int nq = 0, nb = 0;
      for (int i = 0; i < P; ++i) {
        nq += p[i].st == QUEUED;
        nb += p[i].st == RUNNING || p[i].st == LOADING || p[i].st == READY;
      }
      if (nq == 0 || nb >= eng[5]) break;
      if (budget() > 0 && left <= 0) break;  // R32: no token budget left this iteration
      int h = head();
      const int32_t* tr = turn_rec(h, p[h].turn);
      // R12: reserve the whole request; R27 (growth): up to the slot of the next token
      const int64_t upto = growth() ? p[h].emitted + 1 : tr[1];
      int64_t need = ceil_div(p[h].ctx + tr[0] + upto, bs) - p[h].gblk;
      if (need > free_blk && (admitted == 0 || (pol[3] & FLAG_VICTIMS_ANY))) {
        while (need > free_blk) {
          int v = -1;
          for (int i = P - 1; i >= 0; --i) if (p[i].pinned && i != h) { v = i; break; }
          if (v < 0) break;
          evict(v); p[v].pinned = false; victims++;
          if (audit) {
            char x[48];
            snprintf(x, sizeof x, ",\"why\":\"victim\",\"for\":%d", h);
            log("unpin", v, x);
          }
        }
      }
      if (need > free_blk) break;  // HOL break
      free_blk -= need;
      p[h].gblk += need;
      bubble += now - p[h].req_arr;
      p[h].bubble += now - p[h].req_arr;
      int64_t cached;
      bool loading = false;
      if (p[h].pinned) {
        cached = p[h].ctx; p[h].pinned = false; hits++;
        log("unpin", h, ",\"why\":\"hit\"");
      } else if (dram_on() && p[h].dblk > 0 && p[h].dblk == ceil_div(p[h].ctx, bs)) {
        cached = p[h].ctx; loading = true;
        int64_t start = now > chan_free ? now : chan_free;
        p[h].load_done = start + ceil_div((i128)p[h].dblk * eng[3], 1000000);
        chan_free = p[h].load_done;
        reloads++;
      } else {
        cached = 0;
      }
      // recomputed: the context without a cached copy, plus (R30) the prompt and emitted
      // tokens a preemption dropped
      recompute += p[h].ctx - cached + (p[h].preempted ? tr[0] + p[h].emitted : 0);
      p[h].preempted = false;
      int64_t uncached = p[h].ctx + tr[0] + p[h].emitted - cached;
      prefill += uncached;
      if (audit) {
        char x[96];
        snprintf(x, sizeof x, ",\"cached\":%lld,\"uncached\":%lld,\"load\":%d",
                 (long long)cached, (long long)uncached, loading ? 1 : 0);
        log("admit", h, x);
      }
      unc[h] = uncached;
      if (loading) {
        set_state(h, LOADING);
      } else {
        set_state(h, RUNNING);
        p[h].prem = uncached;
        if (budget() > 0) {  // R32: a new request takes what is left (a decode takes one token)
          p[h].chunk = std::min(uncached, left);
          left -= uncached > 0 ? p[h].chunk : 1;
        }
      }
      admitted++;
    }
    // (d) unschedulable: nothing can ever free memory for the head
    int nq = 0, nb = 0;
    for (int i = 0; i < P; ++i) {
      nq += p[i].st == QUEUED;
      nb += p[i].st == RUNNING || p[i].st == LOADING || p[i].st == READY;
    }
    if (nq > 0 && admitted == 0 && nb == 0) {
      int h = head();
      bool other_pin = false;
      for (int i = 0; i < P; ++i) if (p[i].pinned && i != h) other_pin = true;
      if (!other_pin) { status = ST_UNSCHED; return false; }
    }
    // (e) start the next iteration
    int nrun = 0;
    for (int i = 0; i < P; ++i) nrun += p[i].st == RUNNING;
    if (nrun > 0) {
      if (iterations >= eng[7]) { status = ST_BUDGET; return false; }
      i128 pf = 0, kvsum = 0;
      for (int i = 0; i < P; ++i) {
        if (p[i].st != RUNNING) continue;
        kvsum += p[i].gblk;
        // R16: without a budget the whole prefill runs in the request's first iteration;
        // R31: with one, this iteration's chunk.  The iteration that completes the prefill (or
        // any iteration of a decoding request) emits one token.
        const int64_t c = budget() > 0 ? p[i].chunk : p[i].prem;
        p[i].emit = p[i].prem == 0 || c == p[i].prem;
        pf += c;
        p[i].prem -= c;
        p[i].chunk = 0;
      }
      i128 ps = (i128)eng[0] + (i128)eng[1] * pf + (i128)eng[2] * bs * kvsum;
      int64_t dur = ceil_div(ps, 1000000);
      iter_end = now + dur;
      in_flight = true;
      iterations++;
      busy += dur;
      for (int i = 0; i < P; ++i)
        if (p[i].st == RUNNING) p[i].service += dur;  // PLAS attained service
    }
    return true;
  }

  std::vector<int64_t> unc;  // uncached tokens of the current request, set at admission

  bool check_invariants() {
    int64_t g = free_blk, d = dram_free;
    for (int i = 0; i < P; ++i) { g += p[i].gblk; d += p[i].dblk; }
    if (g != kv) return false;
    if (dram_on() && d != eng[6]) return false;
    if (free_blk < 0 || dram_free < 0) return false;
    for (int i = 0; i < P; ++i) {
      if (p[i].pinned && !(p[i].st == TOOL || p[i].st == QUEUED)) return false;
      if (p[i].st == TOOL && !p[i].pinned && p[i].gblk != 0) return false;
    }
    return true;
  }

  void run(int64_t* summary, int64_t* jct, int64_t* bub) {
    p.assign(P, Prog());
    unc.assign(P, 0);
    tool.assign(F, Row());
    free_blk = kv;
    dram_free = dram_on() ? eng[6] : 0;
    for (int i = 0; i < P; ++i) p[i].arrival = arrival_time(i);
    int64_t last_now = 0;
    for (;;) {
      // next event (R1, R3): pin expiry (eager), tool return, load done, arrival, iteration end
      int64_t t = INF;
      for (int i = 0; i < P; ++i) {
        if (p[i].st == TOOL) {
          t = std::min(t, p[i].t_ret);
          if (p[i].pinned && eager() && p[i].expiry != INF) t = std::min(t, p[i].expiry + 1);
        }
        if (p[i].st == LOADING) t = std::min(t, p[i].load_done);
      }
      if (next_arr < P) t = std::min(t, p[next_arr].arrival);
      if (in_flight) t = std::min(t, iter_end);
      if (t == INF) break;
      now = t;
      if (now < last_now) { status = ST_INVARIANT; break; }
      last_now = now;
      // PinExpiry: first instant with now > expiry, program not in Q
      if (eager())
        for (int i = 0; i < P; ++i)
          if (p[i].st == TOOL && p[i].pinned && p[i].expiry != INF && p[i].expiry + 1 == now) {
            evict(i); p[i].pinned = false; expiries++;
            log("unpin", i, ",\"why\":\"expiry\"");
          }
      // ToolReturn = OnRequestArrive of a seen program
      for (int i = 0; i < P; ++i)
        if (p[i].st == TOOL && p[i].t_ret == now) {
          const int32_t* tr = turn_rec(i, p[i].turn);
          record(tr[2], tr[3]);  // Δ_obs = now - t_finish = dur_us
          p[i].turn += 1;
          set_state(i, QUEUED);
          p[i].req_arr = now;
          p[i].emitted = 0;
        }
      // LoadDone
      for (int i = 0; i < P; ++i)
        if (p[i].st == LOADING && p[i].load_done == now) set_state(i, READY);
      // ProgramArrival
      while (next_arr < P && p[next_arr].arrival == now) {
        Prog& q = p[next_arr];
        q.since = now;  // the program's lifetime starts at its arrival
        set_state(next_arr, QUEUED);
        q.turn = 0; q.ctx = 0; q.req_arr = now;
        next_arr++;
      }
      // IterationEnd: every batch member emits one token; finishes in index order
      if (in_flight && iter_end == now) {
        in_flight = false;
        for (int i = 0; i < P; ++i)
          if (p[i].st == RUNNING && p[i].emit) {
            p[i].emitted += 1;
            if (p[i].emitted == turn_rec(i, p[i].turn)[1]) finish(i);
          }
      }
      if (!check_invariants()) { status = ST_INVARIANT; break; }
      if (in_flight) continue;  // mid-iteration: no scheduling point (R2)
      if (!schedule()) break;
      if (!check_invariants()) { status = ST_INVARIANT; break; }
    }
    if (status == ST_OK && D != P) status = ST_UNSCHED;
    if (status == ST_OK && pins_created != hits + expiries + victims) status = ST_INVARIANT;
    // JCT = sum of bubbles + in-engine time + tool time + load stalls, per program.
    // Bubbles come from the req_arr bookkeeping of the admit loop, tool time from the trace,
    // engine and load time from the state clock; the queue-state clock must equal the bubbles.
    for (int i = 0; status == ST_OK && i < P; ++i) {
      const Prog& q = p[i];
      const int64_t engine = q.in_state[RUNNING], load = q.in_state[LOADING] + q.in_state[READY];
      if (q.completion - q.arrival != q.bubble + engine + q.tool_us + load ||
          q.in_state[QUEUED] != q.bubble || q.in_state[TOOL] != q.tool_us)
        status = ST_INVARIANT;
    }
    std::memset(summary, 0, 16 * 8);
    if (status != ST_OK) {
      summary[0] = (int64_t)(uint32_t)status;
      if (jct) for (int i = 0; i < P; ++i) jct[i] = -1;
      if (bub) for (int i = 0; i < P; ++i) bub[i] = -1;
      return;
    }
    std::vector<int64_t> js(P);
    int64_t sum = 0, mx = 0, min_arr = INF, max_comp = 0;
    for (int i = 0; i < P; ++i) {
      js[i] = p[i].completion - p[i].arrival;
      sum += js[i];
      mx = std::max(mx, js[i]);
      min_arr = std::min(min_arr, p[i].arrival);
      max_comp = std::max(max_comp, p[i].completion);
      if (jct) jct[i] = js[i];
      if (bub) bub[i] = p[i].bubble;
    }
    std::vector<int64_t> s = js;
    std::sort(s.begin(), s.end());
    int64_t r50 = (50 * (int64_t)P + 99) / 100, r99 = (99 * (int64_t)P + 99) / 100;  // nearest rank (R20)
    summary[0] = ((int64_t)D << 32) | (uint32_t)status;
    summary[1] = turns_done;
    summary[2] = sum;
    summary[3] = mx;
    summary[4] = s[r50 - 1];
    summary[5] = s[r99 - 1];
    summary[6] = bubble;
    summary[7] = max_comp - min_arr;
    summary[8] = iterations;
    summary[9] = busy;
    summary[10] = prefill;
    summary[11] = recompute;
    summary[12] = hits;
    summary[13] = expiries;
    summary[14] = victims;
    summary[15] = reloads;
  }
};

}  // namespace

int or_simulate(const void* progs, const int32_t* turns, int64_t n_turns, int S, int P, int F,
                const int64_t* gap_us, int n_rate, const int64_t* kv_blocks, int n_kv,
                const int64_t* policies, int n_pol, const int64_t* est, const int64_t* eng,
                const int64_t* fitted, int J, int64_t r_begin, int64_t r_end, int n_threads,
                int64_t* summary, int64_t* jct, int64_t* bubble) {
  (void)n_turns;
  if (P < 1 || S < 1 || n_rate < 1 || n_kv < 1 || n_pol < 1 || r_begin < 0 || r_end < r_begin)
    return -1;
  if (r_end > (int64_t)S * n_rate * n_kv * n_pol) return -1;
  if (eng[0] < 1 || eng[4] < 1 || eng[5] < 1) return -1;
  // chunked prefill needs room for every decode (budget >= max_batch), reservation mode only
  if (eng[8] < 0 || eng[8] > 1 || eng[9] < 0) return -1;
  if (eng[9] > 0 && (eng[9] < eng[5] || eng[8] != 0)) return -1;
  auto one = [&](int64_t r) {
    int64_t pol_i = r % n_pol, kv_i = (r / n_pol) % n_kv, rate_i = (r / ((int64_t)n_pol * n_kv)) % n_rate;
    int64_t seed = r / ((int64_t)n_pol * n_kv * n_rate);
    Sim sim;
    sim.progs = (const uint8_t*)progs;
    sim.turns = turns;
    sim.P = P; sim.F = F; sim.J = J;
    sim.gap = gap_us[rate_i]; sim.kv = kv_blocks[kv_i];
    sim.pol = policies + 8 * pol_i;
    sim.est = est; sim.eng = eng; sim.fitted = fitted;
    sim.seed = (int)seed;
    int64_t k = r - r_begin;
    sim.run(summary + 16 * k, jct ? jct + (int64_t)P * k : nullptr,
            bubble ? bubble + (int64_t)P * k : nullptr);
  };
  int64_t n = r_end - r_begin;
  if (n_threads <= 1 || n < 2) {
    for (int64_t r = r_begin; r < r_end; ++r) one(r);
  } else {
    std::vector<std::thread> th;
    for (int t = 0; t < n_threads; ++t)
      th.emplace_back([&, t]() {
        for (int64_t r = r_begin + t; r < r_end; r += n_threads) one(r);
      });
    for (auto& x : th) x.join();
  }
  return 0;
}

int or_simulate_audit(const void* progs, const int32_t* turns, int64_t n_turns, int S, int P, int F,
                      const int64_t* gap_us, int n_rate, const int64_t* kv_blocks, int n_kv,
                      const int64_t* policies, int n_pol, const int64_t* est, const int64_t* eng,
                      const int64_t* fitted, int J, int64_t replica, char* buf, int64_t cap,
                      int64_t* len, int64_t* summary) {
  (void)n_turns;
  if (P < 1 || S < 1 || replica < 0 || replica >= (int64_t)S * n_rate * n_kv * n_pol) return -1;
  const int64_t r = replica;
  const int64_t pol_i = r % n_pol, kv_i = (r / n_pol) % n_kv, rate_i = (r / ((int64_t)n_pol * n_kv)) % n_rate;
  Sim sim;
  sim.progs = (const uint8_t*)progs;
  sim.turns = turns;
  sim.P = P; sim.F = F; sim.J = J;
  sim.gap = gap_us[rate_i]; sim.kv = kv_blocks[kv_i];
  sim.pol = policies + 8 * pol_i;
  sim.est = est; sim.eng = eng; sim.fitted = fitted;
  sim.seed = (int)(r / ((int64_t)n_pol * n_kv * n_rate));
  std::string log;
  sim.audit = &log;
  sim.run(summary, nullptr, nullptr);
  *len = (int64_t)log.size();
  if (buf && cap > 0) std::memcpy(buf, log.data(), (size_t)std::min<int64_t>(cap, *len));
  return *len <= cap ? 0 : 1;  // 1: buffer too small (len holds the size needed)
}

int or_jct_stats(const int64_t* summary, int64_t n_replicas, int n_cells, int64_t* out) {
  if (n_cells < 1 || n_replicas % n_cells) return -1;
  std::memset(out, 0, (size_t)n_cells * 8 * 8);
  for (int64_t r = 0; r < n_replicas; ++r) {
    const int64_t* s = summary + 16 * r;
    int64_t* o = out + 8 * (r % n_cells);
    int status = (int)(uint32_t)(s[0] & 0xffffffff);
    if (status != 0) { o[1] += 1; continue; }
    o[0] += 1;
    o[2] += s[0] >> 32;
    o[3] += s[1];
    o[4] += s[2];
    o[5] = std::max(o[5], s[3]);
    o[6] += s[6];
    o[7] += s[7];
  }
  return 0;
}
