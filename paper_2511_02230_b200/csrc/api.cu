// api.cu — libcontinuum host runtime: the C ABI of include/continuum.h.
// Validation, launch planning (occupancy-sized persistent grids), scratch ownership and the
// host-buffer end-to-end path.  No compute happens here: every step of the hot path runs in
// the kernels of replay.cu, ttl_fit.cu and jct_stats.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "ct_internal.h"

struct ct_ctx {
  int device = 0;
  int sm_count = 0;
  unsigned long long* counter = nullptr;
  void* axes = nullptr;
  size_t axes_cap = 0;
  void* fitbuf[2] = {nullptr, nullptr};  // double-buffered fit accumulator (ct_fit_ttl)
  size_t fitbuf_cap[2] = {0, 0};
  int64_t fit_clean[2] = {0, 0};  // leading words known to be zero
  int fit_cur = 0;
  void* h_progs = nullptr;
  size_t h_progs_cap = 0;
  void* h_turns = nullptr;
  size_t h_turns_cap = 0;
  void* h_out = nullptr;
  size_t h_out_cap = 0;
  void* h_jct = nullptr;
  size_t h_jct_cap = 0;
  void* fb = nullptr;  // MODE 4 fallback replica list
  size_t fb_cap = 0;
  void* syn = nullptr;  // synthesis: tables | cdf | class | per-program class | seed totals | blocks
  size_t syn_cap = 0;
  ct_launch_info last{};
  int fit_occ = 0, fit_occ_key = -1;
  bool timing = false;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};  // replay start/end, fit start/end
  bool replay_timed = false, fit_timed = false;
};

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  return fail(CT_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

#define CT_CUDA(call)                                        \
  do {                                                       \
    cudaError_t _e = (call);                                 \
    if (_e != cudaSuccess) return cuda_fail(_e, #call);      \
  } while (0)

int ensure(void** p, size_t* cap, size_t need) {
  if (*cap >= need && *p) return CT_OK;
  if (*p) cudaFree(*p);
  *p = nullptr;
  *cap = 0;
  size_t n = std::max<size_t>(need, 256);
  cudaError_t e = cudaMalloc(p, n);
  if (e != cudaSuccess) return fail(CT_ENOMEM, "cudaMalloc(%zu): %s", n, cudaGetErrorString(e));
  *cap = n;
  return CT_OK;
}

// Estimator bounds: T_default^2 < 2^80 and (D a_den + a_num turns_done) < 2^45 (D <= 256,
// turns_done <= 256 CT_MAX_TURNS = 2^24) keep CalcTTL's numerator below 2^125.
bool est_valid(const ct_estimator_params& e) {
  return e.lq > 0 && e.b_us > 0 && e.t_default_us > 0 && e.n_min >= 1 && e.a_num >= 0 &&
         e.a_den >= 1 && e.ttl_max_us >= 0 && e.b_us < (1ll << 40) &&
         e.t_default_us < (1ll << 40) && e.lq < (1ull << 40) && e.a_num < (1ll << 20) &&
         e.a_den < (1ll << 20) && e.ttl_max_us < CT_TTL_SAT && e.n_min < (1ll << 40);
}

// Largest arr_q with arr_q * gap < 2^62 for every gap of the sweep (arrivals < 2^42 µs).
int64_t arr_q_max(const ct_sweep* sw) {
  int64_t g = 0;
  for (int i = 0; i < sw->n_rates; ++i) g = std::max<int64_t>(g, sw->gap_us[i]);
  return g == 0 ? INT64_MAX : (int64_t)(((1ll << 62) - 1) / g);
}

const char* check_reason(uint32_t bits) {
  if (bits & CT_CHECK_NTURNS) return "nturns outside [1, CT_MAX_TURNS]";
  if (bits & CT_CHECK_TURN_RANGE) return "turn0 / nturns outside the turn array";
  if (bits & CT_CHECK_ARRIVAL) return "arr_q negative, arr_q * gap >= 2^62, or arrivals not sorted";
  if (bits & CT_CHECK_TOKENS) return "decode_tokens < 1 or new_tokens < 0";
  if (bits & CT_CHECK_TOOL) return "non-final turn with tool outside [0, n_tools) or dur_us < 1";
  if (bits & CT_CHECK_CONTEXT) return "total new + decode tokens of a program > CT_MAX_CONTEXT";
  if (bits & CT_CHECK_FITTED) return "FITTED table entry outside [0, CT_TTL_SAT)";
  return "invalid trace set";
}

typedef __int128 i128;

}  // namespace

void ct::set_last_error(const char* msg) { g_err = msg; }

extern "C" {

int ct_version(void) { return CT_ABI_VERSION; }
const char* ct_last_error(void) { return g_err.c_str(); }

int ct_ctx_create(int device, ct_ctx** out) {
  if (!out) return fail(CT_EINVAL, "out is NULL");
  *out = nullptr;
  cudaDeviceProp prop;
  cudaError_t e = cudaGetDeviceProperties(&prop, device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceProperties");
  if (prop.major != 10 || prop.minor != 0)
    return fail(CT_EUNSUPPORTED, "device %d is sm_%d%d; libcontinuum is built for sm_100a", device,
                prop.major, prop.minor);
  CT_CUDA(cudaSetDevice(device));
  ct_ctx* c = new ct_ctx();
  c->device = device;
  c->sm_count = prop.multiProcessorCount;
  e = cudaMalloc((void**)&c->counter, 64);
  if (e != cudaSuccess) {
    delete c;
    return fail(CT_ENOMEM, "cudaMalloc counter: %s", cudaGetErrorString(e));
  }
  *out = c;
  return CT_OK;
}

int ct_ctx_destroy(ct_ctx* c) {
  if (!c) return CT_OK;
  void* ps[] = {c->counter, c->axes, c->fitbuf[0], c->fitbuf[1], c->h_progs, c->h_turns, c->h_out, c->h_jct, c->syn,
                c->fb};
  for (void* p : ps)
    if (p) cudaFree(p);
  for (auto e : c->ev)
    if (e) cudaEventDestroy(e);
  delete c;
  return CT_OK;
}

int ct_ctx_set_timing(ct_ctx* c, int enable) {
  if (!c) return fail(CT_EINVAL, "NULL argument");
  if (enable && !c->ev[0])
    for (auto& e : c->ev) CT_CUDA(cudaEventCreate(&e));
  c->timing = enable != 0;
  return CT_OK;
}

int ct_last_launch(ct_ctx* c, ct_launch_info* info) {
  if (!c || !info) return fail(CT_EINVAL, "NULL argument");
  c->last.replay_ms = -1.f;
  c->last.fit_hist_ms = -1.f;
  if (c->replay_timed) {
    CT_CUDA(cudaEventSynchronize(c->ev[1]));
    CT_CUDA(cudaEventElapsedTime(&c->last.replay_ms, c->ev[0], c->ev[1]));
  }
  if (c->fit_timed) {
    CT_CUDA(cudaEventSynchronize(c->ev[3]));
    CT_CUDA(cudaEventElapsedTime(&c->last.fit_hist_ms, c->ev[2], c->ev[3]));
  }
  *info = c->last;
  return CT_OK;
}

// ---------------------------------------------------------------------------------------------
int ct_simulate_batch(ct_ctx* c, const ct_trace_set* tr, const ct_sweep* sw,
                      const ct_engine_params* eng, int64_t rb, int64_t re,
                      ct_replica_summary* out, int64_t* jct, void* stream) {
  const ct_replay_outputs o = {out, jct, nullptr};
  return ct_simulate_batch_ex(c, tr, sw, eng, rb, re, &o, stream);
}

int ct_simulate_batch_ex(ct_ctx* c, const ct_trace_set* tr, const ct_sweep* sw,
                         const ct_engine_params* eng, int64_t rb, int64_t re,
                         const ct_replay_outputs* outs, void* stream) {
  if (!c || !tr || !sw || !eng || !outs) return fail(CT_EINVAL, "NULL argument");
  ct_replica_summary* out = outs->summary;
  int64_t* jct = outs->jct_us;
  const int P = tr->n_programs, F = tr->n_tools;
  if (P < 1 || P > CT_MAX_PROGRAMS) return fail(CT_EINVAL, "n_programs %d not in [1, %d]", P, CT_MAX_PROGRAMS);
  if (F < 1 || F > CT_MAX_TOOLS) return fail(CT_EINVAL, "n_tools %d not in [1, %d]", F, CT_MAX_TOOLS);
  if (!tr->programs || !tr->turns || tr->n_turns < 1) return fail(CT_EINVAL, "empty trace set");
  if (sw->n_seeds < 1 || sw->n_rates < 1 || sw->n_kv < 1 || sw->n_policies < 1)
    return fail(CT_EINVAL, "sweep axes must be non-empty");
  if (sw->n_seeds > tr->n_seeds) return fail(CT_EINVAL, "sweep has more seeds than the trace set");
  if (!sw->gap_us || !sw->kv_blocks || !sw->policies) return fail(CT_EINVAL, "NULL sweep axis");
  const int64_t R = (int64_t)sw->n_seeds * sw->n_rates * sw->n_kv * sw->n_policies;
  if (rb < 0 || re < rb || re > R) return fail(CT_EINVAL, "replica range [%lld, %lld) outside [0, %lld)",
                                               (long long)rb, (long long)re, (long long)R);
  const ct_engine_params& E = *eng;
  if (E.c0_ps < 1 || E.bs < 1 || E.max_batch < 1 || E.c_pf_ps < 0 || E.c_kv_ps < 0 ||
      E.c_h2d_ps < 0 || E.dram_blocks < 0 || E.max_iters < 0)
    return fail(CT_EINVAL, "invalid engine parameters (R16/R25)");
  if (E.c0_ps >= (1ll << 48) || E.c_pf_ps >= (1ll << 40) || E.c_kv_ps >= (1ll << 30) ||
      E.c_h2d_ps >= (1ll << 40) || E.bs >= (1 << 20) || E.dram_blocks >= (1ll << 30))
    return fail(CT_EINVAL, "engine constants exceed the int64 fixed-point bounds");
  {  // one iteration's ps: c0 + c_pf x prefill + c_kv x bs x resident blocks, where prefill and
     // resident tokens are both bounded by the pool (kv_max x bs); one DRAM load: blocks x c_h2d
    int64_t kvm = 0;
    for (int i = 0; i < sw->n_kv; ++i) kvm = std::max<int64_t>(kvm, sw->kv_blocks[i]);
    const i128 it = (i128)E.c0_ps + ((i128)E.c_pf_ps + E.c_kv_ps) * E.bs * kvm;
    if (it >= ((i128)1 << 62))
      return fail(CT_EINVAL, "c0 + (c_pf + c_kv) bs max(kv_blocks) >= 2^62 ps (iteration cost overflow)");
    if ((i128)E.dram_blocks * E.c_h2d_ps >= ((i128)1 << 62))
      return fail(CT_EINVAL, "dram_blocks x c_h2d >= 2^62 ps (load time overflow)");
  }
  if (E.kv_growth != 0 && E.kv_growth != 1) return fail(CT_EINVAL, "kv_growth must be 0 or 1");
  if (E.prefill_chunk < 0 || (E.prefill_chunk > 0 && E.prefill_chunk < E.max_batch))
    return fail(CT_EINVAL, "prefill_chunk must be 0 (off) or >= max_batch (R31)");
  if (E.prefill_chunk > 0 && E.kv_growth != 0)
    return fail(CT_EINVAL, "chunked prefill is modelled with reservation (kv_growth = 0) only");
  bool need_est = false, need_fit = false, need_h2d = false;
  for (int i = 0; i < sw->n_policies; ++i) {
    const ct_policy& p = sw->policies[i];
    if (p.priority < CT_PRIO_PROG_FCFS || p.priority > CT_PRIO_PLAS)
      return fail(CT_EINVAL, "policy %d: priority %d", i, p.priority);
    if (p.pause < CT_PAUSE_EVICT || p.pause > CT_PAUSE_INFERCEPT)
      return fail(CT_EINVAL, "policy %d: pause %d", i, p.pause);
    if (p.flags & ~(CT_FLAG_VICTIMS_ANY | CT_FLAG_STEP_EXPIRY))
      return fail(CT_EINVAL, "policy %d: unknown flags", i);
    if (p.t_pin_us < 0 || p.t_pin_us >= CT_TTL_SAT) return fail(CT_EINVAL, "policy %d: t_pin", i);
    need_est |= p.pause == CT_PAUSE_PAPER || p.pause == CT_PAUSE_INFERCEPT ||
                (p.pause == CT_PAUSE_FIXED && p.t_thresh_us != CT_ALWAYS);
    need_fit |= p.pause == CT_PAUSE_FITTED;
    need_h2d |= p.dram != 0 && E.dram_blocks > 0;
  }
  if (need_est && !est_valid(sw->est)) return fail(CT_EINVAL, "invalid estimator parameters");
  if (need_fit && (!sw->fitted_ttl || sw->fitted_j < 1 || sw->fitted_j > CT_MAX_J ||
                   sw->fitted_rows < F))
    return fail(CT_EINVAL, "FITTED policy needs fitted_ttl[fitted_rows >= n_tools][fitted_j]");
  if (need_h2d && E.c_h2d_ps < 1) return fail(CT_EINVAL, "DRAM tier needs c_h2d_ps >= 1 (R25)");
  for (int i = 0; i < sw->n_rates; ++i)
    if (sw->gap_us[i] < 0 || sw->gap_us[i] >= (1ll << 30)) return fail(CT_EINVAL, "gap_us[%d]", i);
  for (int i = 0; i < sw->n_kv; ++i)
    if (sw->kv_blocks[i] < 0 || sw->kv_blocks[i] >= (1ll << 30)) return fail(CT_EINVAL, "kv_blocks[%d]", i);
  if (re == rb) return CT_OK;
  if (!out) return fail(CT_EINVAL, "out is NULL");
  cudaStream_t s = (cudaStream_t)stream;

  // device copy of the sweep axes
  const size_t n_gap = sw->n_rates, n_kv = sw->n_kv, n_pol = sw->n_policies;
  // axes: gaps, KV budgets, policies, then the policy order of a split launch (TTL-grid class
  // first, ascending indices within each part)
  const size_t bytes = 8 * (n_gap + n_kv) + sizeof(ct_policy) * n_pol + 4 * n_pol;
  int rc = ensure(&c->axes, &c->axes_cap, bytes);
  if (rc) return rc;
  std::vector<unsigned char> hb(bytes);
  std::memcpy(hb.data(), sw->gap_us, 8 * n_gap);
  std::memcpy(hb.data() + 8 * n_gap, sw->kv_blocks, 8 * n_kv);
  std::memcpy(hb.data() + 8 * (n_gap + n_kv), sw->policies, sizeof(ct_policy) * n_pol);
  {
    int* order = (int*)(hb.data() + 8 * (n_gap + n_kv) + sizeof(ct_policy) * n_pol);
    int k = 0;
    for (size_t i = 0; i < n_pol; ++i)
      if (ct::fast_policy(sw->policies[i], E)) order[k++] = (int)i;
    for (size_t i = 0; i < n_pol; ++i)
      if (!ct::fast_policy(sw->policies[i], E)) order[k++] = (int)i;
  }
  CT_CUDA(cudaMemcpyAsync(c->axes, hb.data(), bytes, cudaMemcpyHostToDevice, s));
  // counter block: [0] replica counter, [1] fallback list count, [2] fallback counter,
  // [4..5] trace check result
  CT_CUDA(cudaMemsetAsync(c->counter, 0, 48, s));
  {
    ct::CheckArgs ck;
    const int64_t per_seed = (int64_t)sw->n_rates * sw->n_kv * sw->n_policies;
    ck.progs = tr->programs;
    ck.turns = (const int4*)tr->turns;
    ck.n_turns = tr->n_turns;
    ck.p_begin = rb / per_seed * P;
    ck.p_end = ((re - 1) / per_seed + 1) * P;
    ck.P = P;
    ck.F = F;
    ck.arr_max = arr_q_max(sw);
    ck.fitted = need_fit ? sw->fitted_ttl : nullptr;
    ck.n_fitted = need_fit ? (int64_t)F * sw->fitted_j : 0;
    ck.err = c->counter + 4;
    cudaError_t e = ct::launch_check_traces(ck, c->sm_count, s);
    if (e != cudaSuccess) return cuda_fail(e, "trace check launch");
  }

  ct::ReplayArgs a;
  a.progs = tr->programs;
  a.turns = (const int4*)tr->turns;
  a.P = P;
  a.F = F;
  a.gap = (const int64_t*)c->axes;
  a.kv = a.gap + n_gap;
  a.pols = (const ct_policy*)(a.kv + n_kv);
  a.n_rate = sw->n_rates;
  a.n_kv = sw->n_kv;
  a.n_pol = sw->n_policies;
  a.est = sw->est;
  a.fitted = sw->fitted_ttl;
  a.J = sw->fitted_j > 0 ? sw->fitted_j : 1;
  a.eng = E;
  a.r_begin = rb;
  a.r_end = re;
  a.out = out;
  a.jct = jct;
  a.bubble = outs->bubble_us;
  a.sel = nullptr;
  a.n_sel = 0;
  a.blk0 = 0;
  a.sel_total = 0;
  a.counter = c->counter;
  a.err = c->counter + 4;
  a.bs_magic = E.bs == 1 ? 0
                         : (uint64_t)(((((unsigned __int128)1) << 64) + (uint64_t)E.bs - 1) /
                                      (unsigned __int128)(uint64_t)E.bs);
  const int ns = (P + 31) / 32;  // slots per lane
  const bool growth = E.kv_growth != 0 || E.prefill_chunk > 0;  // the vLLM-engine kernels
  // the FAST kernels also need every no-prefill iteration below 2^31 µs (32-bit macro-steps)
  int64_t kv_max = 0;
  for (size_t i = 0; i < n_kv; ++i) kv_max = std::max<int64_t>(kv_max, sw->kv_blocks[i]);
  const i128 d_max = ((i128)E.c0_ps + (i128)E.c_kv_ps * E.bs * kv_max + 999999) / 1000000;
  a.d32 = d_max < ((i128)1 << 31) ? 1 : 0;
  {  // 32-bit iteration duration when c_kv bs max(kv) + 1e6 < 2^32 (replay.cu iter_us_kv32)
    const i128 u = (i128)E.c_kv_ps * E.bs;
    const i128 q = ((i128)E.c0_ps + 999999) / 1000000;
    a.kv32 = (u * kv_max + 1000000 < ((i128)1 << 32) && q < ((i128)1 << 31)) ? 1 : 0;
    a.kv_unit = a.kv32 ? (uint32_t)u : 0;
    a.c0q = a.kv32 ? (uint32_t)q : 0;
    a.c0r = a.kv32 ? (uint32_t)(q * 1000000 - E.c0_ps) : 0;
    a.pf_q = (uint32_t)(E.c_pf_ps / 1000000);  // c_pf < 2^40: pf_q < 2^20
    a.pf_r = (uint32_t)(E.c_pf_ps % 1000000);
    a.pf32 = a.pf_r == 0 ? 0x7fffffffu : (uint32_t)(((1ull << 32) - 1000001ull) / a.pf_r);
  }
  int n_fast = 0;
  if (a.d32)
    for (size_t i = 0; i < n_pol; ++i) n_fast += ct::fast_policy(sw->policies[i], E) ? 1 : 0;
  int n_prog = 0;
  for (size_t i = 0; i < n_pol; ++i) n_prog += ct::prog_policy(sw->policies[i], E) ? 1 : 0;
  // P <= 32 32-bit-time kernels need d < 2^31 µs (a.d32); see replay.cu MODE
  int n_simple32 = 0;
  if (a.d32)
    for (size_t i = 0; i < n_pol; ++i) n_simple32 += ct::simple_policy(sw->policies[i], E) ? 1 : 0;
  int n_ext32 = 0;
  if (a.d32)
    for (size_t i = 0; i < n_pol; ++i) n_ext32 += ct::ext_policy(sw->policies[i], E) ? 1 : 0;
  const int mode = growth    ? 0
                   : ns == 1 ? (n_fast == (int)n_pol       ? 1
                                : n_simple32 == (int)n_pol ? 3
                                : n_ext32 == (int)n_pol    ? 6
                                : n_simple32 > 0           ? 2
                                                           : 0)
                             : (n_prog == (int)n_pol ? 1 : 0);
  const int wpb = 4;
  a.from_list = 0;
  a.fb_list = nullptr;
  a.fb_count = c->counter + 1;
  // P > 32, program-FCFS class: the 32-bit kernel (MODE 4) first, then MODE 1 over the replicas
  // it handed back (horizon reached, or the bubble output requested)
  // (simple class: program or request FCFS; the fallback launch is MODE 1 when every policy is
  // in the program-FCFS class, else the generic kernel)
  const bool ns32 = ns > 1 && !growth && n_simple32 == (int)n_pol && !a.bubble;
  if (ns32) {
    rc = ensure(&c->fb, &c->fb_cap, 8 * (size_t)(re - rb));
    if (rc) return rc;
    a.fb_list = (int64_t*)c->fb;
  }
  const int mode1 = ns32 ? (mode == 1 ? 4 : 5) : mode;
  a.smem_per_warp = ns32 ? ct::replay_ns32_smem_per_warp(ns, F)
                         : ct::replay_smem_per_warp(ns, F, growth, mode);
  const int smem = a.smem_per_warp * wpb;
  int occ = ct::replay_occupancy(ns, growth, mode1, wpb, smem);
  if (occ < 1) return fail(CT_ECUDA, "replay kernel cannot be resident (smem %d)", smem);
  const int64_t need_blocks = (re - rb + wpb - 1) / wpb;
  const int grid = (int)std::min<int64_t>((int64_t)c->sm_count * occ, need_blocks);
  // P <= 32 sweeps that mix TTL-grid policies with other 32-bit classes: two launches over
  // policy subsets (ReplayArgs.sel), the TTL-grid kernel (MODE 1, no estimator, 10 CTAs/SM)
  // for the replicas of those policies and the estimator / extended kernel for the rest
  const int64_t nblk = (re - 1) / (int64_t)n_pol - rb / (int64_t)n_pol + 1;
  const bool split = ns == 1 && !growth && !a.bubble && n_fast > 0 && n_fast < (int)n_pol &&
                     (mode == 2 || mode == 3 || mode == 6) && nblk * (int64_t)n_pol < (1ll << 31);
  a.blk0 = rb / (int64_t)n_pol;
  if (c->timing) CT_CUDA(cudaEventRecord(c->ev[0], s));
  cudaError_t e;
  if (split) {
    const int* order = (const int*)(a.pols + n_pol);
    ct::ReplayArgs g = a;
    g.sel = order;
    g.n_sel = n_fast;
    g.sel_total = nblk * n_fast;
    const int occg = ct::replay_occupancy(1, false, 1, wpb, smem);
    if (occg < 1) return fail(CT_ECUDA, "replay kernel cannot be resident (smem %d)", smem);
    const int gridg = (int)std::min<int64_t>((int64_t)c->sm_count * occg, (nblk * n_fast + wpb - 1) / wpb);
    e = ct::launch_replay(g, 1, false, 1, wpb, gridg, s);
    if (e != cudaSuccess) return cuda_fail(e, "replay launch (TTL-grid part)");
    a.sel = order + n_fast;
    a.n_sel = (int)n_pol - n_fast;
    a.sel_total = nblk * a.n_sel;
    a.counter = c->counter + 3;
    const int grido = (int)std::min<int64_t>((int64_t)c->sm_count * occ,
                                             (nblk * a.n_sel + wpb - 1) / wpb);
    e = ct::launch_replay(a, 1, false, mode1, wpb, grido, s);
    if (e != cudaSuccess) return cuda_fail(e, "replay launch");
  } else {
    e = ct::launch_replay(a, ns, growth, mode1, wpb, grid, s);
    if (e != cudaSuccess) return cuda_fail(e, "replay launch");
  }
  if (ns32) {
    ct::ReplayArgs b = a;
    b.from_list = 1;
    b.counter = c->counter + 2;
    b.smem_per_warp = ct::replay_smem_per_warp(ns, F, growth, mode);
    const int smem2 = b.smem_per_warp * wpb;
    const int occ2 = ct::replay_occupancy(ns, growth, mode, wpb, smem2);
    if (occ2 < 1) return fail(CT_ECUDA, "replay kernel cannot be resident (smem %d)", smem2);
    const int grid2 = (int)std::min<int64_t>((int64_t)c->sm_count * occ2, need_blocks);
    e = ct::launch_replay(b, ns, growth, mode, wpb, grid2, s);
    if (e != cudaSuccess) return cuda_fail(e, "replay fallback launch");
  }
  if (c->timing) CT_CUDA(cudaEventRecord(c->ev[1], s));
  c->replay_timed = c->timing;
  c->last.grid = grid;
  c->last.block = 32 * wpb;
  c->last.warps_per_block = wpb;
  c->last.slots_per_lane = ns;
  c->last.smem_per_block = smem;
  c->last.launches = (ns32 || split ? 2 : 1) + 1;  // + the trace check
  c->last.kernel_mode = split ? 10 + mode1 : mode1;
  return CT_OK;
}

int ct_validate_trace_set(ct_ctx* c, const ct_trace_set* tr, const ct_sweep* sw,
                          int64_t rb, int64_t re, void* stream) {
  if (!c || !tr || !sw) return fail(CT_EINVAL, "NULL argument");
  const int P = tr->n_programs, F = tr->n_tools;
  if (P < 1 || P > CT_MAX_PROGRAMS || F < 1 || F > CT_MAX_TOOLS || !tr->programs || !tr->turns ||
      tr->n_turns < 1)
    return fail(CT_EINVAL, "invalid trace-set shape");
  if (sw->n_seeds < 1 || sw->n_rates < 1 || sw->n_kv < 1 || sw->n_policies < 1 || !sw->gap_us ||
      sw->n_seeds > tr->n_seeds)
    return fail(CT_EINVAL, "invalid sweep axes");
  const int64_t per_seed = (int64_t)sw->n_rates * sw->n_kv * sw->n_policies;
  const int64_t R = per_seed * sw->n_seeds;
  if (rb < 0 || re < rb || re > R) return fail(CT_EINVAL, "replica range");
  if (re == rb) return CT_OK;
  bool need_fit = false;
  for (int i = 0; sw->policies && i < sw->n_policies; ++i) need_fit |= sw->policies[i].pause == CT_PAUSE_FITTED;
  cudaStream_t s = (cudaStream_t)stream;
  CT_CUDA(cudaMemsetAsync(c->counter + 4, 0, 16, s));
  ct::CheckArgs ck;
  ck.progs = tr->programs;
  ck.turns = (const int4*)tr->turns;
  ck.n_turns = tr->n_turns;
  ck.p_begin = rb / per_seed * P;
  ck.p_end = ((re - 1) / per_seed + 1) * P;
  ck.P = P;
  ck.F = F;
  ck.arr_max = arr_q_max(sw);
  ck.fitted = need_fit ? sw->fitted_ttl : nullptr;
  if (need_fit && (!sw->fitted_ttl || sw->fitted_j < 1 || sw->fitted_j > CT_MAX_J || sw->fitted_rows < F))
    return fail(CT_EINVAL, "FITTED policy needs fitted_ttl[fitted_rows >= n_tools][fitted_j]");
  ck.n_fitted = need_fit ? (int64_t)F * sw->fitted_j : 0;
  ck.err = c->counter + 4;
  cudaError_t e = ct::launch_check_traces(ck, c->sm_count, s);
  if (e != cudaSuccess) return cuda_fail(e, "trace check launch");
  unsigned long long h[2];
  CT_CUDA(cudaMemcpyAsync(h, c->counter + 4, 16, cudaMemcpyDeviceToHost, s));
  CT_CUDA(cudaStreamSynchronize(s));
  if (h[0] == 0) return CT_OK;
  if (h[1] != 0)
    return fail(CT_EINVAL, "program %lld: %s", (long long)~h[1], check_reason((uint32_t)h[0]));
  return fail(CT_EINVAL, "%s", check_reason((uint32_t)h[0]));
}

int ct_simulate_batch_host(ct_ctx* c, const ct_trace_set* ht, const ct_sweep* sw,
                           const ct_engine_params* eng, int64_t rb, int64_t re,
                           ct_replica_summary* host_out, int64_t* host_jct, void* stream) {
  if (!c || !ht || !sw || !eng || !host_out) return fail(CT_EINVAL, "NULL argument");
  const int P = ht->n_programs, F = ht->n_tools;
  if (P < 1 || P > CT_MAX_PROGRAMS || F < 1 || F > CT_MAX_TOOLS || ht->n_seeds < 1 || ht->n_turns < 1)
    return fail(CT_EINVAL, "invalid trace-set shape");
  if (!sw || !sw->gap_us || sw->n_rates < 1) return fail(CT_EINVAL, "NULL sweep axis");
  const int64_t np = (int64_t)ht->n_seeds * P;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t R = re - rb;
  int rc;
  if ((rc = ensure(&c->h_progs, &c->h_progs_cap, 16 * np))) return rc;
  if ((rc = ensure(&c->h_turns, &c->h_turns_cap, 16 * ht->n_turns))) return rc;
  if ((rc = ensure(&c->h_out, &c->h_out_cap, sizeof(ct_replica_summary) * std::max<int64_t>(R, 1)))) return rc;
  if (host_jct && (rc = ensure(&c->h_jct, &c->h_jct_cap, 8 * std::max<int64_t>(R, 1) * P))) return rc;
  CT_CUDA(cudaMemcpyAsync(c->h_progs, ht->programs, 16 * np, cudaMemcpyHostToDevice, s));
  CT_CUDA(cudaMemcpyAsync(c->h_turns, ht->turns, 16 * ht->n_turns, cudaMemcpyHostToDevice, s));
  ct_trace_set dt = *ht;
  dt.programs = (const ct_program*)c->h_progs;
  dt.turns = (const ct_turn*)c->h_turns;
  // the records are checked where they now are (check_traces_kernel, synchronous): an invalid
  // trace set returns CT_EINVAL naming the first bad program, as on the host before, without a
  // single-threaded pass over every record on the host (≈ 40 ms for cfg2's 18.8 M turns)
  rc = ct_validate_trace_set(c, &dt, sw, rb, re, stream);
  if (rc) return rc;
  rc = ct_simulate_batch(c, &dt, sw, eng, rb, re, (ct_replica_summary*)c->h_out,
                         host_jct ? (int64_t*)c->h_jct : nullptr, stream);
  if (rc) return rc;
  CT_CUDA(cudaMemcpyAsync(host_out, c->h_out, sizeof(ct_replica_summary) * R, cudaMemcpyDeviceToHost, s));
  if (host_jct) CT_CUDA(cudaMemcpyAsync(host_jct, c->h_jct, 8 * R * P, cudaMemcpyDeviceToHost, s));
  CT_CUDA(cudaStreamSynchronize(s));
  return CT_OK;
}

// ---------------------------------------------------------------------------------------------
namespace {

// Validation and launch arguments shared by the fit calls.  Fills fa (except acc/zero) and sa
// (except acc and the outputs).
int fit_prepare(ct_ctx* c, const ct_samples* sm, const ct_cost_params* cp,
                const ct_estimator_params* est, int rank, int world, ct::FitArgs& fa,
                ct::ScanArgs& sa, ct::FitPlan& plan) {
  if (!c || !sm || !cp || !est) return fail(CT_EINVAL, "NULL argument");
  const int F = sm->n_tools, K = cp->K, J = cp->J;
  if (F < 1 || F > CT_MAX_TOOLS) return fail(CT_EINVAL, "n_tools %d", F);
  if (K < 1 || K > CT_MAX_K || J < 1 || J > CT_MAX_J) return fail(CT_EINVAL, "K %d / J %d", K, J);
  if (world < 1 || rank < 0 || rank >= world) return fail(CT_EINVAL, "rank %d of %d", rank, world);
  const bool pairs = sm->tool_off == nullptr;
  if (sm->n < 0) return fail(CT_EINVAL, "n < 0");
  if (sm->n > 0 && !sm->dur_us) return fail(CT_EINVAL, "dur_us is NULL");
  if (pairs) {
    if (sm->n > 0 && !sm->tool_u8) return fail(CT_EINVAL, "unsorted layout needs tool_u8");
    if (world != 1) return fail(CT_EINVAL, "the unsorted layout is fitted on one rank");
    if (((uintptr_t)sm->dur_us & 15) || ((uintptr_t)sm->tool_u8 & 3))
      return fail(CT_EINVAL, "unsorted layout: dur_us must be 16-B and tool_u8 4-B aligned");
  } else {
    if (sm->tool_off[0] != 0 || sm->tool_off[F] != sm->n)
      return fail(CT_EINVAL, "tool_off must run from 0 to n");
    for (int f = 0; f < F; ++f)
      if (sm->tool_off[f + 1] < sm->tool_off[f]) return fail(CT_EINVAL, "tool_off not monotone");
    if (sm->n > 0 && ((uintptr_t)sm->dur_us & 15)) return fail(CT_EINVAL, "dur_us must be 16-B aligned");
  }
  if (!est_valid(*est)) return fail(CT_EINVAL, "invalid estimator parameters");
  if (cp->grid_step_us < 1 || cp->bs < 1 || cp->a_den < 1 || cp->a_num < 0 || cp->c_pf_ps < 0 ||
      cp->c_pin_ps < 0 || cp->avg_turns_num < 0 || cp->avg_turns_den < 0 ||
      cp->a_den >= (1ll << 32) || cp->a_num >= (1ll << 32) || cp->c_pf_ps >= (1ll << 40) ||
      cp->c_pin_ps >= (1ll << 40) || cp->bs >= (1ll << 20) || cp->avg_turns_num >= (1ll << 40) ||
      cp->avg_turns_den >= (1ll << 31))
    return fail(CT_EINVAL, "invalid cost parameters");
  if (cp->grid_step_us >= (1ll << 31) || est->b_us >= (1ll << 31))
    return fail(CT_EINVAL, "grid_step_us and b_us must be < 2^31");
  const i128 tau_max = (i128)(K - 1) * cp->grid_step_us;
  if (tau_max >= ((i128)1 << 43)) return fail(CT_EINVAL, "grid too long: (K-1)*step >= 2^43");
  const i128 n = sm->n;
  if (n >= ((i128)1 << 32)) return fail(CT_EINVAL, "too many samples (n >= 2^32)");
  // 128-bit headroom of n U(k) (extension C-4): V cnt and C (sum + tau (n - cnt)), sum < n 2^31
  for (int j = 0; j < J; ++j) {
    if (cp->ctx_tokens[j] < 0 || cp->ctx_tokens[j] >= (1ll << 32) || cp->turn_weight[j] < 0 ||
        cp->turn_weight[j] >= (1ll << 32))
      return fail(CT_EINVAL, "ctx_tokens / turn_weight[%d] out of range", j);
    const i128 V = ((i128)cp->c_pf_ps * cp->ctx_tokens[j] *
                    ((i128)cp->a_den + (i128)cp->a_num * cp->turn_weight[j])) / cp->a_den;
    const i128 C = (i128)cp->c_pin_ps * ((cp->ctx_tokens[j] + cp->bs - 1) / cp->bs);
    const i128 lim = (i128)1 << 125;
    if (V > lim / (n + 1) || C > lim / ((n + 1) * (((i128)1 << 31) + tau_max + 1)))
      return fail(CT_EINVAL, "cost products could overflow 128-bit arithmetic");
  }
  if (n * (i128)est->b_us * est->b_us >= ((i128)1 << 95))
    return fail(CT_EINVAL, "n * b^2 >= 2^95: sum of squares could overflow");
  plan = ct::fit_plan(K, F, pairs);
  if (!plan.ok)
    return fail(CT_EINVAL, pairs ? "unsorted layout: F x (K+1) bins exceed shared memory (use CSR)"
                                 : "K too large for the histogram pass");
  std::memset(&fa, 0, sizeof fa);
  fa.dur = sm->dur_us;
  fa.tool_u8 = sm->tool_u8;
  fa.n = sm->n;
  fa.F = F;
  fa.K = K;
  fa.step = cp->grid_step_us;
  fa.b_us = est->b_us;
  if (!pairs) {  // rank's slice of every tool segment; world 1 = everything
    fa.voff[0] = 0;
    for (int f = 0; f < F; ++f) {
      const int64_t lo = sm->tool_off[f], len = sm->tool_off[f + 1] - lo;
      fa.seg_lo[f] = lo + (int64_t)((i128)len * rank / world);
      fa.seg_hi[f] = lo + (int64_t)((i128)len * (rank + 1) / world);
      fa.voff[f + 1] = fa.voff[f] + (fa.seg_hi[f] - fa.seg_lo[f]);
    }
  }
  // piece bound: a lane-index replica sees <= ch/lr + 64 samples of one piece (remainder sums
  // < step each stay < 2^32), a thread <= ch/256 + 8 (64-bit sum of squares < 2^64); pairs:
  // a (tool, bucket) bin sees <= ch samples
  int64_t ch = 1ll << 20;
  const int64_t rdiv = pairs ? 1 : plan.lr;
  while (ch > 256 && (ch / rdiv + 64) * (uint64_t)cp->grid_step_us >= (1ull << 32)) ch >>= 1;
  {
    const unsigned __int128 b2 = (unsigned __int128)est->b_us * est->b_us;
    while (ch > 256 && (unsigned __int128)(ch / 256 + 8) * b2 >= ((unsigned __int128)1 << 64)) ch >>= 1;
  }
  if (ch <= 256 && (256 / rdiv + 64) * (uint64_t)cp->grid_step_us >= (1ull << 32))
    return fail(CT_EINVAL, "grid step too large for the histogram pass");
  fa.ch = ch;
  if (cp->grid_step_us >= 2) {  // Granlund-Montgomery: floor(x / d) for every x < 2^32
    const uint32_t d = (uint32_t)cp->grid_step_us;
    const int fl = 31 - __builtin_clz(d);
    if ((d & (d - 1)) == 0) {
      fa.div_m = 1u << (32 - fl), fa.div_sh = 0, fa.div_add = 0;  // x >> fl
    } else {
      const uint64_t num = 1ull << (32 + fl);
      uint32_t pm = (uint32_t)(num / d), rem = (uint32_t)(num % d);
      if (d - rem < (1u << fl)) {
        fa.div_m = pm + 1, fa.div_sh = fl, fa.div_add = 0;
      } else {
        pm += pm;
        const uint32_t tr = rem + rem;
        if (tr >= d || tr < rem) pm += 1;
        fa.div_m = pm + 1, fa.div_sh = fl, fa.div_add = 1;
      }
    }
  }
  std::memset(&sa, 0, sizeof sa);
  sa.F = F;
  sa.K = K;
  sa.J = J;
  sa.cost = *cp;
  sa.est = *est;
  return CT_OK;
}

int fit_grid(ct_ctx* c, const ct::FitArgs& fa, const ct::FitPlan& plan) {
  const int dv = fa.step == 1 ? 0 : fa.div_add ? 2 : 1;  // the kernel instantiation
  const int key = (plan.smem * 8 + (plan.pairs ? 4 : 0) + (fa.b_us < (1ll << 26) ? 1 : 0)) * 4 + dv;
  if (c->fit_occ_key != key) {
    c->fit_occ = ct::fit_hist_occupancy(fa, plan);
    c->fit_occ_key = key;
  }
  return c->sm_count * c->fit_occ;
}

int ensure_fit_buffers(ct_ctx* c, int64_t words) {
  for (int i = 0; i < 2; ++i) {
    if (c->fitbuf_cap[i] >= (size_t)(8 * words) && c->fitbuf[i]) continue;
    int rc = ensure(&c->fitbuf[i], &c->fitbuf_cap[i], 8 * (size_t)words);
    if (rc) return rc;
    c->fit_clean[i] = 0;
  }
  return CT_OK;
}

}  // namespace

int ct_bernstein(ct_ctx* c, const ct_stat_row* rows, int64_t n, const ct_estimator_params* est,
                 int64_t* out, void* stream) {
  if (!c || !est || n < 0 || (n > 0 && (!rows || !out))) return fail(CT_EINVAL, "NULL argument");
  if (!est_valid(*est)) return fail(CT_EINVAL, "invalid estimator parameters");
  cudaError_t e = ct::launch_bernstein(rows, n, *est, out, c->sm_count, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "bernstein launch");
  return CT_OK;
}

int ct_calc_ttl_batch(ct_ctx* c, const ct_stat_row* g, const ct_stat_row* f,
                      const int64_t* n_done, const int64_t* turns_done, int64_t n,
                      const ct_estimator_params* est, int64_t* out, void* stream) {
  if (!c || !est || n < 0 || (n > 0 && (!g || !f || !n_done || !turns_done || !out)))
    return fail(CT_EINVAL, "NULL argument");
  if (!est_valid(*est)) return fail(CT_EINVAL, "invalid estimator parameters");
  cudaError_t e = ct::launch_calc_ttl(g, f, n_done, turns_done, n, *est, out, c->sm_count,
                                      (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "calc_ttl launch");
  return CT_OK;
}

int64_t ct_bernstein_ref(const ct_stat_row* row, const ct_estimator_params* est) {
  if (!row || !est || !est_valid(*est)) return CT_TTL_INVALID;
  return ct::bernstein_row(*row, *est);
}

int64_t ct_calc_ttl_ref(const ct_stat_row* g, const ct_stat_row* f, const ct_estimator_params* est,
                        int64_t n_done, int64_t turns_done) {
  if (!g || !f || !est || !est_valid(*est)) return CT_TTL_INVALID;
  return ct::calc_ttl_row(*g, *f, *est, n_done, turns_done);
}

int64_t ct_fit_acc_words(int32_t n_tools, int32_t K) {
  if (n_tools < 1 || n_tools > CT_MAX_TOOLS || K < 1 || K > CT_MAX_K) return -1;
  return ct::fit_acc_words(n_tools, K);
}

int ct_fit_ttl(ct_ctx* c, const ct_samples* sm, const ct_cost_params* cp,
               const ct_estimator_params* est, ct_ttl_table* out, void* stream) {
  ct::FitArgs fa;
  ct::ScanArgs sa;
  ct::FitPlan plan;
  int rc = fit_prepare(c, sm, cp, est, 0, 1, fa, sa, plan);
  if (rc) return rc;
  if (!out || !out->ttl_argmax || !out->ttl_paper) return fail(CT_EINVAL, "NULL output table");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t W = ct::fit_acc_words(fa.F, fa.K);
  if ((rc = ensure_fit_buffers(c, W))) return rc;
  const int cur = c->fit_cur;
  if (c->fit_clean[cur] < W) CT_CUDA(cudaMemsetAsync(c->fitbuf[cur], 0, 8 * (size_t)W, s));
  c->fit_clean[cur] = 0;  // dirty from here on
  fa.acc = (unsigned long long*)c->fitbuf[cur];
  sa.acc = fa.acc;
  sa.ttl_argmax = out->ttl_argmax;
  sa.ttl_paper = out->ttl_paper;
  sa.stats_out = out->stats;
  sa.n_invalid = out->n_invalid;
  if (!plan.pairs) {  // the histogram kernel zeroes the other half for the next call
    fa.zero = (unsigned long long*)c->fitbuf[cur ^ 1];
    fa.zero_words = W;
  }
  const int grid = fit_grid(c, fa, plan);
  if (grid < 1) return fail(CT_ECUDA, "fit kernel cannot be resident");
  if (c->timing) CT_CUDA(cudaEventRecord(c->ev[2], s));
  cudaError_t e = ct::launch_fit_hist(fa, plan, grid, s);
  if (e != cudaSuccess) return cuda_fail(e, "fit launch");
  e = ct::launch_fit_finish(sa, s);
  if (e != cudaSuccess) return cuda_fail(e, "fit finish launch");
  if (c->timing) CT_CUDA(cudaEventRecord(c->ev[3], s));
  c->fit_timed = c->timing;
  if (!plan.pairs) c->fit_clean[cur ^ 1] = W;
  c->fit_cur = cur ^ 1;
  c->last.launches = 2;
  return CT_OK;
}

int ct_fit_ttl_partial(ct_ctx* c, const ct_samples* sm, const ct_cost_params* cp,
                       const ct_estimator_params* est, int32_t rank, int32_t world, int64_t* acc,
                       void* stream) {
  ct::FitArgs fa;
  ct::ScanArgs sa;
  ct::FitPlan plan;
  int rc = fit_prepare(c, sm, cp, est, rank, world, fa, sa, plan);
  if (rc) return rc;
  if (!acc) return fail(CT_EINVAL, "acc is NULL");
  cudaStream_t s = (cudaStream_t)stream;
  CT_CUDA(cudaMemsetAsync(acc, 0, 8 * (size_t)ct::fit_acc_words(fa.F, fa.K), s));
  fa.acc = (unsigned long long*)acc;
  const int grid = fit_grid(c, fa, plan);
  if (grid < 1) return fail(CT_ECUDA, "fit kernel cannot be resident");
  if (c->timing) CT_CUDA(cudaEventRecord(c->ev[2], s));
  cudaError_t e = ct::launch_fit_hist(fa, plan, grid, s);
  if (e != cudaSuccess) return cuda_fail(e, "fit launch");
  if (c->timing) CT_CUDA(cudaEventRecord(c->ev[3], s));
  c->fit_timed = c->timing;
  c->last.launches = 1;
  return CT_OK;
}

int ct_fit_ttl_finish(ct_ctx* c, const int64_t* acc, int32_t n_tools, const ct_cost_params* cp,
                      const ct_estimator_params* est, ct_ttl_table* out, void* stream) {
  if (!c || !acc || !cp || !est || !out || !out->ttl_argmax || !out->ttl_paper)
    return fail(CT_EINVAL, "NULL argument");
  // the same parameter checks as the histogram pass (an empty CSR set of n_tools tools)
  int64_t off[CT_MAX_TOOLS + 1] = {0};
  if (n_tools < 1 || n_tools > CT_MAX_TOOLS) return fail(CT_EINVAL, "n_tools %d", n_tools);
  ct_samples none{};
  none.tool_off = off;
  none.n_tools = n_tools;
  ct::FitArgs fa;
  ct::ScanArgs sa;
  ct::FitPlan plan;
  int rc = fit_prepare(c, &none, cp, est, 0, 1, fa, sa, plan);
  if (rc) return rc;
  sa.acc = (const unsigned long long*)acc;
  sa.ttl_argmax = out->ttl_argmax;
  sa.ttl_paper = out->ttl_paper;
  sa.stats_out = out->stats;
  sa.n_invalid = out->n_invalid;
  cudaError_t e = ct::launch_fit_finish(sa, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "fit finish launch");
  c->last.launches = 1;
  return CT_OK;
}

int ct_jct_stats(ct_ctx* c, const ct_replica_summary* sum, int64_t n, int32_t n_cells,
                 ct_cell_stats* out, void* stream) {
  if (!c || !sum || !out) return fail(CT_EINVAL, "NULL argument");
  if (n_cells < 1 || n < 0 || n % n_cells) return fail(CT_EINVAL, "n_replicas must be a multiple of n_cells");
  cudaError_t e = ct::launch_jct_stats(sum, n, n_cells, out, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "jct_stats launch");
  return CT_OK;
}


// ---------------------------------------------------------------------------------------------
int ct_synthesize_traces(ct_ctx* c, const ct_synth_params* sp, int64_t seed0, int32_t n_seeds,
                         int32_t P, ct_program* programs, ct_turn* turns, int64_t turns_cap,
                         int64_t* n_turns, void* stream) {
  if (!c || !sp || !n_turns) return fail(CT_EINVAL, "NULL argument");
  *n_turns = 0;
  if (P < 1 || P > CT_MAX_PROGRAMS) return fail(CT_EINVAL, "n_programs %d not in [1, %d]", P, CT_MAX_PROGRAMS);
  if (n_seeds < 0 || seed0 < 0) return fail(CT_EINVAL, "seed range");
  const int F = sp->n_tools;
  if (F < 1 || F > CT_MAX_TOOLS) return fail(CT_EINVAL, "n_tools %d", F);
  if (sp->ctx_cap < 8192 || sp->ctx_cap >= (1ll << 31)) return fail(CT_EINVAL, "ctx_cap not in [8192, 2^31)");
  if (sp->max_turns < 2 || sp->max_turns > 1024) return fail(CT_EINVAL, "max_turns not in [2, 1024]");
  if (sp->n_bfcl < 0 || sp->n_bfcl > P) return fail(CT_EINVAL, "n_bfcl not in [0, P]");
  if (!sp->turns_swe || !sp->obs || !sp->dec || !sp->dur || !sp->exp_q20 || !sp->tool_cdf || !sp->tool_class)
    return fail(CT_EINVAL, "NULL table");
  if (turns_cap < 0 || turns_cap >= (1ll << 31)) return fail(CT_EINVAL, "turns_cap not in [0, 2^31)");
  const int nt = 6 + F;
  const int64_t* rows[6] = {sp->turns_swe, sp->obs, sp->obs + CT_SYNTH_TABLE, sp->dec,
                            sp->dec + CT_SYNTH_TABLE, sp->exp_q20};
  std::vector<int64_t> tab((size_t)nt * CT_SYNTH_TABLE);
  for (int r = 0; r < nt; ++r) {
    const int64_t* src = r < 6 ? rows[r] : sp->dur + (size_t)(r - 6) * CT_SYNTH_TABLE;
    for (int i = 0; i < CT_SYNTH_TABLE; ++i) {
      if (src[i] < 0 || src[i] >= (1ll << 46) || (i && src[i] < src[i - 1]))
        return fail(CT_EINVAL, "table %d is not monotone in [0, 2^46)", r);
      tab[(size_t)r * CT_SYNTH_TABLE + i] = src[i];
    }
  }
  bool has[2] = {false, false};
  for (int f = 0; f < F; ++f) {
    if (sp->tool_class[f] != 0 && sp->tool_class[f] != 1) return fail(CT_EINVAL, "tool_class[%d]", f);
    has[sp->tool_class[f]] = true;
  }
  if (!has[0] || !has[1]) return fail(CT_EINVAL, "each class needs at least one tool");
  if (n_seeds == 0) return CT_OK;
  if (!programs || (turns_cap > 0 && !turns)) return fail(CT_EINVAL, "NULL output");
  const int64_t S = n_seeds, nb = (S + 1023) / 1024;
  const size_t o_tab = 0, o_cdf = o_tab + 8 * tab.size(), o_cls = o_cdf + 4 * (size_t)F,
               o_pcls = (o_cls + 4 * (size_t)F + 15) & ~(size_t)15, o_tot = (o_pcls + (size_t)S * P + 15) & ~(size_t)15,
               o_blk = o_tot + 8 * (size_t)S, bytes = o_blk + 8 * (size_t)(nb + 1);
  int rc = ensure(&c->syn, &c->syn_cap, bytes);
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  unsigned char* base = (unsigned char*)c->syn;
  CT_CUDA(cudaMemcpyAsync(base + o_tab, tab.data(), 8 * tab.size(), cudaMemcpyHostToDevice, s));
  CT_CUDA(cudaMemcpyAsync(base + o_cdf, sp->tool_cdf, 4 * (size_t)F, cudaMemcpyHostToDevice, s));
  CT_CUDA(cudaMemcpyAsync(base + o_cls, sp->tool_class, 4 * (size_t)F, cudaMemcpyHostToDevice, s));
  ct::SynthLaunch L;
  L.sp = sp;
  L.seed0 = seed0;
  L.n_seeds = S;
  L.P = P;
  L.tab = (const int64_t*)(base + o_tab);
  L.cdf = (const uint32_t*)(base + o_cdf);
  L.cls = (const int32_t*)(base + o_cls);
  L.progs = programs;
  L.turns = turns;
  L.turns_cap = turns_cap;
  L.pcls = base + o_pcls;
  L.seed_tot = (int64_t*)(base + o_tot);
  L.blk = (int64_t*)(base + o_blk);
  int64_t total = 0;
  cudaError_t e = ct::launch_synth(L, c->sm_count, s, &total);
  if (e != cudaSuccess) return cuda_fail(e, "synthesis");
  *n_turns = total;
  if (total > turns_cap)
    return fail(CT_EINVAL, "turns_cap %lld < %lld turn records", (long long)turns_cap, (long long)total);
  return CT_OK;
}
}  // extern "C"
