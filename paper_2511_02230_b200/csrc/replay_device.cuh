// replay_device.cuh — warp-per-replica discrete-event replay of Continuum's scheduler (sm_100a).
//
// One warp simulates one replica (a seed x rate x KV budget x policy point of the sweep):
// Alg. 1 — OnRequestArrive, OnRequestFinish + CalcTTL, Schedule with
// release / pinning-aware priority / HOL break — plus §5.3 (pin only when
// TTL != 0, unpin on expiry when the program is not waiting, victims by latest arrival), in the
// integer engine model of DESIGN.md C-5/C-6.  Program p lives on lane p % 32, slot p / 32.
// Per-program scalars are SoA in shared memory (written only by the owner lane); the sets
// Q / pinned / running are per-lane bit registers queried with ballots.  Identical engine
// iterations are macro-stepped: the warp jumps straight to the first iteration boundary that
// is a finish or lies at/after the next external event, which parity tests prove equal to the
// oracle's one-iteration-at-a-time stepping.
#pragma once
#include <cstdlib>

#include "ct_device.cuh"
#include "ct_internal.h"

namespace ct {

enum : int { S_OUT = 0, S_QUEUED = 1, S_RUN = 2, S_LOAD = 3, S_READY = 4, S_TOOL = 5, S_DONE = 6 };


// -----------------------------------------------------------------------------------------------
// P <= 32: one program per lane, all per-program state in registers.  Every event source is a
// per-lane time (program arrival, tool return, load done, pin expiry), so the next event is one
// 64-bit REDUX minimum; events of one kind at one instant are applied by their owner lanes in
// parallel, and only order-dependent work (finishes, DRAM write-through, estimator updates,
// admission) is serialised in program-index order with the operands broadcast by shuffles.
// Same semantics as replay_one<NS> (C-5/C-6), checked byte for byte by the tests.
// Iterations in one macro-step: the smallest j <= m (m = iterations until the first finish)
// whose end dur1 + (j-1) d is at or after the next external event at offset gap (INF-safe),
// i.e. min(m, 1 + ceil(g / d)) with g = gap - dur1.  Past the integer test g <= (m-1) d the
// quotient is below m (a few thousand at most), so the float estimate g * rd (rd ~ 1/d, one
// MUFU.RCP per batch change) is within one of it and two integer corrections make it exact.
__device__ __forceinline__ int64_t macro_iters(int64_t m, int64_t gap, int64_t dur1, int64_t d,
                                               float rd) {
  if (gap >= CT_INF64 / 2) return m;
  const int64_t g = gap - dur1;
  if (g <= 0) return 1;
  if (g > (m - 1) * d) return m;
  int64_t c = (int64_t)((float)g * rd);
  while (c * d < g) ++c;
  while (c > 0 && (c - 1) * d >= g) --c;
  return 1 + c;
}

__device__ __forceinline__ float rcp_approx(float x) {  // one MUFU.RCP, max error ~1 ulp
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// 32-bit variant for d < 2^31 µs (host-checked for the FAST kernels): m - 1 < 2^31 (m is at
// most a request's decode tokens), so every product is one 32 x 32 -> 64-bit multiply.
__device__ __forceinline__ int64_t macro_iters32(int64_t m, int64_t gap, int64_t dur1, uint32_t d,
                                                 float rd) {
  if (gap >= CT_INF64 / 2) return m;
  const int64_t g = gap - dur1;
  if (g <= 0) return 1;
  if ((uint64_t)g > (uint64_t)(uint32_t)(m - 1) * d) return m;
  uint32_t c = (uint32_t)((float)g * rd);
  while ((uint64_t)c * d < (uint64_t)g) ++c;
  while (c > 0 && (uint64_t)(c - 1) * d >= (uint64_t)g) --c;
  return 1 + (int64_t)c;
}

enum : int {  // summary counter index (FAST path: the lane that holds it)
  ACC_BUBBLE = 0, ACC_PREFILL, ACC_RECOMP, ACC_BUSY, ACC_HITS, ACC_EXP, ACC_VICT, ACC_RELOAD
};

struct Acc {  // per-replica summary counters (P <= 32 path)
  int64_t bubble, prefill, recomp, busy;
  int32_t hits, exp, vict, reload;
};

__device__ __forceinline__ int64_t shfl64(int64_t v, int src) {
  return (int64_t)__shfl_sync(FULL_MASK, (unsigned long long)v, src);
}

// FAST: the policy is in the TTL-grid class (fast_policy(), ct_internal.h), so the estimator,
// DRAM, request-FCFS / PLAS and the other pause actions compile away.
template <bool FAST>
__device__ __forceinline__ void replay_one_w32(const ReplayArgs& a, int64_t r, Stat* stats,
                                               int lane) {
  const int P = a.P, F = a.F;
  const int64_t npol = a.n_pol, nkv = a.n_kv, nrate = a.n_rate;
  const int pol_i = (int)(r % npol);
  const int kv_i = (int)((r / npol) % nkv);
  const int rate_i = (int)((r / (npol * nkv)) % nrate);
  const int64_t seed = r / (npol * nkv * nrate);
  const ct_policy* polp = a.pols + pol_i;  // t_pin / t_thresh re-read from L1 when needed
  const int prio = FAST ? CT_PRIO_PROG_FCFS : polp->priority;
  const int pause = FAST ? CT_PAUSE_FIXED : polp->pause;
  const int pflags = FAST ? 0 : polp->flags;
  const int64_t gap = a.gap[rate_i];
  const ct_engine_params& E = a.eng;
  const ct_estimator_params& est = a.est;
  const int64_t bs = E.bs;
  DivMagic bsm;
  bsm.mhi = (uint32_t)(a.bs_magic >> 32);
  bsm.mlo = (uint32_t)a.bs_magic;
  bsm.dm1 = (uint32_t)(bs - 1);
  bsm.ident = bs == 1 ? 1u : 0u;
  const bool eager = (pflags & CT_FLAG_STEP_EXPIRY) == 0;
  const bool vany = (pflags & CT_FLAG_VICTIMS_ANY) != 0;
  const bool dram_on = !FAST && polp->dram != 0 && E.dram_blocks > 0;
  const bool need_stats = !FAST && (pause == CT_PAUSE_PAPER || pause == CT_PAUSE_INFERCEPT ||
                                    (pause == CT_PAUSE_FIXED && polp->t_thresh_us != CT_ALWAYS));
  const bool plas = !FAST && prio == CT_PRIO_PLAS;
  if (need_stats) {
    for (int i = lane; i < 4 * (F + 1); i += 32) ((int64_t*)stats)[i] = 0;
    __syncwarp();
  }

  // ---- this lane's program -----------------------------------------------------------------
  const bool live = lane < P;
  int32_t turn0 = 0, nturns = 1;
  int64_t arr = CT_INF64;
  if (live) {
    const ct_program pr = a.progs[seed * P + lane];
    turn0 = pr.turn0;
    nturns = pr.nturns;
    arr = (pr.arr_q * gap) >> 20;
  }
  const int64_t arr0 = shfl64(arr, 0);  // programs arrive in index order: min arrival
  // per-program bubble series (NEXT-3), accumulated in place by the owner lane (the address
  // is recomputed at each use: no register is held for it across the event loop)
  if (a.bubble && live) a.bubble[(r - a.r_begin) * P + lane] = 0;
  int st = S_OUT;
  int64_t tev = arr;          // arrival (OUT), tool return (TOOL), load done (LOAD); INF otherwise
  int64_t texp = CT_INF64;    // expiry + 1 while pinned in a tool call
  int64_t req = 0;            // request arrival; JCT once done
  int64_t fin = 0;            // iteration index at whose end the running request finishes
  int32_t ctx = 0, gblk = 0, dblk = 0, unc = 0, turn = 0;
  bool pin = false;
  int64_t svc = 0;  // attained engine time of the program (PLAS)
  int4 rec = make_int4(0, 0, -1, 0);  // current turn record (new, decode, tool, dur)

  int64_t now = 0, iter_end = 0, n_it = 0;
  bool in_flight = false;
  // block counts are < 2^30 (host-validated): 32-bit registers
  int32_t free_blk = (int32_t)a.kv[kv_i];
  int32_t dfree = dram_on ? (int32_t)E.dram_blocks : 0;
  int64_t chan = 0;
  int32_t D = 0, turns_done = 0;  // completed programs and their turns (P <= 32)
  int n_run = 0, n_load = 0;  // n_load counts LOADING and READY
  int32_t kv_sum = 0;
  int64_t pf = 0;
  int status = CT_R_OK;
  // summary counters: generic path in shared memory (lane 0 updates them) to keep registers for
  // occupancy; FAST path one counter per lane in a register (lane k holds counter k of ACC_*)
  Acc* acc = (Acc*)(stats + F + 1);
  if (!FAST && lane == 0) *acc = Acc{0, 0, 0, 0, 0, 0, 0, 0};
  int64_t accv = 0;
#define ACC_ADD(field, k, v)                     \
  do {                                           \
    if (FAST) {                                  \
      if (lane == (k)) accv += (int64_t)(v);     \
    } else if (lane == 0) {                      \
      acc->field += (v);                         \
    }                                            \
  } while (0)
  // duration of a no-prefill iteration for the current batch (depends on kv_sum only) and its
  // reciprocal for the macro-step division, recomputed only when kv_sum changes
  int32_t kv_at = -1;
  int64_t d_cur = 0, base_ps = 0;  // base_ps = c0 + c_kv bs kv_sum (ps), d_cur = ceil(base_ps / 1e6)
  float rd_cur = 0.0f;

  // evict(v): free its GPU blocks; DRAM write-through when the tier is on (R18).  Uniform.
  auto evict = [&](int v) {
    const int32_t g = __shfl_sync(FULL_MASK, gblk, v);
    free_blk += g;
    int32_t keep = 0;
    if (dram_on) {
      const uint32_t vctx = __shfl_sync(FULL_MASK, (uint32_t)ctx, v);
      const int64_t nb = ceil_div_magic(vctx, bsm);
      dfree += __shfl_sync(FULL_MASK, dblk, v);
      if (nb > 0 && nb <= dfree) { keep = (int32_t)nb; dfree -= (int32_t)nb; }
    }
    if (lane == v) { gblk = 0; dblk = keep; pin = false; texp = CT_INF64; }
  };

  for (;;) {
    // ---- next event (R1, R3) --------------------------------------------------------------
    // With an iteration in flight nothing can be scheduled before its end (R2), so every
    // program event up to iter_end is applied in one pass at the boundary, each program's own
    // events in R1 order: their effects commute (per-program state, block and statistics sums),
    // except DRAM write-through, which is applied in (time, index) order.  Idle, the next event
    // instant is one REDUX minimum.
    int64_t t;
    if (in_flight) {
      t = iter_end;
    } else {
      t = warp_min64_redux(eager ? min(tev, texp) : tev);
      if (t == CT_INF64) break;
    }
    now = t;

    if (__any_sync(FULL_MASK, (eager ? min(tev, texp) : tev) <= now)) {
      // PinExpiry (EAGER, R4/R15): first µs with now > expiry while not in Q; it precedes the
      // program's own tool return at the same µs (R1)
      if (eager) {
        const bool xd = texp <= now && texp <= tev;
        uint32_t m = __ballot_sync(FULL_MASK, xd);
        if (m) {
          ACC_ADD(exp, ACC_EXP, __popc(m));
          if (dram_on) {  // write-through order matters: (time, index) order
            while (m) {
              const int64_t tm = warp_min64_redux((m >> lane) & 1u ? texp : CT_INF64);
              const int p = __ffs(__ballot_sync(FULL_MASK, ((m >> lane) & 1u) && texp == tm)) - 1;
              m &= ~(1u << p);
              evict(p);
            }
          } else {
            free_blk += (int32_t)__reduce_add_sync(FULL_MASK, xd ? (uint32_t)gblk : 0u);
            if (xd) { gblk = 0; pin = false; texp = CT_INF64; }
          }
        }
      }
      const bool due = tev <= now;
      // ToolReturn == OnRequestArrive of a seen program
      const bool ret = due && st == S_TOOL;
      if (need_stats) {
        uint32_t m = __ballot_sync(FULL_MASK, ret);
        while (m) {  // estimator rows: Δ_obs = dur of the finished turn's tool, clamped (R5)
          const int p = __ffs(m) - 1;
          m &= m - 1;
          const int f = __shfl_sync(FULL_MASK, rec.z, p);
          const int64_t x = min((int64_t)__shfl_sync(FULL_MASK, rec.w, p), est.b_us);
          const uint64_t x2 = (uint64_t)x * (uint64_t)x;
          if (lane == 0) {
            Stat* rows[2] = {&stats[F], &stats[f]};
#pragma unroll
            for (int k = 0; k < 2; ++k) {
              Stat* q = rows[k];
              q->n += 1;
              q->s1 += x;
              const uint64_t lo = q->s2lo + x2;
              q->s2hi += (lo < x2);
              q->s2lo = lo;
            }
          }
          __syncwarp();
        }
      }
      if (ret) {
        ++turn;
        rec = __ldg((const int4*)a.turns + turn0 + turn);
        st = S_QUEUED;
        req = tev;  // the event's own instant
        tev = CT_INF64;
        texp = CT_INF64;  // a retained pin has no expiry event while waiting
      }
      // LoadDone
      if (due && st == S_LOAD) { st = S_READY; tev = CT_INF64; }
      // ProgramArrival
      if (due && st == S_OUT) {
        st = S_QUEUED;
        req = tev;
        tev = CT_INF64;
        rec = __ldg((const int4*)a.turns + turn0);
      }
    }

    // IterationEnd: members whose last token was emitted finish, in index order (C-6)
    if (in_flight && iter_end == now) {
      in_flight = false;
      uint32_t m = __ballot_sync(FULL_MASK, st == S_RUN && fin == n_it);
      while (m) {
        const int p = __ffs(m) - 1;
        m &= m - 1;
        // OnRequestFinish
        const int pt = __shfl_sync(FULL_MASK, turn, p);
        const int pn = __shfl_sync(FULL_MASK, nturns, p);
        const int pg = __shfl_sync(FULL_MASK, gblk, p);
        const int ptool = __shfl_sync(FULL_MASK, rec.z, p);
        --n_run;
        kv_sum -= pg;
        if (lane == p) ctx += rec.x + rec.y;
        if (pt == pn - 1) {  // last request: free its KV, the program completes
          free_blk += pg;
          dfree += __shfl_sync(FULL_MASK, dblk, p);
          if (lane == p) { gblk = 0; dblk = 0; st = S_DONE; req = now - arr; }
          ++D;
          turns_done += pn;
        } else {
          int64_t ttl = 0;
          switch (pause) {
            case CT_PAUSE_FIXED:
            case CT_PAUSE_PAPER: {
              if (FAST) {  // FIXED with CT_ALWAYS pins for t_pin; EVICT never pins
                ttl = polp->pause == CT_PAUSE_FIXED ? polp->t_pin_us : 0;
                break;
              }
              const Stat sg = stats[F], sf = stats[ptool];
              ttl = pause == CT_PAUSE_PAPER
                        ? calc_ttl(sg, sf, est, D, turns_done)
                        : simplified_ttl(sg, sf, est, polp->t_pin_us, polp->t_thresh_us);
              break;
            }
            case CT_PAUSE_FITTED:
              ttl = __ldg(&a.fitted[(int64_t)ptool * a.J + min(pt, a.J - 1)]);
              break;
            case CT_PAUSE_INFERCEPT: {  // preserve (no TTL) iff prediction < swap round trip
              const int64_t pred = infercept_predict(stats[F], stats[ptool], est);
              const uint32_t pctx = __shfl_sync(FULL_MASK, (uint32_t)ctx, p);
              const int64_t blocks = ceil_div_magic(pctx, bsm);
              const int64_t swap = 2 * ceil_ps_to_us((uint64_t)(blocks * E.c_h2d_ps));
              ttl = pred < swap ? CT_INF64 : 0;
              break;
            }
            default:
              ttl = 0;
          }
          if (ttl > 0) {  // pin_request only if TTL != 0
            if (lane == p) { pin = true; texp = ttl == CT_INF64 ? CT_INF64 : now + ttl + 1; }
          } else {
            evict(p);
          }
          if (lane == p) { tev = now + rec.w; st = S_TOOL; }
        }
      }
    }
    if (in_flight) continue;  // mid-iteration: events only mutate Q / stats / pins (R2)

    // ---- scheduling point (R3) --------------------------------------------------------------
    // (a) STEP reading: release expired pins of programs not waiting
    if (!eager) {
      uint32_t m = __ballot_sync(FULL_MASK, pin && st == S_TOOL && texp <= now);
      ACC_ADD(exp, ACC_EXP, __popc(m));
      while (m) {
        const int p = __ffs(m) - 1;
        m &= m - 1;
        evict(p);
      }
    }
    // fast path: nothing waiting and nothing loaded -> (b)-(d) are no-ops
    const bool work = __any_sync(FULL_MASK, st == S_QUEUED || st == S_READY);
    int admitted = 0;
    bool stable = true;
    if (work) {
    // (b) loaded requests join the batch
    {
      const bool join = st == S_READY;
      const uint32_t m = __ballot_sync(FULL_MASK, join);
      if (m) {
        kv_sum += (int32_t)__reduce_add_sync(FULL_MASK, join ? (uint32_t)gblk : 0u);
        pf += (int64_t)__reduce_add_sync(FULL_MASK, join ? (uint32_t)unc : 0u);
        n_run += __popc(m);
        n_load -= __popc(m);
        if (join) { st = S_RUN; fin = n_it + rec.y; }
      }
    }
    // (c) admit loop (victims PAPER.md:645-655)
    for (;;) {
      const uint32_t mq = __ballot_sync(FULL_MASK, st == S_QUEUED);
      if (!mq) break;
      if (n_run + n_load >= E.max_batch) break;
      int h;
      if (prio == CT_PRIO_PROG_FCFS) {
        const uint32_t mp = __ballot_sync(FULL_MASK, st == S_QUEUED && pin);
        h = __ffs(mp ? mp : mq) - 1;
      } else {  // REQ_FCFS: earliest request; PLAS: least attained service; ties: index
        const bool q = st == S_QUEUED;
        const int64_t key = plas ? svc : req;
        const int64_t mr = warp_min64_redux(q ? key : CT_INF64);
        h = __ffs(__ballot_sync(FULL_MASK, q && key == mr)) - 1;
      }
      const int32_t hctx = __shfl_sync(FULL_MASK, ctx, h);
      const int32_t hg = __shfl_sync(FULL_MASK, gblk, h);
      const int32_t hnew = __shfl_sync(FULL_MASK, rec.x, h);
      const int32_t hdec = __shfl_sync(FULL_MASK, rec.y, h);
      const int64_t need = (int64_t)ceil_div_magic((uint32_t)(hctx + hnew + hdec), bsm) - hg;
      if (need > free_blk && (admitted == 0 || vany)) {
        while (need > free_blk) {  // victims: latest program arrival first, never the head
          const uint32_t mv = __ballot_sync(FULL_MASK, pin && lane != h);
          if (!mv) break;
          evict(31 - __clz(mv));
          ACC_ADD(vict, ACC_VICT, 1);
        }
      }
      if (need > free_blk) {  // HOL break
        if (admitted > 0 && !vany && __ballot_sync(FULL_MASK, pin && lane != h)) stable = false;
        break;
      }
      // issue h
      free_blk -= (int32_t)need;
      const int32_t ng = hg + (int32_t)need;
      const int64_t hreq = shfl64(req, h);
      ACC_ADD(bubble, ACC_BUBBLE, now - hreq);
      const bool hp = __shfl_sync(FULL_MASK, pin ? 1 : 0, h) != 0;
      const int32_t hd = __shfl_sync(FULL_MASK, dblk, h);
      int64_t cached;
      bool loading = false;
      int64_t ld = 0;
      if (hp) {
        cached = hctx;
        ACC_ADD(hits, ACC_HITS, 1);
      } else if (dram_on && hd > 0 && hd == (int32_t)ceil_div_magic((uint32_t)hctx, bsm)) {
        cached = hctx;
        loading = true;
        ld = max(now, chan) + ceil_ps_to_us((uint64_t)((int64_t)hd * E.c_h2d_ps));
        chan = ld;
        ACC_ADD(reload, ACC_RELOAD, 1);
      } else {
        cached = 0;
        ACC_ADD(recomp, ACC_RECOMP, hctx);
      }
      const int64_t u = hctx + hnew - cached;
      ACC_ADD(prefill, ACC_PREFILL, u);
      if (lane == h) {
        if (a.bubble) a.bubble[(r - a.r_begin) * P + lane] += now - req;
        pin = false;
        texp = CT_INF64;
        gblk = ng;
        unc = (int32_t)u;
        if (loading) {
          st = S_LOAD;
          tev = ld;
        } else {
          st = S_RUN;
          fin = n_it + rec.y;
        }
      }
      if (loading) {
        ++n_load;
      } else {
        ++n_run;
        kv_sum += ng;
        pf += u;
      }
      ++admitted;
    }
    // (d) unschedulable: the head missed with nothing running or loading; the victim loop has
    // already released every other pin, so no future event can free memory for it (C-5 5c)
    if (admitted == 0 && n_run == 0 && n_load == 0 && __any_sync(FULL_MASK, st == S_QUEUED)) {
      status = CT_R_UNSCHEDULABLE;
      break;
    }
    }  // work
    // (e) start the next iteration(s) (linear cost model, R16)
    if (n_run > 0) {
      if (kv_sum != kv_at) {
        kv_at = kv_sum;
        base_ps = E.c0_ps + E.c_kv_ps * bs * kv_sum;
        d_cur = ceil_ps_to_us((uint64_t)base_ps);
        rd_cur = __frcp_rn((float)d_cur);
      }
      const int64_t d = d_cur;
      // the first iteration carries the prefill of newly admitted requests (R16)
      const int64_t dur1 = pf > 0 ? ceil_ps_to_us((uint64_t)(base_ps + E.c_pf_ps * pf)) : d;
      pf = 0;
      int64_t k = 1;
      if (stable) {
        // macro-step: the first iteration plus identical decode iterations, up to the first
        // finish or the first boundary at or after the next external event
        const int64_t mfin = warp_min64_redux(st == S_RUN ? fin : CT_INF64);
        const int64_t te = warp_min64_redux(min(tev, texp));
        k = FAST ? macro_iters32(mfin - n_it, te - now, dur1, (uint32_t)d, rd_cur)
                 : macro_iters(mfin - n_it, te - now, dur1, d, rd_cur);
      }
      const int64_t dur = dur1 + (k - 1) * d;
      if (n_it + k > E.max_iters) { status = CT_R_EVENT_BUDGET; break; }
      n_it += k;
      iter_end = now + dur;
      ACC_ADD(busy, ACC_BUSY, dur);
      if (plas && st == S_RUN) svc += dur;  // every running request accrues the iterations
      in_flight = true;
    }
  }
  if (status == CT_R_OK && D != P) status = CT_R_UNSCHEDULABLE;

  // ---- per-replica summary (A-8) --------------------------------------------------------------
  const int64_t ri = r - a.r_begin;
  int64_t jsum = 0, jmax = 0, p50 = 0, p99 = 0;
  if (status == CT_R_OK) {
    const int64_t jv = live ? req : 0;
    jsum = (int64_t)warp_sum_u64((uint64_t)jv);
    jmax = warp_max64(jv);
    const int r50 = (50 * P + 99) / 100, r99 = (99 * P + 99) / 100;
    int lt = 0, le = 0;
    for (int q = 0; q < P; ++q) {
      const int64_t x = shfl64(req, q);
      lt += x < req;
      le += x <= req;
    }
    const bool c5 = live && lt < r50 && r50 <= le, c9 = live && lt < r99 && r99 <= le;
    p50 = shfl64(req, __ffs(__ballot_sync(FULL_MASK, c5)) - 1);
    p99 = shfl64(req, __ffs(__ballot_sync(FULL_MASK, c9)) - 1);
  }
  int64_t av[8];
  if (FAST) {
#pragma unroll
    for (int k = 0; k < 8; ++k) av[k] = shfl64(accv, k);
  }
#undef ACC_ADD
  if (lane == 0) {
    if (!FAST) {
      av[ACC_BUBBLE] = acc->bubble;
      av[ACC_PREFILL] = acc->prefill;
      av[ACC_RECOMP] = acc->recomp;
      av[ACC_BUSY] = acc->busy;
      av[ACC_HITS] = acc->hits;
      av[ACC_EXP] = acc->exp;
      av[ACC_VICT] = acc->vict;
      av[ACC_RELOAD] = acc->reload;
    }
    ct_replica_summary o;
    if (status == CT_R_OK) {
      o.status = status;
      o.n_done = D;
      o.turns_done = turns_done;
      o.sum_jct_us = jsum;
      o.max_jct_us = jmax;
      o.p50_jct_us = p50;
      o.p99_jct_us = p99;
      o.sum_bubble_us = av[ACC_BUBBLE];
      o.makespan_us = now - arr0;  // the last event processed is the last completion
      o.iterations = n_it;
      o.busy_us = av[ACC_BUSY];
      o.prefill_tokens = av[ACC_PREFILL];
      o.recompute_tokens = av[ACC_RECOMP];
      o.pin_hits = av[ACC_HITS];
      o.pin_expiries = av[ACC_EXP];
      o.victims = av[ACC_VICT];
      o.reloads = av[ACC_RELOAD];
    } else {
      int64_t* w = (int64_t*)&o;
#pragma unroll
      for (int i = 0; i < 16; ++i) w[i] = 0;
      o.status = status;
    }
    a.out[ri] = o;
  }
  if (a.jct && live) a.jct[ri * P + lane] = status == CT_R_OK ? req : -1;
  if (a.bubble && live && status != CT_R_OK) a.bubble[ri * P + lane] = -1;
  __syncwarp();
}

// -----------------------------------------------------------------------------------------------
// TTL-grid class with 32-bit replica-relative times.  Every time is µs since the replica's first
// arrival (program 0), saturated at T32_LIM; every iteration lasts >= 1 µs, so iteration indices
// stay below the time and fit too.  The moment the next event (or an iteration end) lies at or
// beyond T32_LIM the function returns false and the caller replays the replica on the 64-bit
// path (replay_one_w32<true>): the saturated values are only ever compared, never applied.
// Otherwise identical to replay_one_w32<true> step for step (C-5/C-6); the parity
// tests cover both, including horizons beyond 2^32 µs.
// CalcTTL cache of one tool row (PAPER mode, P > 32 32-bit kernel; measured 2-3 % slower in the
// P <= 32 one, which does not use it).  Once n_f >= N the offset depends
// only on row f's statistics and on (D, turns_done) (g.n >= f.n >= N), and n_f
// grows by one per recorded sample: the key (n_f, D) identifies the inputs exactly.
struct TtlCache {
  uint64_t key;  // n_f << 32 | D, ~0 = empty
  int64_t ttl;
};

// PAPER-mode TTL of a finish with tool f through the cache (warp-uniform; lane 0 writes).
__device__ __forceinline__ int64_t calc_ttl_cached(const Stat* stats, TtlCache* tcache, int F,
                                                   int f, const ct_estimator_params& est,
                                                   int32_t D, int32_t turns_done, int lane) {
  const int64_t nf = stats[f].n;
  const bool keyed = nf >= est.n_min;
  const uint64_t key = ((uint64_t)nf << 32) | (uint32_t)D;
  if (keyed && tcache[f].key == key) return tcache[f].ttl;
  const int64_t ttl = calc_ttl<true, true>(stats[F], stats[f], est, D, turns_done);  // one inlined copy
  if (keyed) {
    __syncwarp();
    if (lane == 0) { tcache[f].key = key; tcache[f].ttl = ttl; }
    __syncwarp();
  }
  return ttl;
}

// Duration (µs) of a no-prefill iteration with kv resident blocks, ceil((c0 + c_kv bs kv) / 1e6),
// for the 32-bit kernels.  When c_kv bs max(kv) + 1e6 < 2^32 (host-checked, ReplayArgs.kv32)
// it is c0q + ceil((c_kv bs kv - c0r) / 1e6) (0 when that is negative) with c0 = c0q 1e6 - c0r,
// 0 <= c0r < 1e6: one 32-bit constant division instead of the 64-bit one.  *rb receives
// d 1e6 - (c0 + c_kv bs kv), in [0, 1e6), for iter_us_prefill.
__device__ __forceinline__ uint32_t iter_us_kv32(const ReplayArgs& a, uint32_t kv, uint32_t* rb) {
  if (a.kv32) {
    const uint32_t x = a.kv_unit * kv;
    const uint32_t e = x > a.c0r ? (x - a.c0r + 999999u) / 1000000u : 0u;
    *rb = e * 1000000u + a.c0r - x;
    return a.c0q + e;
  }
  *rb = 0;
  return (uint32_t)ceil_ps_to_us((uint64_t)(a.eng.c0_ps + a.eng.c_kv_ps * a.eng.bs * (int64_t)kv));
}

// Duration (µs) of an iteration that also prefills pf tokens: ceil((c0 + c_kv bs kv + c_pf pf)
// / 1e6).  With c_pf = pfq 1e6 + pfr and d, rb from iter_us_kv32 it is d + pfq pf +
// ceil((pfr pf - rb) / 1e6) (0 when negative), one 32-bit division while pfr pf + 1e6 < 2^32
// (pf < a.pf32); otherwise the 64-bit sum.
__device__ __forceinline__ int64_t iter_us_prefill(const ReplayArgs& a, uint32_t d, uint32_t rb,
                                                   uint32_t kv, int64_t pf) {
  if (a.kv32 && pf < (int64_t)a.pf32) {
    const uint32_t y = a.pf_r * (uint32_t)pf;
    return (int64_t)d + (int64_t)a.pf_q * pf + (y > rb ? (y - rb + 999999u) / 1000000u : 0u);
  }
  return ceil_ps_to_us((uint64_t)(a.eng.c0_ps + a.eng.c_kv_ps * a.eng.bs * (int64_t)kv +
                                  a.eng.c_pf_ps * pf));
}

constexpr uint32_t T32_INF = 0xFFFFFFFFu;
constexpr uint32_t T32_LIM = 0xFFFFFFF0u;

// Macro-step on 32-bit times (replay_one_t32): the first iteration ends at end1; the result is
// the number j of further iterations of d µs (all identical, no finish before the m1-th), the
// smallest j <= m1 with end1 + j d >= te (the next external event; T32_INF = none), i.e.
// min(m1, ceil((te - end1) / d)), 0 when te <= end1.  Same value as macro_iters32 - 1.  Past
// the test g <= m1 d the quotient is at most m1 (a request's decode tokens), so the float
// estimate is within one of it and the two integer corrections make it exact.
__device__ __forceinline__ uint32_t extra_iters32(uint32_t m1, uint32_t te, uint32_t end1,
                                                  uint32_t d, float rd) {
  if (te == T32_INF) return m1;
  if (te <= end1) return 0;
  const uint32_t g = te - end1;
  if ((uint64_t)m1 * d < g) return m1;
  uint32_t c = (uint32_t)((float)g * rd);
  while ((uint64_t)c * d < g) ++c;
  while (c > 0 && (uint64_t)(c - 1) * d >= g) --c;
  return c;
}

// min(t + x, T32_LIM) for a time t < T32_LIM and a duration x >= 0, in 32-bit arithmetic
__device__ __forceinline__ uint32_t add_sat32(uint32_t t, uint32_t x) {
  return x >= T32_LIM - t ? T32_LIM : t + x;
}

__device__ __forceinline__ uint32_t sat32(int64_t v) {  // v >= 0
  return v >= (int64_t)T32_LIM ? T32_LIM : (uint32_t)v;
}

// STATS = false: the TTL-grid class (fast_policy); STATS = true: program or request FCFS with
// the estimator (simple_policy: EVICT, FIXED with a threshold, PAPER CalcTTL, FITTED), whose
// statistic rows live in shared memory as on the 64-bit path.  EXT (with STATS): the extended
// class (ext_policy: any priority, any pause action, the DRAM tier; flags 0) adds Autellix PLAS,
// InferCept, the DRAM write-through / serialized H2D channel / async load of R18 (LOADING ->
// READY -> joined at the next scheduling point) on the same 32-bit times.
template <bool STATS, bool EXT = false>
__device__ __forceinline__ bool replay_one_t32(const ReplayArgs& a, int64_t r, Stat* stats,
                                               int lane) {
  static_assert(STATS || !EXT, "the extended class needs the estimator rows");
  const int P = a.P;
  const int64_t npol = a.n_pol, nkv = a.n_kv, nrate = a.n_rate;
  const int pol_i = (int)(r % npol);
  const int kv_i = (int)((r / npol) % nkv);
  const int rate_i = (int)((r / (npol * nkv)) % nrate);
  const int64_t seed = r / (npol * nkv * nrate);
  const ct_policy* polp = a.pols + pol_i;
  // TTL-grid class: FIXED with CT_ALWAYS pins for t_pin; EVICT never pins (fast_policy)
  const int pause = polp->pause;
  const int prio = polp->priority;  // STATS: program or request FCFS (simple_policy)
  const int64_t ttl_fixed = pause == CT_PAUSE_FIXED ? polp->t_pin_us : 0;
  // expiry offset ttl + 1 of a FIXED pin, saturated at the horizon (ttl < CT_TTL_SAT)
  const uint32_t ttl1 = ttl_fixed >= (int64_t)T32_LIM ? T32_LIM : (uint32_t)ttl_fixed + 1;
  const int F = a.F;
  const ct_estimator_params& est = a.est;
  const bool need_stats =
      STATS && (pause == CT_PAUSE_PAPER || (EXT && pause == CT_PAUSE_INFERCEPT) ||
                (pause == CT_PAUSE_FIXED && polp->t_thresh_us != CT_ALWAYS));
  const bool dram_on = EXT && polp->dram != 0 && a.eng.dram_blocks > 0;
  const bool plas = EXT && prio == CT_PRIO_PLAS;
  if (need_stats) {
    for (int i = lane; i < 4 * (F + 1); i += 32) ((int64_t*)stats)[i] = 0;
    __syncwarp();
  }
  const int64_t gap = a.gap[rate_i];
  const ct_engine_params& E = a.eng;
  DivMagic bsm;
  bsm.mhi = (uint32_t)(a.bs_magic >> 32);
  bsm.mlo = (uint32_t)a.bs_magic;
  bsm.dm1 = (uint32_t)(E.bs - 1);
  bsm.ident = E.bs == 1 ? 1u : 0u;

  if (a.bubble) return false;  // the per-program bubble output runs on the 64-bit path
  const bool live = lane < P;
  int32_t turn0 = 0, nturns = 1;
  int64_t arr64 = CT_INF64;
  if (live) {
    const ct_program pr = a.progs[seed * P + lane];
    turn0 = pr.turn0;
    nturns = pr.nturns;
    arr64 = (pr.arr_q * gap) >> 20;
  }
  const int64_t arr0 = shfl64(arr64, 0);  // programs arrive in index order: the time origin
  const uint32_t arr = live ? sat32(arr64 - arr0) : T32_INF;
  int st = S_OUT;
  uint32_t tev = arr;      // arrival (OUT), tool return (TOOL), load done (LOAD); INF otherwise
  uint32_t texp = T32_INF; // expiry + 1 while pinned in a tool call
  uint32_t req = 0;        // request arrival; JCT once done
  uint32_t fin = 0;        // iteration index at whose end the running request finishes
  int32_t ctx = 0, gblk = 0, turn = 0;
  int32_t dblk = 0, unc = 0;  // EXT: DRAM copy blocks; uncached tokens of a loading request
  uint32_t svc = 0;           // EXT: attained engine time (PLAS), <= now on this path
  bool pin = false;
  int4 rec = make_int4(0, 0, -1, 0);

  uint32_t now = 0, iter_end = 0, n_it = 0;
  bool in_flight = false;
  int32_t free_blk = (int32_t)a.kv[kv_i];
  int32_t dfree = dram_on ? (int32_t)E.dram_blocks : 0;
  uint32_t chan = 0;  // EXT: the H2D channel is busy until chan
  int32_t D = 0, turns_done = 0;
  int n_run = 0, n_load = 0;  // n_load counts LOADING and READY (EXT)
  int32_t kv_sum = 0;
  int64_t pf = 0;
  int status = CT_R_OK;
  // summary counters (ACC_*): with the estimator, lane k holds counter k in one register; the
  // TTL-grid class accumulates the warp-uniform values in every lane (uniform registers),
  // measured 5 % faster there and 5 % slower with the estimator's register pressure
  // (TTL-grid class: the time and count counters, ACC_BUSY onward, are 32-bit: busy time lies
  // within the replica's span, below the 32-bit horizon, and each count is below 2^31)
  int64_t accv = 0;
  int64_t A[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  uint32_t A32[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  auto acc_add = [&](int k, int64_t v) {
    if (STATS) {
      if (lane == k) accv += v;
    } else if (k >= ACC_BUSY) {
      A32[k] += (uint32_t)v;
    } else {
      A[k] += v;
    }
  };
  const int max_batch = (int)min(E.max_batch, (int64_t)0x7fffffff);
  // iteration budget as a 32-bit bound (n_it < 2^32 on this path)
  const uint32_t it_cap = E.max_iters >= (int64_t)T32_INF ? T32_INF : (uint32_t)E.max_iters;
  int32_t kv_at = -1;
  uint32_t d_cur = 0, rb_cur = 0;
  float rd_cur = 0.0f;
  // evict(v): free its GPU blocks; DRAM write-through when the tier is on (R18).  Uniform.
  auto evict = [&](int v) {
    free_blk += __shfl_sync(FULL_MASK, gblk, v);
    int32_t keep = 0;
    if (dram_on) {
      const uint32_t vctx = __shfl_sync(FULL_MASK, (uint32_t)ctx, v);
      const int32_t nb = (int32_t)ceil_div_magic(vctx, bsm);
      dfree += __shfl_sync(FULL_MASK, dblk, v);
      if (nb > 0 && nb <= dfree) { keep = nb; dfree -= nb; }
    }
    if (lane == v) { gblk = 0; dblk = keep; pin = false; texp = T32_INF; }
  };

  // qleft: a program was still queued after the last admit loop.  Only then can a pin expiry
  // change a decision (it frees blocks for the blocked head or removes a victim candidate);
  // with the queue empty, an expiry is applied at the next event or iteration boundary that
  // is taken anyway: free_blk and the pin set are read only by admission, every program is
  // processed in the order of its own events (expiry before its tool return, R1), and the
  // skipped boundaries lie inside a macro-step with no finish, so nothing else reads them.
  bool qleft = false;
  for (;;) {
    uint32_t t;
    if (in_flight) {
      t = iter_end;
    } else {
      t = __reduce_min_sync(FULL_MASK, qleft ? min(tev, texp) : tev);
      if (t == T32_INF) break;
    }
    if (t >= T32_LIM) return false;  // beyond the 32-bit horizon: replay on the 64-bit path
    now = t;

    if (__any_sync(FULL_MASK, min(tev, texp) <= now)) {
      // PinExpiry (EAGER, R4/R15) precedes the program's own tool return at the same µs (R1)
      const bool xd = texp <= now && texp <= tev;
      uint32_t m = __ballot_sync(FULL_MASK, xd);
      if (m) {
        acc_add(ACC_EXP, __popc(m));
        if (dram_on) {  // write-through order matters: (time, index) order
          while (m) {
            const uint32_t tm = __reduce_min_sync(FULL_MASK, (m >> lane) & 1u ? texp : T32_INF);
            const int p = __ffs(__ballot_sync(FULL_MASK, ((m >> lane) & 1u) && texp == tm)) - 1;
            m &= ~(1u << p);
            evict(p);
          }
        } else {
          free_blk += (int32_t)__reduce_add_sync(FULL_MASK, xd ? (uint32_t)gblk : 0u);
          if (xd) { gblk = 0; pin = false; texp = T32_INF; }
        }
      }
      const bool due = tev <= now;
      if (need_stats) {  // estimator rows: Δ_obs = dur of the finished turn's tool, clamped (R5)
        uint32_t mr = __ballot_sync(FULL_MASK, due && st == S_TOOL);
        while (mr) {
          const int p = __ffs(mr) - 1;
          mr &= mr - 1;
          const int f = __shfl_sync(FULL_MASK, rec.z, p);
          const int64_t x = min((int64_t)__shfl_sync(FULL_MASK, rec.w, p), est.b_us);
          const uint64_t x2 = (uint64_t)x * (uint64_t)x;
          if (lane == 0) {
            Stat* rows[2] = {&stats[F], &stats[f]};
#pragma unroll
            for (int k = 0; k < 2; ++k) {
              Stat* q = rows[k];
              q->n += 1;
              q->s1 += x;
              const uint64_t lo = q->s2lo + x2;
              q->s2hi += (lo < x2);
              q->s2lo = lo;
            }
          }
          __syncwarp();
        }
      }
      if (due && st == S_TOOL) {  // ToolReturn == OnRequestArrive
        ++turn;
        rec = __ldg((const int4*)a.turns + turn0 + turn);
        st = S_QUEUED;
        req = tev;
        tev = T32_INF;
        texp = T32_INF;  // a retained pin has no expiry event while waiting
      } else if (due && st == S_OUT) {  // ProgramArrival
        st = S_QUEUED;
        req = tev;
        tev = T32_INF;
        rec = __ldg((const int4*)a.turns + turn0);
      } else if (EXT && due && st == S_LOAD) {  // LoadDone
        st = S_READY;
        tev = T32_INF;
      }
    }

    // IterationEnd: members whose last token was emitted finish, in index order (C-6)
    if (!STATS && in_flight && iter_end == now) {
      // TTL-grid class: every finish takes the same pause action (pin for ttl_fixed, or evict)
      // and touches only its own program and order-free sums, so the finishing lanes apply
      // it in parallel; D and turns_done are counted once at the end
      in_flight = false;
      const bool f = st == S_RUN && fin == n_it;
      const uint32_t m = __ballot_sync(FULL_MASK, f);
      if (m) {
        const bool last = turn == nturns - 1;
        const bool rel = last || ttl_fixed <= 0;  // the blocks return to the pool
        n_run -= __popc(m);
        kv_sum -= (int32_t)__reduce_add_sync(FULL_MASK, f ? (uint32_t)gblk : 0u);
        free_blk += (int32_t)__reduce_add_sync(FULL_MASK, f && rel ? (uint32_t)gblk : 0u);
        if (f) {
          ctx += rec.x + rec.y;
          if (last) {
            gblk = 0;
            st = S_DONE;
            req = now - arr;
          } else {
            if (ttl_fixed > 0) {  // pin_request only if TTL != 0
              pin = true;
              texp = add_sat32(now, ttl1);
            } else {
              gblk = 0;
              pin = false;
              texp = T32_INF;
            }
            tev = add_sat32(now, (uint32_t)rec.w);
            st = S_TOOL;
          }
        }
      }
    }
    if (STATS && in_flight && iter_end == now) {
      in_flight = false;
      uint32_t m = __ballot_sync(FULL_MASK, st == S_RUN && fin == n_it);
      while (m) {
        const int p = __ffs(m) - 1;
        m &= m - 1;
        const int pt = __shfl_sync(FULL_MASK, turn, p);
        const int pn = __shfl_sync(FULL_MASK, nturns, p);
        const int pg = __shfl_sync(FULL_MASK, gblk, p);
        --n_run;
        kv_sum -= pg;
        if (lane == p) ctx += rec.x + rec.y;
        if (pt == pn - 1) {  // last request: free its KV (and DRAM copy), the program completes
          free_blk += pg;
          if (EXT) dfree += __shfl_sync(FULL_MASK, dblk, p);
          if (lane == p) { gblk = 0; dblk = 0; st = S_DONE; req = now - arr; }
          ++D;
          turns_done += pn;
        } else {
          int64_t ttl = ttl_fixed;
          if (STATS) {
            const int ptool = __shfl_sync(FULL_MASK, rec.z, p);
            if (pause == CT_PAUSE_FIXED) {
              ttl = simplified_ttl(stats[F], stats[ptool], est, polp->t_pin_us, polp->t_thresh_us);
            } else if (pause == CT_PAUSE_PAPER) {
              // exact path: the cache and the clamp shortcut both measured slower here
              // (P <= 32: few samples per tool row, register pressure)
              ttl = calc_ttl(stats[F], stats[ptool], est, D, turns_done);
            } else if (pause == CT_PAUSE_FITTED) {
              ttl = __ldg(&a.fitted[(int64_t)ptool * a.J + min(pt, a.J - 1)]);
            } else if (EXT && pause == CT_PAUSE_INFERCEPT) {
              // preserve (no TTL) iff the predicted tool time < the swap round trip
              const int64_t pred = infercept_predict(stats[F], stats[ptool], est);
              const uint32_t pctx = __shfl_sync(FULL_MASK, (uint32_t)ctx, p);
              const int64_t blocks = ceil_div_magic(pctx, bsm);
              const int64_t swap = 2 * ceil_ps_to_us((uint64_t)(blocks * E.c_h2d_ps));
              ttl = pred < swap ? CT_INF64 : 0;
            }
          }
          if (ttl > 0) {  // pin_request only if TTL != 0
            if (lane == p) {
              pin = true;
              texp = (EXT && ttl == CT_INF64) ? T32_INF  // InferCept: preserved, no expiry
                     : ttl >= (int64_t)T32_LIM ? T32_LIM : sat32((int64_t)now + ttl + 1);
            }
          } else if (EXT) {
            evict(p);
          } else {  // evict
            free_blk += pg;
            if (lane == p) { gblk = 0; pin = false; texp = T32_INF; }
          }
          if (lane == p) { tev = sat32((int64_t)now + rec.w); st = S_TOOL; }
        }
      }
    }
    if (in_flight) continue;  // mid-iteration: events only mutate Q / pins (R2)

    // ---- scheduling point (R3) --------------------------------------------------------------
    int admitted = 0;
    bool stable = true;
    qleft = false;
    if (__any_sync(FULL_MASK, st == S_QUEUED || (EXT && st == S_READY))) {
      if (EXT) {  // loaded requests join the batch
        const bool join = st == S_READY;
        const uint32_t m = __ballot_sync(FULL_MASK, join);
        if (m) {
          kv_sum += (int32_t)__reduce_add_sync(FULL_MASK, join ? (uint32_t)gblk : 0u);
          pf += (int64_t)__reduce_add_sync(FULL_MASK, join ? (uint32_t)unc : 0u);
          n_run += __popc(m);
          n_load -= __popc(m);
          if (join) { st = S_RUN; fin = sat32((int64_t)n_it + rec.y); }
        }
      }
      for (;;) {  // admit loop (victims PAPER.md:645-655)
        const uint32_t mq = __ballot_sync(FULL_MASK, st == S_QUEUED);
        if (!mq) break;
        if (n_run + n_load >= max_batch) { qleft = true; break; }
        int h;
        if (!STATS || prio == CT_PRIO_PROG_FCFS) {  // pinned-queued first, then queued, by index
          const uint32_t mp = __ballot_sync(FULL_MASK, st == S_QUEUED && pin);
          h = __ffs(mp ? mp : mq) - 1;
        } else {  // REQ_FCFS (vanilla vLLM): earliest request; PLAS (Autellix,
                  // PAPER.md:207): least attained service; ties by index
          const bool q = st == S_QUEUED;
          const uint32_t key = plas ? svc : req;
          const uint32_t mr = __reduce_min_sync(FULL_MASK, q ? key : T32_INF);
          h = __ffs(__ballot_sync(FULL_MASK, q && key == mr)) - 1;
        }
        const int32_t hctx = __shfl_sync(FULL_MASK, ctx, h);
        const int32_t hg = __shfl_sync(FULL_MASK, gblk, h);
        const int32_t hnew = __shfl_sync(FULL_MASK, rec.x, h);
        const int32_t hdec = __shfl_sync(FULL_MASK, rec.y, h);
        // blocks, contexts and token counts are below 2^30 (validated): 32-bit arithmetic
        const int32_t need = (int32_t)ceil_div_magic((uint32_t)(hctx + hnew + hdec), bsm) - hg;
        if (need > free_blk && admitted == 0) {
          while (need > free_blk) {  // victims: latest program arrival first, never the head
            const uint32_t mv = __ballot_sync(FULL_MASK, pin && lane != h);
            if (!mv) break;
            const int v = 31 - __clz(mv);
            if (EXT) {
              evict(v);
            } else {
              free_blk += __shfl_sync(FULL_MASK, gblk, v);
              if (lane == v) { gblk = 0; pin = false; texp = T32_INF; }
            }
            acc_add(ACC_VICT, 1);
          }
        }
        if (need > free_blk) {  // HOL break
          if (admitted > 0 && __ballot_sync(FULL_MASK, pin && lane != h)) stable = false;
          qleft = true;
          break;
        }
        free_blk -= need;
        const int32_t ng = hg + need;
        acc_add(ACC_BUBBLE, (int64_t)(now - __shfl_sync(FULL_MASK, req, h)));
        const bool hp = __shfl_sync(FULL_MASK, pin ? 1 : 0, h) != 0;
        const int32_t hd = dram_on ? __shfl_sync(FULL_MASK, dblk, h) : 0;
        bool loading = false;
        uint32_t ld = 0;
        int32_t cached;
        if (hp) {
          cached = hctx;
          acc_add(ACC_HITS, 1);
        } else if (dram_on && hd > 0 && hd == (int32_t)ceil_div_magic((uint32_t)hctx, bsm)) {
          // the DRAM copy covers the context: load it through the serialized H2D channel
          cached = hctx;
          loading = true;
          ld = sat32((int64_t)max(now, chan) + ceil_ps_to_us((uint64_t)((int64_t)hd * E.c_h2d_ps)));
          chan = ld;
          acc_add(ACC_RELOAD, 1);
        } else {
          cached = 0;
          acc_add(ACC_RECOMP, hctx);
        }
        const int32_t u = hctx + hnew - cached;  // < 2^31
        acc_add(ACC_PREFILL, u);
        if (lane == h) {
          pin = false;
          texp = T32_INF;
          gblk = ng;
          if (EXT && loading) {
            st = S_LOAD;
            tev = ld;
            unc = (int32_t)u;
          } else {
            st = S_RUN;
            fin = STATS ? sat32((int64_t)n_it + rec.y) : add_sat32(n_it, (uint32_t)rec.y);
          }
        }
        if (EXT && loading) {
          ++n_load;
        } else {
          ++n_run;
          kv_sum += ng;
          pf += u;
        }
        ++admitted;
      }
      // unschedulable: the head missed with nothing running or loading (C-5 5c)
      if (admitted == 0 && n_run == 0 && n_load == 0 && __any_sync(FULL_MASK, st == S_QUEUED)) {
        status = CT_R_UNSCHEDULABLE;
        break;
      }
    }
    // start the next iteration(s) (linear cost model, R16)
    if (n_run > 0) {
      if (kv_sum != kv_at) {
        kv_at = kv_sum;
        d_cur = iter_us_kv32(a, (uint32_t)kv_sum, &rb_cur);  // < 2^31 (host-checked)
        rd_cur = rcp_approx((float)d_cur);  // estimate only: macro_iters32 corrects
      }
      const int64_t dur1 = pf <= 0 ? d_cur : iter_us_prefill(a, d_cur, rb_cur, (uint32_t)kv_sum, pf);
      pf = 0;
      // every end below is checked against the 32-bit horizon (else: the 64-bit path replays
      // the replica), so the macro-step is computed on 32-bit times
      if (dur1 >= (int64_t)(T32_LIM - now)) return false;
      const uint32_t end1 = now + (uint32_t)dur1;
      uint32_t kk = 0;  // iterations of d_cur after the first one
      if (stable) {
        const uint32_t mfin = __reduce_min_sync(FULL_MASK, st == S_RUN ? fin : T32_INF);
        const uint32_t te = __reduce_min_sync(FULL_MASK, qleft ? min(tev, texp) : tev);
        kk = extra_iters32(mfin - n_it - 1, te, end1, d_cur, rd_cur);
      }
      const uint64_t end = (uint64_t)end1 + (uint64_t)kk * d_cur;
      if (STATS ? (uint64_t)n_it + kk + 1 > it_cap : kk >= it_cap - n_it) {  // n_it + kk + 1 > it_cap
        status = CT_R_EVENT_BUDGET;
        break;
      }
      if (end >= T32_LIM) return false;  // beyond the 32-bit horizon
      const uint32_t dur = (uint32_t)end - now;
      n_it += kk + 1;
      iter_end = (uint32_t)end;
      acc_add(ACC_BUSY, dur);
      if (plas && st == S_RUN) svc += dur;  // every running request accrues the iterations
      in_flight = true;
    }
  }
  if (!STATS) {
    D = __popc(__ballot_sync(FULL_MASK, st == S_DONE));
    turns_done = (int32_t)__reduce_add_sync(FULL_MASK, st == S_DONE ? (uint32_t)nturns : 0u);
  }
  if (status == CT_R_OK && D != P) status = CT_R_UNSCHEDULABLE;

  // ---- per-replica summary (A-8) --------------------------------------------------------------
  const int64_t ri = r - a.r_begin;
  int64_t jsum = 0, jmax = 0, p50 = 0, p99 = 0;
  if (status == CT_R_OK) {
    const uint32_t jv = live ? req : 0;
    jsum = (int64_t)__reduce_add_sync(FULL_MASK, jv >> 16) * 65536 +
           (int64_t)__reduce_add_sync(FULL_MASK, jv & 0xFFFFu);
    jmax = __reduce_max_sync(FULL_MASK, jv);
    const int r50 = (50 * P + 99) / 100, r99 = (99 * P + 99) / 100;
    int lt = 0, le = 0;
    for (int q = 0; q < P; ++q) {
      const uint32_t x = __shfl_sync(FULL_MASK, req, q);
      lt += x < req;
      le += x <= req;
    }
    const bool c5 = live && lt < r50 && r50 <= le, c9 = live && lt < r99 && r99 <= le;
    p50 = __shfl_sync(FULL_MASK, req, __ffs(__ballot_sync(FULL_MASK, c5)) - 1);
    p99 = __shfl_sync(FULL_MASK, req, __ffs(__ballot_sync(FULL_MASK, c9)) - 1);
  }
  int64_t av[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) av[k] = STATS ? shfl64(accv, k) : k >= ACC_BUSY ? (int64_t)A32[k] : A[k];
  if (lane == 0) {
    ct_replica_summary o;
    if (status == CT_R_OK) {
      o.status = status;
      o.n_done = D;
      o.turns_done = turns_done;
      o.sum_jct_us = jsum;
      o.max_jct_us = jmax;
      o.p50_jct_us = p50;
      o.p99_jct_us = p99;
      o.sum_bubble_us = av[ACC_BUBBLE];
      o.makespan_us = now;  // the last event processed is the last completion; origin = arr0
      o.iterations = n_it;
      o.busy_us = av[ACC_BUSY];
      o.prefill_tokens = av[ACC_PREFILL];
      o.recompute_tokens = av[ACC_RECOMP];
      o.pin_hits = av[ACC_HITS];
      o.pin_expiries = av[ACC_EXP];
      o.victims = av[ACC_VICT];
      o.reloads = av[ACC_RELOAD];
    } else {
      int64_t* w = (int64_t*)&o;
#pragma unroll
      for (int i = 0; i < 16; ++i) w[i] = 0;
      o.status = status;
    }
    a.out[ri] = o;
  }
  if (a.jct && live) a.jct[ri * P + lane] = status == CT_R_OK ? (int64_t)req : -1;
  __syncwarp();
  return true;
}

// -----------------------------------------------------------------------------------------------
// 32 < P <= 256: program p lives on lane p % 32, slot p / 32.  Per-program scalars are SoA in
// shared memory (written only by the owner lane); lifecycle sets are per-lane bit registers
// (bit s = slot s); every lane caches the minimum of its own programs' event times (tool return /
// load done, pin expiry) and of their finishing iterations, refreshed only when one of its
// programs changes.  The next event, the macro-step bound and the first finish are therefore one
// REDUX minimum each, and only lanes that own a due program scan their slots.  Same semantics as
// replay_one_w32 (C-5/C-6), checked byte for byte by the tests.
// PROG: the policy is in the program-FCFS class (prog_policy(), ct_internal.h): request FCFS,
// PLAS, the DRAM tier, InferCept and the alternative readings compile away.
template <int NS, bool VLLM, bool PROG>
__device__ __forceinline__ void replay_one_ns(const ReplayArgs& a, int64_t r, unsigned char* wm,
                                              int lane) {
  constexpr int PM = 32 * NS;
  int64_t* tev = (int64_t*)wm;         // tool return / load done, INF otherwise
  int64_t* texp = tev + PM;            // expiry + 1 while pinned in a tool call, INF otherwise
  int64_t* req = texp + PM;            // request arrival; JCT once done
  int64_t* fin = req + PM;             // finishing iteration while running, INF otherwise
  // PROG keeps no svc / dblk arrays (never read): 48 instead of 60 B per program
  int64_t* svc = fin + PM;             // attained engine time (PLAS)
  int32_t* ctx = (int32_t*)(svc + (PROG ? 0 : PM)); // context tokens
  int32_t* gblk = ctx + PM;            // GPU blocks held
  int32_t* dblk = gblk + PM;           // DRAM copy blocks
  int32_t* unc = dblk + (PROG ? 0 : PM);  // uncached tokens of the current request
  int32_t* turn = unc + PM;            // current turn
  // vLLM engine (NEXT-2) only.  KV growth (R27-R30): next iteration boundary at which the
  // running request needs one more block (INF otherwise) and tokens emitted before a
  // preemption.  Chunked prefill (R31-R32): prompt tokens of the current request not computed.
  const bool grow_on = VLLM && a.eng.kv_growth != 0;
  const bool chunk_on = VLLM && a.eng.prefill_chunk > 0;
  int64_t* grow_at = (int64_t*)(turn + PM);
  int32_t* emt = (int32_t*)(grow_at + PM);
  int32_t* prem = emt + PM;
  Stat* stats = (Stat*)(wm + (((VLLM ? 76 : PROG ? 48 : 60) * PM + 15) & ~15));
  Acc* acc = (Acc*)(stats + a.F + 1);

  const int P = a.P, F = a.F;
  const int64_t npol = a.n_pol, nkv = a.n_kv, nrate = a.n_rate;
  const int pol_i = (int)(r % npol);
  const int kv_i = (int)((r / npol) % nkv);
  const int rate_i = (int)((r / (npol * nkv)) % nrate);
  const int64_t seed = r / (npol * nkv * nrate);
  const ct_policy* polp = a.pols + pol_i;
  const int prio = PROG ? CT_PRIO_PROG_FCFS : polp->priority;
  const int pause = polp->pause;
  const int pflags = PROG ? 0 : polp->flags;
  const int64_t gap = a.gap[rate_i];
  const ct_program* prog = a.progs + seed * P;
  const ct_engine_params& E = a.eng;
  const ct_estimator_params& est = a.est;
  const int64_t bs = E.bs;
  DivMagic bsm;
  bsm.mhi = (uint32_t)(a.bs_magic >> 32);
  bsm.mlo = (uint32_t)a.bs_magic;
  bsm.dm1 = (uint32_t)(bs - 1);
  bsm.ident = bs == 1 ? 1u : 0u;
  const bool eager = (pflags & CT_FLAG_STEP_EXPIRY) == 0;
  const bool vany = (pflags & CT_FLAG_VICTIMS_ANY) != 0;
  const bool dram_on = !PROG && polp->dram != 0 && E.dram_blocks > 0;
  const bool need_stats = pause == CT_PAUSE_PAPER || (!PROG && pause == CT_PAUSE_INFERCEPT) ||
                          (pause == CT_PAUSE_FIXED && polp->t_thresh_us != CT_ALWAYS);
  const bool plas = !PROG && prio == CT_PRIO_PLAS;

#pragma unroll
  for (int s = 0; s < NS; ++s) {
    const int p = lane + 32 * s;
    tev[p] = CT_INF64;
    texp[p] = CT_INF64;
    req[p] = 0;
    fin[p] = CT_INF64;
    if (!PROG) svc[p] = 0;
    ctx[p] = 0;
    gblk[p] = 0;
    if (!PROG) dblk[p] = 0;
    unc[p] = 0;
    turn[p] = 0;
    if (VLLM) {
      grow_at[p] = CT_INF64;
      emt[p] = 0;
      prem[p] = 0;
    }
  }
  // per-program bubble series (NEXT-3): accumulated in place by the owner lane
  int64_t* bub = a.bubble ? a.bubble + (r - a.r_begin) * P : nullptr;
  if (bub) {
#pragma unroll
    for (int s = 0; s < NS; ++s)
      if (lane + 32 * s < P) bub[lane + 32 * s] = 0;
  }
  if (need_stats)
    for (int i = lane; i < 4 * (F + 1); i += 32) ((int64_t*)stats)[i] = 0;
  if (lane == 0) *acc = Acc{0, 0, 0, 0, 0, 0, 0, 0};
  __syncwarp();

  // per-lane sets over this lane's slots and cached minima
  uint32_t qb = 0, pb = 0, rb = 0, lb = 0, yb = 0, tb = 0;
  uint32_t xb = 0;  // preempted (KV growth)
  int64_t lev = CT_INF64, lexp = CT_INF64, fmin = CT_INF64;
  int64_t gmin = CT_INF64;  // cached minimum of grow_at over this lane's programs
  auto own = [&](int p) { return lane == (p & 31); };
  auto bit = [&](int p) { return 1u << (p >> 5); };
  auto turn_rec = [&](int p, int t) -> int4 { return __ldg(&a.turns[prog[p].turn0 + t]); };
  auto arrival = [&](int i) -> int64_t { return (prog[i].arr_q * gap) >> 20; };
  // Visit the programs whose bit is set in the per-lane slot mask `m` in program-index order
  // (slot-major, lane-minor), skipping empty slots with one REDUX.OR.
  auto for_each_set = [&](uint32_t m, auto&& fn) {
    uint32_t slots = __reduce_or_sync(FULL_MASK, m);
    while (slots) {
      const int s = __ffs(slots) - 1;
      slots &= slots - 1;
      uint32_t b = __ballot_sync(FULL_MASK, (m >> s) & 1u);
      while (b) {
        const int p = 32 * s + __ffs(b) - 1;
        b &= b - 1;
        fn(p);
      }
    }
  };
  auto rescan_lev = [&]() {
    int64_t m = CT_INF64;
#pragma unroll
    for (int s = 0; s < NS; ++s) m = min(m, tev[lane + 32 * s]);
    lev = m;
  };
  auto rescan_lexp = [&]() {
    int64_t m = CT_INF64;
#pragma unroll
    for (int s = 0; s < NS; ++s) m = min(m, texp[lane + 32 * s]);
    lexp = m;
  };
  auto rescan_fmin = [&]() {
    int64_t m = CT_INF64;
#pragma unroll
    for (int s = 0; s < NS; ++s) m = min(m, fin[lane + 32 * s]);
    fmin = m;
  };
  auto rescan_gmin = [&]() {
    int64_t m = CT_INF64;
#pragma unroll
    for (int s = 0; s < NS; ++s) m = min(m, grow_at[lane + 32 * s]);
    gmin = m;
  };
  // Priority among running requests (R28): program index (program FCFS), else (request
  // arrival | attained service, index); pick_best = highest priority, pick_worst = lowest.
  auto run_key = [&](int p) -> int64_t { return plas ? svc[p] : req[p]; };
  auto pick_best = [&](uint32_t m) -> int {
    if (prio == CT_PRIO_PROG_FCFS) {
      const uint32_t slots = __reduce_or_sync(FULL_MASK, m);
      const int s0 = __ffs(slots) - 1;
      return 32 * s0 + __ffs(__ballot_sync(FULL_MASK, (m >> s0) & 1u)) - 1;
    }
    int64_t bk = CT_INF64;
    int bp = 0x7fffffff;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const int pl = lane + 32 * s;
      if ((m >> s) & 1u) {
        const int64_t k = run_key(pl);
        if (k < bk) { bk = k; bp = pl; }
      }
    }
    const int64_t mk = warp_min64_redux(bk);
    return (int)__reduce_min_sync(FULL_MASK, (uint32_t)(bk == mk ? bp : 0x7fffffff));
  };
  auto pick_worst = [&](uint32_t m) -> int {
    if (prio == CT_PRIO_PROG_FCFS) {
      const uint32_t slots = __reduce_or_sync(FULL_MASK, m);
      const int s1 = 31 - __clz(slots);
      return 32 * s1 + 31 - __clz(__ballot_sync(FULL_MASK, (m >> s1) & 1u));
    }
    int64_t wk = -1;
    int wp = -1;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const int pl = lane + 32 * s;
      if ((m >> s) & 1u) {
        const int64_t k = run_key(pl);
        if (k >= wk) { wk = k; wp = pl; }  // later slot = higher index wins ties
      }
    }
    const int64_t mk = warp_max64(wk);
    return (int)__reduce_max_sync(FULL_MASK, (uint32_t)(wk == mk ? wp + 1 : 0)) - 1;
  };

  int64_t now = 0, iter_end = 0, n_it = 0, busy = 0;
  bool in_flight = false;
  int64_t free_blk = a.kv[kv_i];
  int64_t dfree = dram_on ? E.dram_blocks : 0, chan = 0;
  int next_arr = 0;
  const int64_t arr0 = arrival(0);
  int64_t t_arr = arr0;
  int32_t D = 0, turns_done = 0;
  int n_run = 0, n_load = 0;  // n_load counts LOADING and READY
  int64_t kv_sum = 0, pf = 0;
  int status = CT_R_OK;
  int64_t kv_at = -1, d_cur = 0, base_ps = 0;  // base_ps = c0 + c_kv bs kv_sum (ps)
  float rd_cur = 0.0f;

  // evict(v): free its GPU blocks, DRAM write-through when the tier is on (R18); unpin.  Uniform.
  auto evict_unpin = [&](int v) {
    const int64_t g = gblk[v];
    free_blk += g;
    int32_t keep = 0;
    if (dram_on) {
      const int64_t nb = ceil_div_magic((uint32_t)ctx[v], bsm);
      dfree += dblk[v];
      if (nb > 0 && nb <= dfree) { keep = (int32_t)nb; dfree -= nb; }
    }
    __syncwarp();  // every lane has read v's fields before the owner rewrites them
    if (own(v)) {
      gblk[v] = 0;
      if (dram_on) dblk[v] = keep;
      if (pb & bit(v)) {
        pb &= ~bit(v);
        if (texp[v] != CT_INF64) { texp[v] = CT_INF64; rescan_lexp(); }
      }
    }
    __syncwarp();
  };
  // owner: first boundary after n_it at which a running request holding ceil(x / bs) blocks
  // for x tokens needs another one (R27); INF when it finishes first
  auto set_grow = [&](int p, int64_t x, int64_t fp) {
    const int64_t B = (int64_t)ceil_div_magic((uint32_t)x, bsm);
    const int64_t nx = n_it + (B * bs - x) + 1;
    grow_at[p] = nx < fp ? nx : CT_INF64;
    gmin = min(gmin, grow_at[p]);
  };
  // vLLM recompute preemption of running request v (R28): its GPU KV is dropped and it
  // re-enters Q marked preempted, remembering the tokens it has emitted.  Uniform.
  auto preempt = [&](int v) {
    const int64_t g = gblk[v];
    const int64_t fv = fin[v];
    const int dec = turn_rec(v, turn[v]).y;
    free_blk += g;
    kv_sum -= g;
    --n_run;
    __syncwarp();
    if (own(v)) {
      rb &= ~bit(v);
      qb |= bit(v);
      xb |= bit(v);
      emt[v] = (int32_t)(dec - (fv - n_it));
      fin[v] = CT_INF64;
      grow_at[v] = CT_INF64;
      gblk[v] = 0;
      req[v] = now;
    }
    __syncwarp();
  };

  for (;;) {
    // ---- next event (R1, R3) --------------------------------------------------------------
    // In flight: every event up to iter_end is applied in one pass at the boundary (as in
    // replay_one_w32: effects commute, DRAM write-through in (time, index) order).
    int64_t t;
    if (in_flight) {
      t = iter_end;
    } else {
      t = min(warp_min64_redux(eager ? min(lev, lexp) : lev), t_arr);
      if (t == CT_INF64) break;
    }
    now = t;

    {
      // PinExpiry (EAGER): first µs with now > expiry while not in Q (R4/R15);
      // it precedes the program's own tool return at the same µs (R1)
      if (eager && __any_sync(FULL_MASK, lexp <= now)) {
        uint32_t me = 0;
        if (lexp <= now) {
#pragma unroll
          for (int s = 0; s < NS; ++s) {
            const int p = lane + 32 * s;
            me |= (texp[p] <= now && texp[p] <= tev[p] ? 1u : 0u) << s;
          }
        }
        const uint32_t cnt = __reduce_add_sync(FULL_MASK, (uint32_t)__popc(me));
        if (lane == 0) acc->exp += cnt;
        if (dram_on) {  // write-through order matters: (time, index)
          while (__any_sync(FULL_MASK, me != 0)) {
            int64_t lm = CT_INF64;
#pragma unroll
            for (int s = 0; s < NS; ++s)
              if ((me >> s) & 1u) lm = min(lm, texp[lane + 32 * s]);
            const int64_t tm = warp_min64_redux(lm);
            uint32_t mt = 0;
#pragma unroll
            for (int s = 0; s < NS; ++s)
              mt |= (((me >> s) & 1u) && texp[lane + 32 * s] == tm ? 1u : 0u) << s;
            me &= ~mt;
            for_each_set(mt, [&](int p) { evict_unpin(p); });
          }
        } else {
          for_each_set(me, [&](int p) { evict_unpin(p); });
        }
      }
      // ToolReturn (OnRequestArrive of a seen program) and LoadDone
      if (__any_sync(FULL_MASK, lev <= now)) {
        uint32_t md = 0;
        if (lev <= now) {
#pragma unroll
          for (int s = 0; s < NS; ++s) md |= (tev[lane + 32 * s] <= now ? 1u : 0u) << s;
        }
        const uint32_t mret = md & tb, mld = md & lb;
        if (need_stats) {
          for_each_set(mret, [&](int p) {  // estimator rows: Δ_obs = dur of the finished turn (R5)
              const int4 tr = turn_rec(p, turn[p]);
              const int64_t x = min((int64_t)tr.w, est.b_us);
              const uint64_t x2 = (uint64_t)x * (uint64_t)x;
              if (lane == 0) {
                Stat* rows[2] = {&stats[F], &stats[tr.z]};
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                  Stat* q = rows[k];
                  q->n += 1;
                  q->s1 += x;
                  const uint64_t lo = q->s2lo + x2;
                  q->s2hi += (lo < x2);
                  q->s2lo = lo;
                }
              }
              __syncwarp();
          });
        }
        if (md) {
          bool rescan_e = false;
#pragma unroll
          for (int s = 0; s < NS; ++s) {
            const int p = lane + 32 * s;
            if ((mret >> s) & 1u) {
              turn[p] += 1;
              req[p] = tev[p];  // the event's own instant
              tev[p] = CT_INF64;
              if (texp[p] != CT_INF64) { texp[p] = CT_INF64; rescan_e = true; }  // retained pin
            }
            if ((mld >> s) & 1u) tev[p] = CT_INF64;
          }
          qb |= mret;
          tb &= ~mret;
          yb |= mld;
          lb &= ~mld;
          rescan_lev();
          if (rescan_e) rescan_lexp();
        }
        __syncwarp();
      }
    }
    // ProgramArrival (programs arrive in index order)
    while (t_arr <= now) {
      const int p = next_arr;
      if (own(p)) { qb |= bit(p); req[p] = t_arr; }
      ++next_arr;
      t_arr = next_arr < P ? arrival(next_arr) : CT_INF64;
    }
    __syncwarp();

    // IterationEnd: requests whose last token was emitted finish, in index order (C-6)
    if (in_flight && iter_end == now) {
      in_flight = false;
      uint32_t mf = 0;
      if (fmin == n_it) {
#pragma unroll
        for (int s = 0; s < NS; ++s) mf |= (fin[lane + 32 * s] == n_it ? 1u : 0u) << s;
      }
      for_each_set(mf, [&](int p) {
          // OnRequestFinish
          const int tp = turn[p];
          const int4 tr = turn_rec(p, tp);
          const int nctx = ctx[p] + tr.x + tr.y;
          const int64_t g = gblk[p];
          --n_run;
          kv_sum -= g;
          __syncwarp();
          if (own(p)) { rb &= ~bit(p); fin[p] = CT_INF64; ctx[p] = nctx; }
          __syncwarp();
          const int nt = prog[p].nturns;
          if (tp == nt - 1) {  // last request: free its KV, the program completes
            free_blk += g;
            if (!PROG) dfree += dblk[p];
            __syncwarp();
            if (own(p)) {
              gblk[p] = 0;
              if (!PROG) dblk[p] = 0;
              req[p] = now - arrival(p);
            }
            ++D;
            turns_done += nt;
            __syncwarp();
          } else {
            const int f = tr.z;
            int64_t ttl = 0;
            switch (pause) {
              case CT_PAUSE_FIXED:
              case CT_PAUSE_PAPER: {
                const Stat sg = stats[F], sf = stats[f];
                ttl = pause == CT_PAUSE_PAPER
                          ? calc_ttl(sg, sf, est, D, turns_done)
                          : simplified_ttl(sg, sf, est, polp->t_pin_us, polp->t_thresh_us);
                break;
              }
              case CT_PAUSE_FITTED:
                ttl = __ldg(&a.fitted[(int64_t)f * a.J + min(tp, a.J - 1)]);
                break;
              case CT_PAUSE_INFERCEPT: {  // preserve (no TTL) iff prediction < swap round trip
                const int64_t pred = infercept_predict(stats[F], stats[f], est);
                const int64_t blocks = ceil_div_magic((uint32_t)nctx, bsm);
                const int64_t swap = 2 * ceil_ps_to_us((uint64_t)(blocks * E.c_h2d_ps));
                ttl = pred < swap ? CT_INF64 : 0;
                break;
              }
              default:
                ttl = 0;
            }
            if (ttl > 0) {  // pin_request only if TTL != 0
              if (own(p)) {
                pb |= bit(p);
                if (ttl != CT_INF64) { texp[p] = now + ttl + 1; lexp = min(lexp, texp[p]); }
              }
            } else {
              evict_unpin(p);
            }
            if (own(p)) { tev[p] = now + tr.w; lev = min(lev, tev[p]); tb |= bit(p); }
            __syncwarp();
          }
      });
      if (mf) rescan_fmin();
    }
    if (in_flight) continue;  // mid-iteration: events only mutate Q / stats / pins (R2)

    // ---- scheduling point (R3) --------------------------------------------------------------
    // (a) STEP reading: release expired pins of programs not waiting
    if (!eager) {
      uint32_t mx = 0;
      if (lexp <= now) {
#pragma unroll
        for (int s = 0; s < NS; ++s) mx |= ((((pb & tb) >> s) & 1u) && texp[lane + 32 * s] <= now ? 1u : 0u) << s;
      }
      const uint32_t cnt = __reduce_add_sync(FULL_MASK, (uint32_t)__popc(mx));
      if (lane == 0) acc->exp += cnt;
      for_each_set(mx, [&](int p) { evict_unpin(p); });
    }
    // (a2) KV growth (NEXT-2, R27/R28): running requests that need a block for their next
    // token, best-ranked first; when the pool is dry the worst-ranked running request is
    // preempted (possibly the requester itself)
    if (grow_on && __any_sync(FULL_MASK, gmin <= n_it)) {
      uint32_t mg = 0;
      if (gmin <= n_it) {
#pragma unroll
        for (int s = 0; s < NS; ++s) mg |= (grow_at[lane + 32 * s] == n_it ? 1u : 0u) << s;
      }
      for (;;) {
        mg &= rb;  // drop candidates preempted as victims
        if (!__any_sync(FULL_MASK, mg != 0)) break;
        const int i = pick_best(mg);
        if (own(i)) mg &= ~bit(i);
        bool alive = true;
        while (free_blk < 1) {
          const int v = pick_worst(rb);
          preempt(v);
          if (v == i) { alive = false; break; }
        }
        if (alive) {
          --free_blk;
          ++kv_sum;
          if (own(i)) {
            gblk[i] += 1;
            const int64_t nx = n_it + bs;  // the next block boundary is bs tokens later
            grow_at[i] = nx < fin[i] ? nx : CT_INF64;
          }
        }
        __syncwarp();
      }
      rescan_gmin();
      rescan_fmin();
    }
    int admitted = 0;
    bool stable = true;
    int64_t left = 1;  // token budget left in this iteration (chunked prefill)
    // (b) loaded requests join the batch
    auto join_ready = [&]() {
      const uint32_t cnt = __reduce_add_sync(FULL_MASK, (uint32_t)__popc(yb));
      {
        int64_t lk = 0, lp = 0;
#pragma unroll
        for (int s = 0; s < NS; ++s) {
          if ((yb >> s) & 1u) {
            const int p = lane + 32 * s;
            const int4 tj = turn_rec(p, turn[p]);
            if (grow_on) {  // a preempted request reloaded from DRAM resumes after emt tokens
              const int32_t e = emt[p];
              fin[p] = n_it + tj.y - e;
              emt[p] = 0;
              set_grow(p, (int64_t)ctx[p] + tj.x + e + 1, fin[p]);
            } else if (chunk_on) {  // its prompt is computed in chunks from (b2) on
              prem[p] = unc[p];
              fin[p] = CT_INF64;
            } else {
              fin[p] = n_it + tj.y;
            }
            fmin = min(fmin, fin[p]);
            lk += gblk[p];
            lp += unc[p];
          }
        }
        rb |= yb;
        yb = 0;
        kv_sum += (int64_t)warp_sum_u64((uint64_t)lk);
        if (!chunk_on) pf += (int64_t)warp_sum_u64((uint64_t)lp);
        n_run += cnt;
        n_load -= cnt;
      }
    };
    if (chunk_on) {  // loaded requests join first: (b2) shares the budget among all running
      if (__any_sync(FULL_MASK, yb != 0)) join_ready();
      // (b2) chunked prefill (R31/R32): one token per decoding request, then the prefilling
      // running requests, best-ranked first, take min(remaining prompt, budget left)
      uint32_t nd = 0, mp = 0;
#pragma unroll
      for (int s = 0; s < NS; ++s)
        if ((rb >> s) & 1u) {
          if (prem[lane + 32 * s] == 0) ++nd; else mp |= 1u << s;
        }
      left = E.prefill_chunk - (int64_t)__reduce_add_sync(FULL_MASK, nd);
      while (__any_sync(FULL_MASK, mp != 0)) {
        const int i = pick_best(mp);
        const int64_t c = min((int64_t)prem[i], max(left, (int64_t)0));
        left -= c;
        pf += c;
        __syncwarp();
        if (own(i)) {
          mp &= ~bit(i);
          prem[i] -= (int32_t)c;
          if (prem[i] == 0) {  // the prompt completes in this iteration, which emits token 1
            fin[i] = n_it + turn_rec(i, turn[i]).y;
            fmin = min(fmin, fin[i]);
          }
        }
        __syncwarp();
      }
    }
    if (__any_sync(FULL_MASK, (qb | yb) != 0)) {
      if (__any_sync(FULL_MASK, yb != 0)) join_ready();
      // (c) admit loop (victims PAPER.md:645-655)
      for (;;) {
        if (!__any_sync(FULL_MASK, qb != 0)) break;
        if (n_run + n_load >= E.max_batch) break;
        if (chunk_on && left <= 0) {  // R32: no token budget left in this iteration; the next
          stable = false;             // boundary has a fresh budget, so it must be a step
          break;
        }
        int h = -1;
        // preempted requests rank first (R29); only KV growth preempts
        const bool any_x = grow_on && __any_sync(FULL_MASK, (qb & xb) != 0);
        const uint32_t cq = any_x ? (qb & xb) : qb;
        if (prio == CT_PRIO_PROG_FCFS) {  // lowest index among pinned-queued, else queued
          uint32_t sel = any_x ? cq : (qb & pb);
          uint32_t slots = __reduce_or_sync(FULL_MASK, sel);
          if (!slots) { sel = qb; slots = __reduce_or_sync(FULL_MASK, sel); }
          const int s0 = __ffs(slots) - 1;
          h = 32 * s0 + __ffs(__ballot_sync(FULL_MASK, (sel >> s0) & 1u)) - 1;
        } else {  // REQ_FCFS: earliest request; PLAS: least attained service; ties: index
          int64_t bk = CT_INF64;
          int bp = 0x7fffffff;
#pragma unroll
          for (int s = 0; s < NS; ++s) {
            const int pl = lane + 32 * s;
            if ((cq >> s) & 1u) {
              const int64_t k = plas ? svc[pl] : req[pl];
              if (k < bk) { bk = k; bp = pl; }
            }
          }
          const int64_t mk = warp_min64_redux(bk);
          const int cand = bk == mk ? bp : 0x7fffffff;
          h = (int)__reduce_min_sync(FULL_MASK, (uint32_t)cand);
        }
        const int4 tr = turn_rec(h, turn[h]);
        const int64_t hctx = ctx[h];
        const int64_t hg = gblk[h];
        // R12: reserve the whole request; R27/R30 (growth): up to the slot of its next token
        const int32_t he = grow_on ? emt[h] : 0;
        const bool hx = grow_on && ((__shfl_sync(FULL_MASK, xb, h & 31) >> (h >> 5)) & 1u);
        const int64_t need =
            (int64_t)ceil_div_magic((uint32_t)(hctx + tr.x + (grow_on ? he + 1 : tr.y)), bsm) - hg;
        if (need > free_blk && (admitted == 0 || vany)) {
          while (need > free_blk) {  // victims: latest program arrival first, never the head
            const uint32_t cand = pb & ~(own(h) ? bit(h) : 0u);
            const uint32_t slots = __reduce_or_sync(FULL_MASK, cand);
            if (!slots) break;
            const int s1 = 31 - __clz(slots);
            const int v = 32 * s1 + 31 - __clz(__ballot_sync(FULL_MASK, (cand >> s1) & 1u));
            evict_unpin(v);
            if (lane == 0) acc->vict += 1;
          }
        }
        if (need > free_blk) {  // HOL break
          if (admitted > 0 && !vany &&
              __reduce_or_sync(FULL_MASK, pb & ~(own(h) ? bit(h) : 0u)))
            stable = false;
          break;
        }
        // issue h
        free_blk -= need;
        const int32_t ng = (int32_t)(hg + need);
        if (lane == 0) acc->bubble += now - req[h];
        if (bub && own(h)) bub[h] += now - req[h];
        const bool hp = (__shfl_sync(FULL_MASK, pb, h & 31) >> (h >> 5)) & 1u;
        const int64_t hd = PROG ? 0 : dblk[h];
        int64_t cached;
        bool loading = false;
        int64_t ld = 0;
        if (hp) {
          cached = hctx;
          if (lane == 0) acc->hits += 1;
        } else if (dram_on && hd > 0 && hd == (int64_t)ceil_div_magic((uint32_t)hctx, bsm)) {
          cached = hctx;
          loading = true;
          ld = max(now, chan) + ceil_ps_to_us((uint64_t)(hd * E.c_h2d_ps));
          chan = ld;
          if (lane == 0) acc->reload += 1;
        } else {
          cached = 0;
        }
        // recomputed: context without a cached copy + (R30) what a preemption dropped
        if (lane == 0) acc->recomp += hctx - cached + (hx ? tr.x + he : 0);
        const int64_t u = hctx + tr.x + he - cached;
        if (lane == 0) acc->prefill += u;
        __syncwarp();  // every lane has read h's fields before the owner rewrites them
        if (own(h)) {
          qb &= ~bit(h);
          pb &= ~bit(h);  // a queued pin has no pending expiry (cleared at its return)
          xb &= ~bit(h);
          gblk[h] = ng;
          unc[h] = (int32_t)u;
          if (loading) {
            lb |= bit(h);
            tev[h] = ld;
            lev = min(lev, ld);
          } else {
            rb |= bit(h);
            fin[h] = n_it + tr.y - he;
            if (grow_on) {
              emt[h] = 0;
              set_grow(h, hctx + tr.x + he + 1, fin[h]);
            }
            if (chunk_on) {  // R32: a newcomer takes what is left of the budget
              prem[h] = (int32_t)(u - min(u, left));
              if (prem[h] > 0) fin[h] = CT_INF64;
            }
            fmin = min(fmin, fin[h]);
          }
        }
        if (loading) {
          ++n_load;
        } else {
          ++n_run;
          kv_sum += ng;
          if (chunk_on) {
            const int64_t c = min(u, left);
            pf += c;
            left -= u > 0 ? c : 1;  // a fully cached request decodes: one token
          } else {
            pf += u;
          }
        }
        ++admitted;
        __syncwarp();
      }
      // (d) unschedulable: the head missed with nothing running or loading; the victim loop
      // has already released every other pin, so no future event can free memory (C-5 5c)
      if (admitted == 0 && n_run == 0 && n_load == 0 && __any_sync(FULL_MASK, qb != 0)) {
        status = CT_R_UNSCHEDULABLE;
        break;
      }
    }
    // (e) start the next iteration(s) (linear cost model, R16)
    if (n_run > 0) {
      if (chunk_on && stable) {  // a prompt still in progress makes the next boundary a step
        bool pending = false;
#pragma unroll
        for (int s = 0; s < NS; ++s) pending |= ((rb >> s) & 1u) && prem[lane + 32 * s] > 0;
        if (__any_sync(FULL_MASK, pending)) stable = false;
      }
      if (kv_sum != kv_at) {
        kv_at = kv_sum;
        base_ps = E.c0_ps + E.c_kv_ps * bs * kv_sum;
        d_cur = ceil_ps_to_us((uint64_t)base_ps);
        rd_cur = rcp_approx((float)d_cur);  // estimate only: macro_iters32 corrects
      }
      const int64_t d = d_cur;
      // the first iteration carries the prefill of newly admitted requests (R16)
      const int64_t dur1 = pf > 0 ? ceil_ps_to_us((uint64_t)(base_ps + E.c_pf_ps * pf)) : d;
      pf = 0;
      int64_t k = 1;
      if (stable) {
        // macro-step: the first iteration plus identical decode iterations, up to the first
        // finish or the first boundary at or after the next external event
        const int64_t mfin = warp_min64_redux(grow_on ? min(fmin, gmin) : fmin);
        const int64_t te = min(warp_min64_redux(min(lev, lexp)), t_arr);
        k = a.d32 ? macro_iters32(mfin - n_it, te - now, dur1, (uint32_t)d, rd_cur)
                  : macro_iters(mfin - n_it, te - now, dur1, d, rd_cur);
      }
      const int64_t dur = dur1 + (k - 1) * d;
      if (n_it + k > E.max_iters) { status = CT_R_EVENT_BUDGET; break; }
      n_it += k;
      iter_end = now + dur;
      busy += dur;
      if (plas) {
#pragma unroll
        for (int s = 0; s < NS; ++s)
          if ((rb >> s) & 1u) svc[lane + 32 * s] += dur;  // owners accrue their running programs
      }
      in_flight = true;
    }
  }
  if (status == CT_R_OK && D != P) status = CT_R_UNSCHEDULABLE;

  // ---- per-replica summary (A-8) --------------------------------------------------------------
  __syncwarp();
  const int64_t ri = r - a.r_begin;
  int64_t jsum = 0, jmax = 0, p50 = 0, p99 = 0;
  if (status == CT_R_OK) {
    int64_t ls = 0, lm = 0;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const int p = lane + 32 * s;
      if (p < P) { ls += req[p]; lm = max(lm, req[p]); }
    }
    jsum = (int64_t)warp_sum_u64((uint64_t)ls);
    jmax = warp_max64(lm);
    // nearest rank (R20): value v with #(x < v) < rank <= #(x <= v)
    const int r50 = (50 * P + 99) / 100, r99 = (99 * P + 99) / 100;
    int64_t c50 = CT_INF64, c99 = CT_INF64;
#pragma unroll 1
    for (int s = 0; s < NS; ++s) {
      const int p = lane + 32 * s;
      if (p < P) {
        const int64_t v = req[p];
        int lt = 0, le = 0;
        for (int q = 0; q < P; ++q) {
          const int64_t x = req[q];
          lt += x < v;
          le += x <= v;
        }
        if (lt < r50 && r50 <= le) c50 = v;
        if (lt < r99 && r99 <= le) c99 = v;
      }
    }
    p50 = warp_min64_redux(c50);
    p99 = warp_min64_redux(c99);
  }
  if (lane == 0) {
    ct_replica_summary o;
    if (status == CT_R_OK) {
      o.status = status;
      o.n_done = D;
      o.turns_done = turns_done;
      o.sum_jct_us = jsum;
      o.max_jct_us = jmax;
      o.p50_jct_us = p50;
      o.p99_jct_us = p99;
      o.sum_bubble_us = acc->bubble;
      o.makespan_us = now - arr0;  // the last event processed is the last completion
      o.iterations = n_it;
      o.busy_us = busy;
      o.prefill_tokens = acc->prefill;
      o.recompute_tokens = acc->recomp;
      o.pin_hits = acc->hits;
      o.pin_expiries = acc->exp;
      o.victims = acc->vict;
      o.reloads = acc->reload;
    } else {
      int64_t* w = (int64_t*)&o;
#pragma unroll
      for (int i = 0; i < 16; ++i) w[i] = 0;
      o.status = status;
    }
    a.out[ri] = o;
  }
  if (a.jct) {
    int64_t* jo = a.jct + ri * P;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const int p = lane + 32 * s;
      if (p < P) jo[p] = status == CT_R_OK ? req[p] : -1;
    }
  }
  if (bub && status != CT_R_OK) {
#pragma unroll
    for (int s = 0; s < NS; ++s)
      if (lane + 32 * s < P) bub[lane + 32 * s] = -1;
  }
  __syncwarp();
}

// -----------------------------------------------------------------------------------------------
// 32 < P <= 256, simple class (simple_policy: program or request FCFS), default engine, with
// 32-bit replica-relative times (as replay_one_t32: µs since the first arrival, saturated at
// T32_LIM; iteration indices stay below the time).  28 B of shared memory per program (tev,
// texp, req/JCT, fin as u32; ctx, gblk, turn), so 28 warps (all 4,096 replicas of cfg2) fit on
// the GPU at once.  Returns false, before writing any output, when the replica reaches the
// horizon or asks for the bubble output; the caller queues it for a 64-bit launch (the
// program-FCFS kernel when every policy is in that class, else the generic one), which
// replays it from scratch.  Otherwise identical to the 64-bit path step for step.


template <int NS, bool REQ>
__device__ __forceinline__ bool replay_one_ns32(const ReplayArgs& a, int64_t r,
                                                unsigned char* wm, int lane) {
  constexpr int PM = 32 * NS;
  if (a.bubble) return false;  // the per-program bubble output runs on the 64-bit path
  uint32_t* tev = (uint32_t*)wm;   // tool return, INF otherwise
  uint32_t* texp = tev + PM;       // expiry + 1 while pinned in a tool call, INF otherwise
  uint32_t* req = texp + PM;       // request arrival; JCT once done
  uint32_t* fin = req + PM;        // finishing iteration while running, INF otherwise
  int32_t* ctx = (int32_t*)(fin + PM);
  int32_t* gblk = ctx + PM;
  int32_t* tix = gblk + PM;        // index of the program's current turn record in a.turns
  Stat* stats = (Stat*)(wm + ((28 * PM + 15) & ~15));
  TtlCache* tcache = (TtlCache*)(wm + ((28 * PM + 15) & ~15) + ((32 * (a.F + 1) + 48 + 15) & ~15));

  const int P = a.P, F = a.F;
  const int64_t npol = a.n_pol, nkv = a.n_kv, nrate = a.n_rate;
  const int pol_i = (int)(r % npol);
  const int kv_i = (int)((r / npol) % nkv);
  const int rate_i = (int)((r / (npol * nkv)) % nrate);
  const int64_t seed = r / (npol * nkv * nrate);
  const ct_policy* polp = a.pols + pol_i;
  const int pause = polp->pause;
  // REQ: the sweep has request-FCFS policies (MODE 5); else every policy is program FCFS
  const int prio = REQ ? polp->priority : CT_PRIO_PROG_FCFS;
  const int64_t gap = a.gap[rate_i];
  const ct_program* prog = a.progs + seed * P;
  const ct_engine_params& E = a.eng;
  const ct_estimator_params& est = a.est;
  const int64_t bs = E.bs;
  DivMagic bsm;
  bsm.mhi = (uint32_t)(a.bs_magic >> 32);
  bsm.mlo = (uint32_t)a.bs_magic;
  bsm.dm1 = (uint32_t)(bs - 1);
  bsm.ident = bs == 1 ? 1u : 0u;
  const bool need_stats = pause == CT_PAUSE_PAPER ||
                          (pause == CT_PAUSE_FIXED && polp->t_thresh_us != CT_ALWAYS);

#pragma unroll
  for (int s = 0; s < NS; ++s) {
    const int p = lane + 32 * s;
    tev[p] = T32_INF;
    texp[p] = T32_INF;
    req[p] = 0;
    fin[p] = T32_INF;
    ctx[p] = 0;
    gblk[p] = 0;
    tix[p] = p < a.P ? a.progs[seed * a.P + p].turn0 : 0;
  }
  if (need_stats)
    for (int i = lane; i < 4 * (F + 1); i += 32) ((int64_t*)stats)[i] = 0;
  if (pause == CT_PAUSE_PAPER)
    for (int i = lane; i < F; i += 32) tcache[i].key = ~0ull;
  __syncwarp();

  uint32_t qb = 0, pb = 0, rb = 0, tb = 0;  // per-lane sets over this lane's slots
  uint32_t lev = T32_INF, lexp = T32_INF, fmin = T32_INF;  // cached minima over this lane's slots
  auto own = [&](int p) { return lane == (p & 31); };
  auto bit = [&](int p) { return 1u << (p >> 5); };
  // current turn record: one shared-memory index, then the record (no dependent program load)
  auto rec_of = [&](int p) -> int4 { return __ldg(&a.turns[tix[p]]); };
  const int64_t arr0 = (prog[0].arr_q * gap) >> 20;  // programs arrive in index order: origin
  auto arrival = [&](int i) -> uint32_t { return sat32(((prog[i].arr_q * gap) >> 20) - arr0); };
  auto for_each_set = [&](uint32_t m, auto&& fn) {
    uint32_t slots = __reduce_or_sync(FULL_MASK, m);
    while (slots) {
      const int s = __ffs(slots) - 1;
      slots &= slots - 1;
      uint32_t b = __ballot_sync(FULL_MASK, (m >> s) & 1u);
      while (b) {
        const int p = 32 * s + __ffs(b) - 1;
        b &= b - 1;
        fn(p);
      }
    }
  };
  auto rescan_lev = [&]() {
    uint32_t m = T32_INF;
#pragma unroll
    for (int s = 0; s < NS; ++s) m = min(m, tev[lane + 32 * s]);
    lev = m;
  };
  auto rescan_lexp = [&]() {
    uint32_t m = T32_INF;
#pragma unroll
    for (int s = 0; s < NS; ++s) m = min(m, texp[lane + 32 * s]);
    lexp = m;
  };
  auto rescan_fmin = [&]() {
    uint32_t m = T32_INF;
#pragma unroll
    for (int s = 0; s < NS; ++s) m = min(m, fin[lane + 32 * s]);
    fmin = m;
  };

  uint32_t now = 0, iter_end = 0, n_it = 0;
  const uint32_t it_cap = E.max_iters >= (int64_t)T32_INF ? T32_INF : (uint32_t)E.max_iters;
  bool in_flight = false;
  int32_t free_blk = (int32_t)a.kv[kv_i];  // blocks, contexts, tokens: below 2^30 (validated)
  int next_arr = 0;
  uint32_t t_arr = 0;  // program 0 arrives at the origin
  int32_t D = 0, turns_done = 0;
  int n_run = 0;
  int32_t kv_sum = 0;
  int64_t pf = 0;
  int status = CT_R_OK;
  int32_t kv_at = -1;
  uint32_t d_cur = 0, rb_cur = 0;
  float rd_cur = 0.0f;
  int64_t accv = 0;  // lane k holds summary counter k (ACC_*)
  auto acc_add = [&](int k, int64_t v) {
    if (lane == k) accv += v;
  };

  // evict(v): free its GPU blocks; unpin.  Uniform.
  auto evict_unpin = [&](int v) {
    free_blk += gblk[v];
    __syncwarp();  // every lane has read v's fields before the owner rewrites them
    if (own(v)) {
      gblk[v] = 0;
      if (pb & bit(v)) {
        pb &= ~bit(v);
        if (texp[v] != T32_INF) { texp[v] = T32_INF; rescan_lexp(); }
      }
    }
    __syncwarp();
  };

  bool qleft = false;  // a program still queued after the last admit loop (see replay_one_t32)
  for (;;) {
    uint32_t t;
    if (in_flight) {
      t = iter_end;
    } else {
      t = min(__reduce_min_sync(FULL_MASK, qleft ? min(lev, lexp) : lev), t_arr);
      if (t == T32_INF) break;
    }
    if (t >= T32_LIM) return false;  // beyond the 32-bit horizon: 64-bit kernel
    now = t;

    // PinExpiry (EAGER): first µs with now > expiry while not in Q (R4/R15); it
    // precedes the program's own tool return at the same µs (R1)
    if (__any_sync(FULL_MASK, lexp <= now)) {
      uint32_t me = 0;
      if (lexp <= now) {
#pragma unroll
        for (int s = 0; s < NS; ++s) {
          const int p = lane + 32 * s;
          me |= (texp[p] <= now && texp[p] <= tev[p] ? 1u : 0u) << s;
        }
      }
      acc_add(ACC_EXP, __reduce_add_sync(FULL_MASK, (uint32_t)__popc(me)));
      for_each_set(me, [&](int p) { evict_unpin(p); });
    }
    // ToolReturn (OnRequestArrive of a seen program)
    if (__any_sync(FULL_MASK, lev <= now)) {
      uint32_t md = 0;
      if (lev <= now) {
#pragma unroll
        for (int s = 0; s < NS; ++s) md |= (tev[lane + 32 * s] <= now ? 1u : 0u) << s;
      }
      const uint32_t mret = md & tb;
      if (need_stats) {
        for_each_set(mret, [&](int p) {  // estimator rows: Δ_obs = dur of the finished turn (R5)
          const int4 tr = rec_of(p);
          const int64_t x = min((int64_t)tr.w, est.b_us);
          const uint64_t x2 = (uint64_t)x * (uint64_t)x;
          if (lane == 0) {
            Stat* rows[2] = {&stats[F], &stats[tr.z]};
#pragma unroll
            for (int k = 0; k < 2; ++k) {
              Stat* q = rows[k];
              q->n += 1;
              q->s1 += x;
              const uint64_t lo = q->s2lo + x2;
              q->s2hi += (lo < x2);
              q->s2lo = lo;
            }
          }
          __syncwarp();
        });
      }
      if (md) {
        bool rescan_e = false;
#pragma unroll
        for (int s = 0; s < NS; ++s) {
          const int p = lane + 32 * s;
          if ((mret >> s) & 1u) {
            tix[p] += 1;
            req[p] = tev[p];  // the event's own instant
            tev[p] = T32_INF;
            if (texp[p] != T32_INF) { texp[p] = T32_INF; rescan_e = true; }  // retained pin
          }
        }
        qb |= mret;
        tb &= ~mret;
        rescan_lev();
        if (rescan_e) rescan_lexp();
      }
      __syncwarp();
    }
    // ProgramArrival (programs arrive in index order)
    while (t_arr <= now) {
      const int p = next_arr;
      if (own(p)) { qb |= bit(p); req[p] = t_arr; }
      ++next_arr;
      t_arr = next_arr < P ? arrival(next_arr) : T32_INF;
    }
    __syncwarp();

    // IterationEnd: requests whose last token was emitted finish, in index order (C-6)
    if (in_flight && iter_end == now) {
      in_flight = false;
      uint32_t mf = 0;
      if (fmin == n_it) {
#pragma unroll
        for (int s = 0; s < NS; ++s) mf |= (fin[lane + 32 * s] == n_it ? 1u : 0u) << s;
      }
      for_each_set(mf, [&](int p) {
        // OnRequestFinish
        const int tx = tix[p];
        const int4 tr = __ldg(&a.turns[tx]);
        const ct_program pr = prog[p];  // issued beside the record load
        const int tp = tx - pr.turn0;
        const int nctx = ctx[p] + tr.x + tr.y;
        const int32_t g = gblk[p];
        --n_run;
        kv_sum -= g;
        __syncwarp();
        if (own(p)) { rb &= ~bit(p); fin[p] = T32_INF; ctx[p] = nctx; }
        __syncwarp();
        const int nt = pr.nturns;
        if (tp == nt - 1) {  // last request: free its KV, the program completes
          free_blk += g;
          __syncwarp();
          if (own(p)) { gblk[p] = 0; req[p] = now - sat32(((pr.arr_q * gap) >> 20) - arr0); }
          ++D;
          turns_done += nt;
          __syncwarp();
        } else {
          const int f = tr.z;
          int64_t ttl = 0;
          if (pause == CT_PAUSE_FIXED) {
            ttl = simplified_ttl(stats[F], stats[f], est, polp->t_pin_us, polp->t_thresh_us);
          } else if (pause == CT_PAUSE_PAPER) {
            ttl = calc_ttl_cached(stats, tcache, F, f, est, D, turns_done, lane);
          } else if (pause == CT_PAUSE_FITTED) {
            ttl = __ldg(&a.fitted[(int64_t)f * a.J + min(tp, a.J - 1)]);
          }
          if (ttl > 0) {  // pin_request only if TTL != 0
            if (own(p)) {
              pb |= bit(p);
              texp[p] = ttl >= (int64_t)T32_LIM ? T32_LIM : sat32((int64_t)now + ttl + 1);
              lexp = min(lexp, texp[p]);
            }
          } else {
            evict_unpin(p);
          }
          if (own(p)) { tev[p] = sat32((int64_t)now + tr.w); lev = min(lev, tev[p]); tb |= bit(p); }
          __syncwarp();
        }
      });
      if (mf) rescan_fmin();
    }
    if (in_flight) continue;  // mid-iteration: events only mutate Q / stats / pins (R2)

    // ---- scheduling point (R3): admit loop (victims PAPER.md:645-655) -----
    int admitted = 0;
    bool stable = true;
    qleft = false;
    if (__any_sync(FULL_MASK, qb != 0)) {
      for (;;) {
        if (!__any_sync(FULL_MASK, qb != 0)) break;
        if (n_run >= E.max_batch) { qleft = true; break; }
        int h;
        if (prio == CT_PRIO_PROG_FCFS) {  // lowest index among pinned-queued, else queued
          uint32_t sel = qb & pb;
          uint32_t slots = __reduce_or_sync(FULL_MASK, sel);
          if (!slots) { sel = qb; slots = __reduce_or_sync(FULL_MASK, sel); }
          const int s0 = __ffs(slots) - 1;
          h = 32 * s0 + __ffs(__ballot_sync(FULL_MASK, (sel >> s0) & 1u)) - 1;
        } else {  // REQ_FCFS (vanilla vLLM): earliest request, ties by index
          uint32_t bk = T32_INF;
          int bp = 0x7fffffff;
#pragma unroll
          for (int s = 0; s < NS; ++s) {
            const int pl = lane + 32 * s;
            if (((qb >> s) & 1u) && req[pl] < bk) { bk = req[pl]; bp = pl; }
          }
          const uint32_t mk = __reduce_min_sync(FULL_MASK, bk);
          h = (int)__reduce_min_sync(FULL_MASK, (uint32_t)(bk == mk ? bp : 0x7fffffff));
        }
        const int4 tr = rec_of(h);
        const int32_t hctx = ctx[h];
        const int32_t hg = gblk[h];
        const int32_t need = (int32_t)ceil_div_magic((uint32_t)(hctx + tr.x + tr.y), bsm) - hg;
        if (need > free_blk && admitted == 0) {
          while (need > free_blk) {  // victims: latest program arrival first, never the head
            const uint32_t cand = pb & ~(own(h) ? bit(h) : 0u);
            const uint32_t vs = __reduce_or_sync(FULL_MASK, cand);
            if (!vs) break;
            const int s1 = 31 - __clz(vs);
            const int v = 32 * s1 + 31 - __clz(__ballot_sync(FULL_MASK, (cand >> s1) & 1u));
            evict_unpin(v);
            acc_add(ACC_VICT, 1);
          }
        }
        if (need > free_blk) {  // HOL break
          if (admitted > 0 && __reduce_or_sync(FULL_MASK, pb & ~(own(h) ? bit(h) : 0u)))
            stable = false;
          qleft = true;
          break;
        }
        // issue h
        free_blk -= need;
        const int32_t ng = hg + need;
        acc_add(ACC_BUBBLE, (int64_t)(now - req[h]));
        const bool hp = (__shfl_sync(FULL_MASK, pb, h & 31) >> (h >> 5)) & 1u;
        const int32_t cached = hp ? hctx : 0;
        if (hp) acc_add(ACC_HITS, 1);
        acc_add(ACC_RECOMP, hctx - cached);
        const int64_t u = hctx + tr.x - cached;
        acc_add(ACC_PREFILL, u);
        __syncwarp();  // every lane has read h's fields before the owner rewrites them
        if (own(h)) {
          qb &= ~bit(h);
          pb &= ~bit(h);  // a queued pin has no pending expiry (cleared at its return)
          gblk[h] = ng;
          rb |= bit(h);
          fin[h] = sat32((int64_t)n_it + tr.y);
          fmin = min(fmin, fin[h]);
        }
        ++n_run;
        kv_sum += ng;
        pf += u;
        ++admitted;
        __syncwarp();
      }
      // unschedulable: the head missed with nothing running (C-5 5c)
      if (admitted == 0 && n_run == 0 && __any_sync(FULL_MASK, qb != 0)) {
        status = CT_R_UNSCHEDULABLE;
        break;
      }
    }
    // start the next iteration(s) (linear cost model, R16)
    if (n_run > 0) {
      if (kv_sum != kv_at) {
        kv_at = kv_sum;
        d_cur = iter_us_kv32(a, (uint32_t)kv_sum, &rb_cur);  // < 2^31 (host-checked)
        rd_cur = rcp_approx((float)d_cur);  // estimate only: macro_iters32 corrects
      }
      const int64_t dur1 = pf > 0 ? iter_us_prefill(a, d_cur, rb_cur, (uint32_t)kv_sum, pf) : d_cur;
      pf = 0;
      // 32-bit macro-step as in replay_one_t32 (every end is checked against the horizon)
      if (dur1 >= (int64_t)(T32_LIM - now)) return false;
      const uint32_t end1 = now + (uint32_t)dur1;
      uint32_t kk = 0;
      if (stable) {
        const uint32_t mfin = __reduce_min_sync(FULL_MASK, fmin);
        const uint32_t te = min(__reduce_min_sync(FULL_MASK, qleft ? min(lev, lexp) : lev), t_arr);
        kk = extra_iters32(mfin - n_it - 1, te, end1, d_cur, rd_cur);
      }
      const uint64_t end = (uint64_t)end1 + (uint64_t)kk * d_cur;
      if ((uint64_t)n_it + kk + 1 > it_cap) { status = CT_R_EVENT_BUDGET; break; }
      if (end >= T32_LIM) return false;  // beyond the 32-bit horizon
      n_it += kk + 1;
      iter_end = (uint32_t)end;
      acc_add(ACC_BUSY, (int64_t)((uint32_t)end - now));
      in_flight = true;
    }
  }
  if (status == CT_R_OK && D != P) status = CT_R_UNSCHEDULABLE;

  // ---- per-replica summary (A-8) --------------------------------------------------------------
  __syncwarp();
  const int64_t ri = r - a.r_begin;
  int64_t jsum = 0, jmax = 0, p50 = 0, p99 = 0;
  if (status == CT_R_OK) {
    int64_t ls = 0;
    uint32_t lm = 0;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const int p = lane + 32 * s;
      if (p < P) { ls += req[p]; lm = max(lm, req[p]); }
    }
    jsum = (int64_t)warp_sum_u64((uint64_t)ls);
    jmax = __reduce_max_sync(FULL_MASK, lm);
    // nearest rank (R20): value v with #(x < v) < rank <= #(x <= v); once per replica, so
    // kept rolled (instruction footprint)
    const int r50 = (50 * P + 99) / 100, r99 = (99 * P + 99) / 100;
    uint32_t c50 = T32_INF, c99 = T32_INF;
#pragma unroll 1
    for (int s = 0; s < NS; ++s) {
      const int p = lane + 32 * s;
      if (p < P) {
        const uint32_t v = req[p];
        int lt = 0, le = 0;
        for (int q = 0; q < P; ++q) {
          const uint32_t x = req[q];
          lt += x < v;
          le += x <= v;
        }
        if (lt < r50 && r50 <= le) c50 = v;
        if (lt < r99 && r99 <= le) c99 = v;
      }
    }
    p50 = __reduce_min_sync(FULL_MASK, c50);
    p99 = __reduce_min_sync(FULL_MASK, c99);
  }
  int64_t av[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) av[k] = shfl64(accv, k);
  if (lane == 0) {
    ct_replica_summary o;
    if (status == CT_R_OK) {
      o.status = status;
      o.n_done = D;
      o.turns_done = turns_done;
      o.sum_jct_us = jsum;
      o.max_jct_us = jmax;
      o.p50_jct_us = p50;
      o.p99_jct_us = p99;
      o.sum_bubble_us = av[ACC_BUBBLE];
      o.makespan_us = now;  // the last event processed is the last completion; origin = arr0
      o.iterations = n_it;
      o.busy_us = av[ACC_BUSY];
      o.prefill_tokens = av[ACC_PREFILL];
      o.recompute_tokens = av[ACC_RECOMP];
      o.pin_hits = av[ACC_HITS];
      o.pin_expiries = av[ACC_EXP];
      o.victims = av[ACC_VICT];
      o.reloads = av[ACC_RELOAD];
    } else {
      int64_t* w = (int64_t*)&o;
#pragma unroll
      for (int i = 0; i < 16; ++i) w[i] = 0;
      o.status = status;
    }
    a.out[ri] = o;
  }
  if (a.jct) {
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const int p = lane + 32 * s;
      if (p < P) a.jct[ri * P + p] = status == CT_R_OK ? (int64_t)req[p] : -1;
    }
  }
  __syncwarp();
  return true;
}

// VLLM: the vLLM engine of NEXT-2 (KV growth, chunked prefill), always through the
// shared-memory path (also P <= 32).
// MODE (default engine): P <= 32: 0 every policy generic; 1 every policy in the TTL-grid class
// (32-bit times, fallback to the 64-bit TTL-grid path); 3 every policy in the simple class
// (program or request FCFS, 32-bit times with the estimator, fallback to the generic path);
// 2 mixed: simple-class replicas as in 3, the others generic; 6 every policy in the extended class
// (ext_policy: DRAM tier, PLAS, InferCept; 32-bit times, fallback to the generic path).  P > 32: 0 generic, 1 every policy in the program-FCFS
// class; 4 every policy in the program-FCFS class with 32-bit times (replay_one_ns32), replicas
// that reach the horizon are queued for a second launch of MODE 1 over that list (from_list);
// 5 the same for the simple class with request FCFS (fallback launch: the generic kernel).
// A trace set that failed the on-device check (validate.cu): no record is read; the replica
// reports CT_R_INVALID_INPUT with a zero summary and -1 per-program outputs.
__device__ __forceinline__ void write_invalid(const ReplayArgs& a, int64_t r, int lane) {
  const int64_t ri = r - a.r_begin;
  if (lane < 16) ((int64_t*)&a.out[ri])[lane] = lane == 0 ? CT_R_INVALID_INPUT : 0;
  for (int p = lane; p < a.P; p += 32) {
    if (a.jct) a.jct[ri * a.P + p] = -1;
    if (a.bubble) a.bubble[ri * a.P + p] = -1;
  }
}

template <int NS, int MINB, bool VLLM = false, int MODE = 0>
__global__ void __launch_bounds__(128, MINB) replay_kernel(ReplayArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31;
  unsigned char* wm = smem + (threadIdx.x >> 5) * a.smem_per_warp;
  // next replica of this warp (persistent grid over an atomic counter); false when done
  auto next = [&](int64_t& r) -> bool {
    for (;;) {
      unsigned long long idx = 0;
      if (lane == 0) idx = atomicAdd(a.counter, 1ull);
      idx = __shfl_sync(FULL_MASK, idx, 0);
      if (a.from_list) {  // replicas queued by a MODE 4 launch earlier on the stream
        if (idx >= *a.fb_count) return false;
        r = a.fb_list[idx];
      } else if (a.n_sel > 0) {  // the replicas of the launch's policy subset in [r_begin, r_end)
        // (32-bit quotient: the host splits only when blocks x n_sel < 2^31)
        if (idx >= (unsigned long long)a.sel_total) return false;
        const uint32_t q = (uint32_t)idx / (uint32_t)a.n_sel;
        r = (a.blk0 + q) * a.n_pol + a.sel[(uint32_t)idx - q * (uint32_t)a.n_sel];
        if (r < a.r_begin || r >= a.r_end) continue;
      } else {
        r = a.r_begin + (int64_t)idx;
        if (r >= a.r_end) return false;
      }
      return true;
    }
  };
  int64_t r;
  if (a.err[0] != 0) {  // the trace check failed: no record is read (kept out of the main loop)
    while (next(r)) write_invalid(a, r, lane);
    return;
  }
  while (next(r)) {
    if (NS == 1 && !VLLM) {
      if (MODE == 1) {
        if (!replay_one_t32<false>(a, r, (Stat*)wm, lane)) replay_one_w32<true>(a, r, (Stat*)wm, lane);
      } else if (MODE == 3 || (MODE == 2 && simple_policy(a.pols[(int)(r % a.n_pol)], a.eng))) {
        if (!replay_one_t32<true>(a, r, (Stat*)wm, lane)) replay_one_w32<false>(a, r, (Stat*)wm, lane);
      } else if (MODE == 6) {
        if (!replay_one_t32<true, true>(a, r, (Stat*)wm, lane)) replay_one_w32<false>(a, r, (Stat*)wm, lane);
      } else {
        replay_one_w32<false>(a, r, (Stat*)wm, lane);
      }
    } else if (MODE == 4 || MODE == 5) {
      if (!replay_one_ns32<NS, MODE == 5>(a, r, wm, lane) && lane == 0)
        a.fb_list[atomicAdd(a.fb_count, 1ull)] = r;
    } else {
      replay_one_ns<NS, VLLM, (MODE == 1)>(a, r, wm, lane);
    }
  }
}

// P <= 32 generic kernel: register budget (min resident CTAs of 4 warps per SM); the TTL-grid
// class kernel (MODE 1) runs at 10 (48 registers, 40 warps/SM, measured best on cfg3).
#ifndef CT_REPLAY_MINB
#define CT_REPLAY_MINB 8
#endif
#ifndef CT_REPLAY_MINB_GRID
#define CT_REPLAY_MINB_GRID 10
#endif
#ifndef CT_REPLAY_MINB_EXT
#define CT_REPLAY_MINB_EXT 7  // extended class (MODE 6): 72 registers, 28 warps/SM, measured best (cfg4)
#endif

#ifndef NS32_MINB
#define NS32_MINB 7  // 7 CTAs of 4 warps per SM: 28 warps, <= 73 registers, 28 B SMEM per program
#endif
#ifndef NS_PROG_MINB
#define NS_PROG_MINB 5  // 5 CTAs of 4 warps per SM: <= 102 registers, 48 B SMEM per program
#endif

}  // namespace ct
