"""Microsecond-stepped brute-force replay (second, independent implementation).

Used only by tests on tiny instances (P <= 3, T <= 3, horizons of a few hundred
µs).  It has no event queue: the clock advances one µs at a time, every timer is
compared against the clock each µs, and a scheduling pass runs at every µs in
which something fired while no iteration is in flight (R3).  Agreement
with the event-driven oracle checks its next-event selection, the R1 order of
same-instant events and the bookkeeping, by a different control structure.  Both expiry
readings (R4): EAGER releases a stale pin the first µs with now > expiry; STEP
(flag 2, §5.3 literal) releases stale pins of programs not waiting in the queue
only at the start of a scheduling pass.

Semantics followed (C-5/C-6, Alg. 1 and §5.3):
  * pin hit iff tool duration <= TTL (expiry checked as now > expiry)
  * requests admitted at iteration boundaries; admission reserves all blocks
  * program-level FCFS (pinned first) or request FCFS priority; HOL break
  * victims: pinned programs with the largest index, only when nothing was admitted
  * engine kv_growth = 1 (NEXT-2, R27-R30): a request holds blocks for its tokens
    so far plus the one it is about to produce; before every scheduling pass each running
    request tops up, best-ranked first, and when the pool is dry the worst-ranked running
    request is thrown back to the queue (recompute), keeping its output so far; thrown-back
    requests are served first
  * engine prefill_chunk = B > 0 (NEXT-2, R31-R32): each iteration computes at most
    B tokens: one per decoding request, then prompt pieces for the requests still prefilling,
    best-ranked first, then newcomers while any budget is left; a request produces output only
    in iterations after (or in the one that finishes) its prompt
"""
from __future__ import annotations

import math

from oracle import oracle as O  # the TTL formula itself is pinned separately


NEVER = 1 << 80  # a preserved pin has no expiry


def simulate(trace, gap_us, kv, pol, est, eng, fitted=None, horizon=200000):
    P = trace.n_programs
    progs = trace.programs
    T = trace.turns
    c0, cpf, ckv, ch2d, bs, maxb, dram_cap, max_it, growth, chunk = [int(x) for x in eng]
    assert chunk == 0 or not growth
    prio, pause, dram, flags, t_pin, t_thresh = [int(x) for x in pol[:6]]
    dram_on = dram != 0 and dram_cap > 0
    victims_any = bool(flags & 1)
    step_expiry = bool(flags & 2)

    arr = [(int(progs["arr_q"][i]) * gap_us) >> 20 for i in range(P)]
    t0 = [int(progs["turn0"][i]) for i in range(P)]
    nt = [int(progs["nturns"][i]) for i in range(P)]

    def rec(i, k):
        return [int(x) for x in T[t0[i] + k]]

    # per-program state as plain dicts
    S = [dict(where="out", turn=0, ctx=0, blk=0, dblk=0, pin=None, waited_since=None,
              tool_back=None, load_at=None, left=0, fresh=0, done_at=None, served=0, out=0,
              thrown=False, waited=0, take=0, speaks=False)
         for _ in range(P)]
    free = kv
    dfree = dram_cap if dram_on else 0
    chan = 0
    stats = {"g": [0, 0, 0]}
    n_done = 0
    turns_done = 0
    cnt = dict(iters=0, busy=0, bubble=0, prefill=0, recompute=0, hits=0, exp=0, vict=0, reload=0,
               thrown=0)
    engine_until = None  # end time of the iteration in flight
    batch = []

    def drop(i):  # free GPU blocks, write through to DRAM
        nonlocal free, dfree
        free += S[i]["blk"]
        S[i]["blk"] = 0
        if dram_on:
            dfree += S[i]["dblk"]
            S[i]["dblk"] = 0
            need = -(-S[i]["ctx"] // bs)
            if 0 < need <= dfree:
                S[i]["dblk"] = need
                dfree -= need

    def row(key):
        return stats.get(key, [0, 0, 0])

    def as_row(r):
        n, s1, s2 = r
        return [n, s1, s2 & (2**64 - 1), s2 >> 64]

    def pause_ttl(i):
        k = S[i]["turn"]
        f = rec(i, k)[2]
        if pause == 0:
            return 0
        if pause == 1:
            return O.simplified(as_row(row("g")), as_row(row(f)), est, t_pin, t_thresh)
        if pause == 2:
            return O.calc_ttl(as_row(row("g")), as_row(row(f)), est, n_done, turns_done)
        if pause == 4:  # InferCept: preserve without TTL iff predicted tool time < swap round trip
            pred = O.infercept_predict(as_row(row("g")), as_row(row(f)), est)
            swap = O.infercept_swap_us(S[i]["ctx"], bs, ch2d)
            return NEVER if pred < swap else 0
        return int(fitted[f][min(k, fitted.shape[1] - 1)])

    now = 0
    while now <= horizon:
        fired = False
        # 1) pins that became stale this µs (first instant with now > expiry)
        for i in range(P):
            s = S[i]
            if not step_expiry and s["where"] == "tool" and s["pin"] is not None and now == s["pin"] + 1:
                drop(i)
                s["pin"] = None
                cnt["exp"] += 1
                fired = True
        # 2) tool results come back: the program re-enters the queue, stats update
        for i in range(P):
            s = S[i]
            if s["where"] == "tool" and s["tool_back"] == now:
                f, d = rec(i, s["turn"])[2:4]
                t = min(d, int(est[1]))
                for key in ("g", f):
                    r = stats.setdefault(key, [0, 0, 0])
                    r[0] += 1
                    r[1] += t
                    r[2] += t * t
                s["turn"] += 1
                s["where"] = "queue"
                s["waited_since"] = now
                s["out"] = 0
                fired = True
        # 3) KV loads complete
        for i in range(P):
            if S[i]["where"] == "loading" and S[i]["load_at"] == now:
                S[i]["where"] = "loaded"
                fired = True
        # 4) new programs
        for i in range(P):
            if S[i]["where"] == "out" and arr[i] == now:
                S[i].update(where="queue", turn=0, ctx=0, waited_since=now)
                fired = True
        # 5) the iteration in flight ends
        if engine_until == now:
            engine_until = None
            fired = True
            for i in sorted(batch):
                s = S[i]
                if not s["speaks"]:
                    continue
                s["left"] -= 1
                s["out"] += 1
                if s["left"] == 0:
                    new, dec, f, d = rec(i, s["turn"])
                    s["ctx"] += new + dec
                    batch.remove(i)
                    if s["turn"] == nt[i] - 1:
                        free += s["blk"]
                        s["blk"] = 0
                        dfree += s["dblk"]
                        s["dblk"] = 0
                        s["where"] = "done"
                        s["done_at"] = now
                        n_done += 1
                        turns_done += nt[i]
                    else:
                        ttl = pause_ttl(i)
                        if ttl > 0:
                            s["pin"] = NEVER if ttl == NEVER else now + ttl
                        else:
                            drop(i)
                        s["tool_back"] = now + d
                        s["where"] = "tool"
        # 6) scheduling pass at an event instant with no iteration in flight (R3)
        if engine_until is None and fired:
            if step_expiry:  # unpin_requests() at the beginning of the scheduling step
                for i in range(P):
                    s = S[i]
                    if s["pin"] is not None and s["where"] != "queue" and now > s["pin"]:
                        drop(i)
                        s["pin"] = None
                        cnt["exp"] += 1

            def rank(i):  # smaller ranks first
                if prio == 0:
                    return (i,)
                if prio == 1:
                    return (S[i]["waited_since"], i)
                return (S[i]["served"], i)

            if growth:
                for i in sorted(batch, key=rank):
                    if i not in batch:
                        continue
                    s = S[i]
                    new = rec(i, s["turn"])[0]
                    want = -(-(s["ctx"] + new + s["out"] + 1) // bs)
                    while want - s["blk"] > free:
                        v = max(batch, key=rank)
                        free += S[v]["blk"]
                        S[v].update(blk=0, where="queue", thrown=True, waited_since=now)
                        batch.remove(v)
                        cnt["thrown"] += 1
                        if v == i:
                            break
                    if i in batch and want > s["blk"]:
                        free -= want - s["blk"]
                        s["blk"] = want
            for i in range(P):
                if S[i]["where"] == "loaded":
                    S[i]["where"] = "run"
                    batch.append(i)
            rest = chunk
            if chunk:
                for i in batch:
                    S[i]["take"] = 0
                rest -= sum(1 for i in batch if S[i]["fresh"] == 0)
                for i in sorted((i for i in batch if S[i]["fresh"] > 0), key=rank):
                    S[i]["take"] = min(S[i]["fresh"], max(rest, 0))
                    rest -= S[i]["take"]
            admitted = 0
            while True:
                waiting = [i for i in range(P) if S[i]["where"] == "queue"]
                busy = len(batch) + sum(1 for i in range(P) if S[i]["where"] == "loading")
                if not waiting or busy >= maxb:
                    break
                if chunk and rest <= 0:
                    break
                thrown = [i for i in waiting if S[i]["thrown"]]
                if thrown:
                    waiting = thrown
                if prio == 0:
                    pinned_w = [i for i in waiting if S[i]["pin"] is not None]
                    h = min(pinned_w) if pinned_w else min(waiting)
                elif prio == 1:
                    h = min(waiting, key=lambda i: (S[i]["waited_since"], i))
                else:  # Autellix PLAS: least attained engine time first
                    h = min(waiting, key=lambda i: (S[i]["served"], i))
                s = S[h]
                new, dec, _, _ = rec(h, s["turn"])
                total = -(-(s["ctx"] + new + (s["out"] + 1 if growth else dec)) // bs)
                need = total - s["blk"]
                if need > free and (admitted == 0 or victims_any):
                    for v in sorted((i for i in range(P) if S[i]["pin"] is not None and i != h),
                                    reverse=True):
                        if need <= free:
                            break
                        drop(v)
                        S[v]["pin"] = None
                        cnt["vict"] += 1
                if need > free:
                    break
                free -= need
                s["blk"] = total
                cnt["bubble"] += now - s["waited_since"]
                s["waited"] += now - s["waited_since"]
                if s["pin"] is not None:
                    cached = s["ctx"]
                    s["pin"] = None
                    cnt["hits"] += 1
                    s["where"] = "run"
                elif dram_on and s["dblk"] > 0 and s["dblk"] == -(-s["ctx"] // bs):
                    cached = s["ctx"]
                    start = max(now, chan)
                    s["load_at"] = start + math.ceil(s["dblk"] * ch2d / 10**6)
                    chan = s["load_at"]
                    cnt["reload"] += 1
                    s["where"] = "loading"
                else:
                    cached = 0
                    s["where"] = "run"
                cnt["recompute"] += s["ctx"] - cached + (new + s["out"] if s["thrown"] else 0)
                s["thrown"] = False
                s["fresh"] = s["ctx"] + new + s["out"] - cached
                cnt["prefill"] += s["fresh"]
                s["left"] = dec - s["out"]
                if s["where"] == "run":
                    batch.append(h)
                    if chunk:
                        s["take"] = min(s["fresh"], rest)
                        rest -= s["take"] if s["fresh"] > 0 else 1
                admitted += 1
            waiting = [i for i in range(P) if S[i]["where"] == "queue"]
            loading = [i for i in range(P) if S[i]["where"] == "loading"]
            if waiting and admitted == 0 and not batch and not loading:
                return "unschedulable", None, None
            if batch:
                if cnt["iters"] >= max_it:
                    return "budget", None, None
                ps = c0 + ckv * bs * sum(S[i]["blk"] for i in batch)
                for i in batch:
                    take = S[i]["take"] if chunk else S[i]["fresh"]
                    S[i]["speaks"] = S[i]["fresh"] == 0 or take == S[i]["fresh"]
                    ps += cpf * take
                    S[i]["fresh"] -= take
                dur = -(-ps // 10**6)
                engine_until = now + dur
                for i in batch:
                    S[i]["served"] += dur
                cnt["iters"] += 1
                cnt["busy"] += dur
        if n_done == P:
            break
        now += 1
    if n_done != P:
        return "horizon", None, None
    jct = [S[i]["done_at"] - arr[i] for i in range(P)]
    makespan = max(S[i]["done_at"] for i in range(P)) - min(arr)
    return "ok", jct, dict(cnt, makespan=makespan, turns=turns_done,
                           waited=[S[i]["waited"] for i in range(P)])
