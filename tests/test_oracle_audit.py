"""The oracle's per-decision audit log (pin / unpin / victim events with their
timestamps, as JSON lines) and the SPEC acceptance checks that are stated against it:
AC7 (victims latest-program-arrival first) and AC11 (SPEC.md:656,
InferCept preserves short tools and swaps long ones).  The log is also checked
against the summary counters it must agree with."""
import random
from dataclasses import replace

import numpy as np
import pytest

from ctgen import configs as cf
from ctgen import traces
from oracle import oracle as O


def contention_trace(n_prog=6, turns=4, tool_us=2_000_000, new=1500, dec=100, gap_q=10_000):
    progs = []
    for p in range(n_prog):
        ts = [(3000 if t == 0 else new, dec, 0, tool_us) for t in range(turns)]
        ts[-1] = (new, dec, -1, 0)
        progs.append((p * gap_q, ts))
    return traces.tiny(progs)


def check_log_consistency(summ, log, ttl_of=None, eager=True):
    """Every pin ends in exactly one unpin (hit / expiry / victim) of that program; counts match
    the summary (pin_hits, pin_expiries, victims); an EAGER expiry happens at pin time + TTL + 1
    (the first µs with now > expiry), a STEP one at a later scheduling point."""
    open_pin = {}
    hits = exps = vics = 0
    last_t = 0
    for e in log:
        assert e["t"] >= last_t  # the log is in time order
        last_t = e["t"]
        p = e["p"]
        if e["ev"] == "pin":
            assert p not in open_pin
            open_pin[p] = e
        elif e["ev"] == "unpin":
            pin = open_pin.pop(p)
            if e["why"] == "hit":
                hits += 1
            elif e["why"] == "expiry":
                exps += 1
                assert pin["ttl"] is not None
                if eager:
                    assert e["t"] == pin["t"] + pin["ttl"] + 1
                else:
                    assert e["t"] > pin["t"] + pin["ttl"]
            else:
                assert e["why"] == "victim" and e["for"] != p
                vics += 1
        elif e["ev"] == "admit":
            assert p not in open_pin  # an admission of a pinned program is logged as its hit
    assert not open_pin
    assert (hits, exps, vics) == (summ[12], summ[13], summ[14])


def test_ac7_victims_latest_arrival_first_from_log():
    tr = contention_trace(n_prog=6, turns=4, tool_us=2_000_000)
    kv = 2 * -(-(3000 + 3 * 1500 + 400) // 16) + 10
    sw = cf.Sweep(1, [1 << 20], [kv], [cf.ttl_grid(10**9)])
    s, log = O.audit(tr, sw, cf.ENGINE_8B, 0)
    assert O.status(s) == 0 and (s[0] >> 32) == 6 and s[14] > 0  # deadlock-free, victims taken
    check_log_consistency(s, log)
    steps = {}
    for e in log:
        if e["ev"] == "unpin" and e["why"] == "victim":
            steps.setdefault((e["t"], e["for"]), []).append(e["p"])
    assert steps
    for (t, h), vs in steps.items():
        assert vs == sorted(vs, reverse=True)  # latest program arrival (largest index) first
        # no program pinned at that instant had a larger index than the first victim, except h
        pinned = set()
        for e in log:
            if e["t"] > t or (e["t"] == t and e["ev"] == "unpin" and e["why"] == "victim"):
                break
            if e["ev"] == "pin":
                pinned.add(e["p"])
            elif e["ev"] == "unpin":
                pinned.discard(e["p"])
        assert max(pinned - {h}) == vs[0]


def test_ac11_infercept_decisions_from_log():
    """Short tools (0.2 s) against a 1 s swap round trip -> preserved without TTL; long tools
    (30 s) -> swapped out (write-through to DRAM, then reloaded)."""
    eng = cf.Engine(c0_ps=2_000_000_000, c_pf_ps=13_400_000, c_kv_ps=16, c_h2d_ps=20_000_000_000,
                    bs=16, max_batch=256, dram_blocks=10_000)
    est = cf.Estimator(n_min=1)
    for tool_us, preserve in ((200_000, True), (30_000_000, False)):
        progs = [(p * 300_000, [(400 if t == 0 else 8, 4, 0, tool_us) for t in range(5)]) for p in range(3)]
        progs = [(a, ts[:-1] + [(8, 4, -1, 0)]) for a, ts in progs]
        tr = traces.tiny(progs)
        sw = cf.Sweep(1, [1 << 20], [100_000], [cf.INFERCEPT], est)
        s, log = O.audit(tr, sw, eng, 0)
        assert O.status(s) == 0
        check_log_consistency(s, log)
        pins = [e for e in log if e["ev"] == "pin"]
        evicts = [e for e in log if e["ev"] == "evict"]
        if preserve:  # predicted 0.2 s < ~1 s round trip, once the tool has a sample (before
            # that the prediction is T_default = 10 s, and the turn swaps)
            first_return = min(e["t"] for e in pins + evicts) + tool_us
            assert pins and all(e["ttl"] is None for e in pins)
            assert all(e["t"] < first_return for e in evicts)
            assert len(pins) > len(evicts)
        else:         # predicted 30 s > round trip: swap out, reload through the H2D channel
            assert evicts and not pins
            assert any(e["ev"] == "admit" and e["load"] == 1 for e in log)


@pytest.mark.parametrize("seed", range(3))
def test_log_agrees_with_summary_random(seed):
    rng = random.Random(seed)
    tr = traces.generate(2, 10, mix="mix", ctx_cap=2500 * 16, stream=30 + seed)
    fitted = np.tile(np.array([[0, 200_000, 3_000_000]], np.int64), (tr.n_tools, 1))
    eng = cf.Engine(**{**cf.ENGINE_8B.__dict__, "dram_blocks": 400})
    pols = [cf.CONTINUUM, cf.ttl_grid(500_000), cf.ttl_grid(5_000_000), cf.VLLM_LMCACHE,
            cf.INFERCEPT, cf.AUTELLIX, cf.Policy(cf.PRIO_PROG_FCFS, cf.PAUSE_FITTED),
            replace(cf.ttl_grid(800_000), flags=cf.FLAG_STEP_EXPIRY),
            replace(cf.CONTINUUM, flags=cf.FLAG_VICTIMS_ANY)]
    sw = cf.Sweep(2, [150_000, 1_000_000], [rng.choice([700, 1200]), 2500], pols, fitted=fitted)
    full, _ = O.simulate(tr, sw, eng)
    for r in range(sw.n_replicas):
        s, log = O.audit(tr, sw, eng, r)
        assert np.array_equal(s, full[r])  # the audited run is the same replay
        if O.status(s) != 0:
            continue
        pol = sw.policies[sw.decode(r)[3]]
        check_log_consistency(s, log, eager=not (pol.flags & cf.FLAG_STEP_EXPIRY))
        assert sum(e["ev"] == "done" for e in log) == tr.n_programs
        assert sum(e["uncached"] for e in log if e["ev"] == "admit") == s[10]  # prefill tokens
        assert sum(e["load"] for e in log if e["ev"] == "admit") == s[15]     # reloads
