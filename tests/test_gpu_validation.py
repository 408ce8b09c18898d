"""Input validation and the integer bounds of the replay (include/continuum.h preconditions).

* Rejected inputs: every trace-record violation is caught on the device (every replica reports
  CT_R_INVALID_INPUT, no record is read; ct_validate_trace_set names the program) and on the
  host path (CT_EINVAL); every host-checked engine / estimator / sweep bound gives CT_EINVAL.
* Accepted inputs at the bounds: arrivals with arr_q * gap just below 2^62, contexts of 2^30
  tokens, iteration costs just below 2^62 ps, DRAM loads near 2^62 ps, CalcTTL saturating at
  CT_TTL_SAT - 1 (reading R36), TTLs of CT_TTL_SAT - 1: the GPU equals the oracle byte for byte.
"""
from dataclasses import replace

import numpy as np
import pytest
import torch

from ctgen import configs as cf
from ctgen import traces
from oracle import oracle as O

pytestmark = pytest.mark.gpu
INVALID_INPUT = 3
TTL_SAT = 1 << 50


@pytest.fixture(scope="module")
def ct():
    from paper_2511_02230_b200 import build
    build.build()
    import paper_2511_02230_b200 as m
    return m


@pytest.fixture(scope="module")
def ctx(ct):
    return ct.Context(0)


def base_trace(P=3):
    return traces.tiny([(i * 10, [(20, 4, 0, 50), (5, 2, 1, 30), (3, 1, -1, 0)]) for i in range(P)],
                       n_tools=2)


ENG = cf.Engine(c0_ps=10**6, c_pf_ps=10**6, c_kv_ps=0, c_h2d_ps=5 * 10**5, bs=4, max_batch=8,
                dram_blocks=100)


def corrupt(kind):
    tr = base_trace()
    p, t = tr.programs.copy(), tr.turns.copy()
    if kind == "nturns0":
        p["nturns"][1] = 0
    elif kind == "turn_range":
        p["turn0"][2] = len(t) - 1
    elif kind == "unsorted":
        p["arr_q"][2] = 1
    elif kind == "arrival_bound":
        p["arr_q"][2] = (1 << 62) // (1 << 20) + 1
    elif kind == "decode0":
        t[1, 1] = 0
    elif kind == "tool_range":
        t[4, 2] = 2
    elif kind == "dur0":
        t[0, 3] = 0
    elif kind == "context":
        t[0, 0] = (1 << 30) - 10
    elif kind == "nturns_max":
        p["nturns"][0] = 65537
    return traces.TraceSet(p, t, 1, tr.n_programs, tr.n_tools, tr.pclass)


KINDS = ["nturns0", "turn_range", "unsorted", "arrival_bound", "decode0", "tool_range", "dur0",
         "context", "nturns_max"]


@pytest.mark.parametrize("kind", KINDS)
def test_invalid_trace_records(ct, ctx, kind):
    from paper_2511_02230_b200 import _lib
    tr = corrupt(kind)
    sw = cf.Sweep(1, [1 << 20], [100, 50], [cf.PROG_FCFS, cf.CONTINUUM])
    dt = ct.DeviceTrace(tr)
    s, j = ct.ct_simulate_batch(ctx, dt, sw, ENG, jct=True)
    s, j = s.cpu().numpy(), j.cpu().numpy()
    assert np.all(s[:, 0] == INVALID_INPUT) and np.all(s[:, 1:] == 0) and np.all(j == -1)
    with pytest.raises(_lib.CtError, match="program"):
        ct.ct_validate_trace_set(ctx, dt, sw)
    with pytest.raises(_lib.CtError):
        ct.ct_simulate_batch_host(ctx, tr, sw, ENG)
    # the check covers only the seeds of the replica range: a clean trace passes
    ct.ct_validate_trace_set(ctx, ct.DeviceTrace(base_trace()), sw)


def test_invalid_fitted_table(ct, ctx):
    tr = base_trace()
    for bad in (-1, TTL_SAT):
        fitted = np.array([[0, 5], [7, bad]], np.int64)
        sw = cf.Sweep(1, [1 << 20], [100], [cf.CONTINUUM_FITTED], fitted=fitted)
        s, _ = ct.ct_simulate_batch(ctx, ct.DeviceTrace(tr), sw, ENG)
        assert np.all(s.cpu().numpy()[:, 0] == INVALID_INPUT)


def test_host_checked_bounds(ct, ctx):
    from paper_2511_02230_b200 import _lib
    tr = base_trace()
    dt = ct.DeviceTrace(tr)
    sw = cf.Sweep(1, [1 << 20], [100], [cf.PROG_FCFS])
    bad_engines = [replace(ENG, c_pf_ps=(1 << 40) - 1, bs=1 << 19),           # iteration >= 2^62 ps
                   replace(ENG, c_kv_ps=(1 << 30) - 1, bs=(1 << 20) - 1),
                   replace(ENG, dram_blocks=(1 << 30) - 1, c_h2d_ps=(1 << 40) - 1)]
    big_kv = cf.Sweep(1, [1 << 20], [(1 << 30) - 1], [cf.PROG_FCFS])
    for eng in bad_engines:
        with pytest.raises(_lib.CtError, match="2\\^62"):
            ct.ct_simulate_batch(ctx, dt, big_kv, eng)
    for est in (cf.Estimator(a_den=1 << 20), cf.Estimator(a_num=1 << 20), cf.Estimator(b_us=1 << 40)):
        with pytest.raises(_lib.CtError):
            ct.ct_simulate_batch(ctx, dt, cf.Sweep(1, [1 << 20], [100], [cf.CONTINUUM], est), ENG)
    with pytest.raises(_lib.CtError):  # a FITTED table with fewer rows than tools
        ct.ct_simulate_batch(ctx, dt, cf.Sweep(1, [1 << 20], [100], [cf.CONTINUUM_FITTED],
                                               fitted=np.zeros((1, 3), np.int64)), ENG)
    with pytest.raises(_lib.CtError):
        ct.ct_simulate_batch(ctx, dt, cf.Sweep(1, [1 << 20], [100], [cf.ttl_grid(TTL_SAT)]), ENG)
    ct.ct_simulate_batch(ctx, dt, sw, ENG)  # and the valid call still works


def compare(ct, ctx, tr, sw, eng):
    s, j = ct.ct_simulate_batch(ctx, ct.DeviceTrace(tr), sw, eng, jct=True)
    os_, oj = O.simulate(tr, sw, eng)
    assert np.array_equal(s.cpu().numpy(), os_), (s.cpu().numpy(), os_)
    assert np.array_equal(j.cpu().numpy(), oj)
    return os_


def test_accepted_extremes_equal_oracle(ct, ctx):
    gap = (1 << 30) - 1
    amax = ((1 << 62) - 1) // gap
    # arrivals up to arr_q * gap < 2^62 (µs ~ 2^62): program arrivals spread over the range
    tr = traces.tiny([(0, [(10, 2, 0, 5), (3, 1, -1, 0)]), (amax // 2, [(7, 3, 1, 9), (1, 1, -1, 0)]),
                      (amax, [(4, 4, -1, 0)])], n_tools=2)
    sw = cf.Sweep(1, [gap, 1 << 20, 1], [64], [cf.PROG_FCFS, cf.ttl_grid(TTL_SAT - 1), cf.VLLM,
                                              cf.CONTINUUM])
    s = compare(ct, ctx, tr, sw, ENG)
    assert np.all(s[:, 0] & 0xFFFFFFFF == 0)
    # contexts of 2^30 tokens with iteration costs just below 2^62 ps
    bs = 1 << 10
    kv = (1 << 20) + 8
    c_pf = ((1 << 62) - 1 - 10**6) // (bs * kv) - 1
    eng = cf.Engine(c0_ps=10**6, c_pf_ps=c_pf, c_kv_ps=0, c_h2d_ps=1, bs=bs, max_batch=4,
                    dram_blocks=(1 << 29), max_iters=1 << 40)
    half = (1 << 29) - 4
    tr = traces.tiny([(0, [(half, 2, 0, 100), (half, 2, -1, 0)]), (5, [(1000, 3, -1, 0)])], n_tools=1)
    sw = cf.Sweep(1, [1 << 20], [kv], [cf.PROG_FCFS, cf.ttl_grid(1 << 49), cf.VLLM_LMCACHE])
    s = compare(ct, ctx, tr, sw, eng)
    assert np.all(s[:, 0] & 0xFFFFFFFF == 0) and s[0, 11] == half + 2  # recomputed context
    # DRAM loads near 2^62 ps: dram_blocks x c_h2d just below the bound
    eng = replace(cf.ENGINE_8B, dram_blocks=(1 << 22), c_h2d_ps=((1 << 62) - 1) // (1 << 22))
    tr = traces.generate(2, 12, mix="mix", ctx_cap=4000 * 16, stream=5)
    sw = cf.Sweep(2, [300_000], [4000, 900], [cf.VLLM_LMCACHE, cf.INFERCEPT])
    compare(ct, ctx, tr, sw, eng)


def test_calc_ttl_saturation_replay(ct, ctx):
    """Without a clamp (ttl_max = 0) CalcTTL = T_default^2 / 𝓑 (1 + alpha AvgTurns) exceeds
    int64 for T_default near 2^40: it saturates at CT_TTL_SAT - 1 (R36) on both sides, so the
    pins never expire within the replay."""
    est = cf.Estimator(t_def_us=(1 << 40) - 1, ttl_max_us=0, n_min=1, b_us=1, a_num=(1 << 20) - 1,
                       a_den=1)
    tr = traces.generate(3, 20, mix="mix", ctx_cap=3000 * 16, stream=8)
    sw = cf.Sweep(3, [200_000, 5_000_000], [3000, 600], [cf.CONTINUUM, replace(cf.CONTINUUM, priority=1)],
                  est)
    s = compare(ct, ctx, tr, sw, cf.ENGINE_8B)
    assert np.all(s[:, 13] == 0)  # no pin expired
    g = (1, 1, 1)
    from paper_2511_02230_b200 import api
    assert api.ct_calc_ttl_ref(g, g, est, 0, 0) == TTL_SAT - 1
