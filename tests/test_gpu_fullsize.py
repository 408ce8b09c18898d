"""Full-size parity at BASELINE.json's configs, in the launch configuration bench.py times.

The whole sweep runs on the GPU through ct_simulate_batch (one persistent launch over all
replicas); a seeded sample of replicas is recomputed by the oracle and compared byte for
byte (summary + per-program JCTs), plus the properties that hold at any size.
"""
import numpy as np
import pytest
import torch

from ctgen import configs as cf
from ctgen import traces
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ct():
    from paper_2511_02230_b200 import build
    build.build()
    import paper_2511_02230_b200 as m
    return m


@pytest.fixture(scope="module")
def ctx(ct):
    return ct.Context(0)


def check_sample(ct, ctx, w, n_sample, seed=0):
    dt = ct.DeviceTrace(w.trace)
    s, j = ct.ct_simulate_batch(ctx, dt, w.sweep, w.engine, jct=True)
    torch.cuda.synchronize()
    s, j = s.cpu().numpy(), j.cpu().numpy()
    R = w.sweep.n_replicas
    rng = np.random.default_rng(seed)
    pick = np.unique(np.concatenate([[0, R - 1], rng.integers(0, R, n_sample)]))
    for r in pick:
        os_, oj = O.simulate(w.trace, w.sweep, w.engine, int(r), int(r) + 1)
        assert np.array_equal(s[r], os_[0]), (r, w.sweep.decode(int(r)), s[r], os_[0])
        assert np.array_equal(j[r], oj[0]), r
    # properties at every replica
    st = s[:, 0] & 0xFFFFFFFF
    ok = st == 0
    P = w.trace.n_programs
    assert np.all(s[ok, 0] >> 32 == P)
    assert np.all(s[ok, 2] == j[ok].sum(axis=1))
    assert np.all(s[ok, 3] == j[ok].max(axis=1))
    assert np.all(j[~ok] == -1)
    return s, j


def test_config3_ttl_sweep_full(ct, ctx):
    w = cf.config3()
    s, j = check_sample(ct, ctx, w, 300)
    assert np.all((s[:, 0] & 0xFFFFFFFF) == 0)
    # TTL = 0 column is exactly the no-pin column: zero pin hits / expiries / victims
    npol = len(w.sweep.policies)
    assert np.all(s[0::npol, 12:15] == 0)
    cells = ct.ct_jct_stats(ctx, torch.from_numpy(s).cuda(), w.sweep.n_cells).cpu().numpy()
    assert np.array_equal(cells, O.jct_stats(s, w.sweep.n_cells))


def test_config2_swe200_full(ct, ctx):
    w = cf.config2()
    check_sample(ct, ctx, w, 14)


def test_config5_policy_sweep_full(ct, ctx):
    w = cf.config5()
    check_sample(ct, ctx, w, 300, seed=5)


def test_config4_dram_fitted(ct, ctx):
    w = cf.config4(n_seeds=1024)
    dur, off = traces.tool_samples(w.trace)
    J = 8
    ctxj = [2000 * (j + 1) for j in range(J)]
    wj = [j + 1 for j in range(J)]
    cp = ct.cost_params(w.engine.c_pf_ps, 200, 16, 1, 10, 50_000, 256, ctxj, wj)
    arg, pap, st = ct.ct_fit_ttl(ctx, torch.from_numpy(dur).cuda(), off, cp, w.sweep.estimator)
    torch.cuda.synchronize()
    oa, op, ost = O.fit(dur, off, [w.engine.c_pf_ps, 200, 16, 1, 10, 50_000, 256, J], ctxj, wj,
                        w.sweep.estimator.as_array())
    assert np.array_equal(arg.cpu().numpy(), oa) and np.array_equal(st.cpu().numpy(), ost)
    w.sweep.fitted = oa[:-1]
    check_sample(ct, ctx, w, 60, seed=4)


def test_fit_full_size(ct, ctx):
    """2^28 samples (the bench's bandwidth run): paper statistics of every row and the argmax
    rows of two tools against the oracle's plain definitions."""
    dur, off = traces.synthetic_samples_torch(28, 32, 1234, "cuda")
    J = 4
    ctxj = [1000, 8000, 32000, 120000]
    wj = [1, 2, 3, 4]
    cp = ct.cost_params(13_400_000, 200, 16, 1, 10, 50_000, 256, ctxj, wj, (900, 100))
    est = cf.Estimator()
    arg, pap, st = ct.ct_fit_ttl(ctx, dur, off, cp, est)
    torch.cuda.synchronize()
    h = dur.cpu().numpy()
    # statistics + CalcTTL of every row (K = 1 keeps the oracle O(n))
    _, op, ost = O.fit(h, off, [13_400_000, 200, 16, 1, 10, 50_000, 1, 1], [1], [1],
                       est.as_array(), (900, 100))
    assert np.array_equal(st.cpu().numpy(), ost)
    assert np.array_equal(pap.cpu().numpy(), op)
    # argmax rows of tools 5 (point mass-like cd slot) and 9, from raw samples
    for f in (5, 9):
        seg = h[off[f]:off[f + 1]]
        oa, _, _ = O.fit(seg, np.array([0, len(seg)], np.int64),
                         [13_400_000, 200, 16, 1, 10, 50_000, 256, J], ctxj, wj, est.as_array())
        assert np.array_equal(arg.cpu().numpy()[f], oa[0]), f
