"""Full-size parity at BASELINE.json's configs, on EVERY replica, in the launch configuration
bench.py times (SURVEY.md §8(c) "GPU vs oracle"; Alg. 1).

tests/golden/fullsize_digests.json holds SHA-256 digests of the CPU oracle's summaries and
per-program JCTs for every replica of configs 2-5 (written by tools/oracle_digests.py, which
calls only oracle/ and ctgen/), per block of replicas.  Here the whole sweep runs through
ct_simulate_batch (one persistent launch) and every block's digest must match; a mismatching
block is replayed by the oracle to name the replica.  Config 4 runs its whole fit -> replay
pipeline on the GPU: ct_fit_ttl's table must hash to the oracle's before the FITTED replay.
"""
import hashlib
import json
import os

import numpy as np
import pytest
import torch

from ctgen import configs as cf
from ctgen import traces
from oracle import oracle as O

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DIGESTS = json.load(open(os.path.join(ROOT, "tests", "golden", "fullsize_digests.json")))


@pytest.fixture(scope="module")
def ct():
    from paper_2511_02230_b200 import build
    build.build()
    import paper_2511_02230_b200 as m
    return m


@pytest.fixture(scope="module")
def ctx(ct):
    return ct.Context(0)


def h16(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()[:16]


def gpu_fit_cfg4(ct, ctx, w):
    dur, off = traces.tool_samples(w.trace)
    p = cf.CFG4_FIT
    c = cf.cfg4_fit_cost(w.engine)
    cp = ct.cost_params(c[0], c[1], c[2], c[3], c[4], c[5], c[6], p["ctx_j"], p["w_j"])
    arg, _, _ = ct.ct_fit_ttl(ctx, torch.from_numpy(dur).cuda(), off, cp, w.sweep.estimator,
                              want_stats=False)
    return arg


@pytest.mark.parametrize("name", ["cfg2", "cfg4", "cfg5", "cfg3"])
def test_every_replica_matches_oracle_digest(ct, ctx, name):
    if name not in DIGESTS:
        pytest.fail("tests/golden/fullsize_digests.json has no %s entry "
                    "(run tools/oracle_digests.py %s)" % (name, name))
    rec = DIGESTS[name]
    w = {"cfg2": cf.config2, "cfg3": cf.config3, "cfg4": cf.config4, "cfg5": cf.config5}[name]()
    assert w.trace.digest() == rec["trace_digest"], "the seeded trace generator changed"
    if name == "cfg4":
        arg = gpu_fit_cfg4(ct, ctx, w)
        assert hashlib.sha256(arg.cpu().numpy().tobytes()).hexdigest() == rec["fitted_sha256"]
        w.sweep.fitted = arg[:-1]
    R, B = w.sweep.n_replicas, rec["block"]
    assert R == rec["replicas"]
    s, j = ct.ct_simulate_batch(ctx, ct.DeviceTrace(w.trace), w.sweep, w.engine, jct=True)
    torch.cuda.synchronize()
    s, j = s.cpu().numpy(), j.cpu().numpy()
    bad = [b for b in range(R // B)
           if h16(s[b * B:(b + 1) * B].tobytes()) != rec["block_summary"][b]
           or h16(np.ascontiguousarray(j[b * B:(b + 1) * B]).tobytes()) != rec["block_jct"][b]]
    if bad:  # name the first mismatching replicas (oracle replay of the first bad block)
        if name == "cfg4":
            w.sweep.fitted = w.sweep.fitted.cpu().numpy()
        b = bad[0]
        os_, oj = O.simulate(w.trace, w.sweep, w.engine, b * B, (b + 1) * B, n_threads=os.cpu_count())
        rows = np.nonzero(np.any(s[b * B:(b + 1) * B] != os_, axis=1) |
                          np.any(j[b * B:(b + 1) * B] != oj, axis=1))[0]
        r = b * B + int(rows[0]) if rows.size else None
        pytest.fail("%d of %d blocks differ; first replica %s %s: GPU %s oracle %s" % (
            len(bad), R // B, r, w.sweep.decode(r) if r is not None else "",
            s[r] if r is not None else "", os_[rows[0]] if rows.size else ""))
    assert hashlib.sha256(s.tobytes()).hexdigest() == rec["summary_sha256"]
    cells = ct.ct_jct_stats(ctx, torch.from_numpy(s).cuda(), w.sweep.n_cells).cpu().numpy()
    assert hashlib.sha256(cells.tobytes()).hexdigest() == rec["cells_sha256"]
    st = s[:, 0] & 0xFFFFFFFF
    assert int(s[st == 0, 1].sum()) == rec["replica_turns"]
    if name == "cfg3":  # TTL = 0 column is exactly the no-pin column
        npol = len(w.sweep.policies)
        assert np.all(s[0::npol, 12:15] == 0)


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
    # the sharded fit over 8 ranks gives the same bytes at full size
    acc = sum(ct.ct_fit_ttl_partial(ctx, dur, off, cp, est, r, 8) for r in range(8))
    a8, p8, s8 = ct.ct_fit_ttl_finish(ctx, acc, 32, cp, est)
    assert torch.equal(a8, arg) and torch.equal(p8, pap) and torch.equal(s8, st)
