"""GPU parity of the TTL fit's layouts and its multi-GPU split.

* unsorted (dur_us, u8 tool) pairs (PAPER.md:444's records S = {(f, t)}): the fallback kernel vs
  the oracle on the same samples grouped by tool (a stable sort prepares the oracle's input);
* the sharded fit: ct_fit_ttl_partial per rank, an int64 sum of the accumulators (what the
  NCCL all-reduce computes), ct_fit_ttl_finish == ct_fit_ttl == the oracle, byte for byte, for
  any number of ranks (the statistics are plain sums);
* invalid samples (outside [0, 2^31), or tool ids >= F): counted, every table entry
  CT_TTL_INVALID, and the context's double-buffered accumulator is clean for the next call;
* the 16-lane-replica histogram for grids too large for the 32-replica layout (K >= 900).
"""
import numpy as np
import pytest
import torch

from ctgen import configs as cf
from oracle import oracle as O

pytestmark = pytest.mark.gpu
TTL_INVALID = -1


@pytest.fixture(scope="module")
def ct():
    from paper_2511_02230_b200 import build
    build.build()
    import paper_2511_02230_b200 as m
    return m


@pytest.fixture(scope="module")
def ctx(ct):
    return ct.Context(0)


def params(ct, K, step, J, avg=(0, 0)):
    ctxj = [int(500 * 2**j) % 200_000 + 17 for j in range(J)]
    wj = [j + 1 for j in range(J)]
    cp = ct.cost_params(13_400_000, 40, 16, 3, 7, step, K, ctxj, wj, avg)
    ocost = [13_400_000, 40, 16, 3, 7, step, K, J]
    return cp, ocost, ctxj, wj


def oracle_fit(dur, off, ocost, ctxj, wj, est, avg=(0, 0)):
    return O.fit(dur, off, ocost, ctxj, wj, est.as_array(), avg)


def host(x):
    return tuple(t.cpu().numpy() for t in x)


def random_csr(rng, F, n_max):
    sizes = rng.integers(0, n_max, size=F)
    sizes[rng.integers(0, F)] = int(rng.integers(0, 4))  # a tool below N
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    dur = np.clip(rng.lognormal(np.log(2e6), 1.2, int(off[-1])), 0, 2**31 - 1).astype(np.int32)
    return dur, off


@pytest.mark.parametrize("seed", range(6))
def test_unsorted_pairs_layout(ct, ctx, seed):
    rng = np.random.default_rng(seed)
    F = int(rng.integers(1, 33))
    n = int(rng.integers(0, 400_000))
    tool = rng.integers(0, F, n).astype(np.uint8)
    dur = np.clip(rng.lognormal(np.log(1e6), 1.0, n), 0, 2**31 - 1).astype(np.int32)
    dur[rng.random(n) < 0.03] = 0
    K = int(rng.choice([1, 64, 256]))
    step = int(rng.choice([1, 50_000, 250_000]))
    J = int(rng.integers(1, 9))
    est = cf.Estimator(n_min=int(rng.integers(1, 6)))
    cp, ocost, ctxj, wj = params(ct, K, step, J, (7, 3))
    g = host(ct.ct_fit_ttl(ctx, torch.from_numpy(dur).cuda(), None, cp, est,
                           tool_u8=torch.from_numpy(tool).cuda(), n_tools=F))
    order = np.argsort(tool, kind="stable")
    off = np.concatenate([[0], np.cumsum(np.bincount(tool, minlength=F))]).astype(np.int64)
    o = oracle_fit(dur[order], off, ocost, ctxj, wj, est, (7, 3))
    for name, x, y in zip(("ttl_argmax", "ttl_paper", "stats"), g, o):
        assert np.array_equal(x, y), (name, F, n, K, step)


@pytest.mark.parametrize("world", [2, 3, 8])
def test_sharded_fit_equals_single(ct, ctx, world):
    rng = np.random.default_rng(world)
    F = 12
    dur, off = random_csr(rng, F, 200_003)
    K, step, J = 256, 50_000, 8
    est = cf.Estimator()
    cp, ocost, ctxj, wj = params(ct, K, step, J, (40, 9))
    d = torch.from_numpy(dur).cuda()
    single = host(ct.ct_fit_ttl(ctx, d, off, cp, est))
    acc = sum(ct.ct_fit_ttl_partial(ctx, d, off, cp, est, r, world) for r in range(world))
    sharded = host(ct.ct_fit_ttl_finish(ctx, acc, F, cp, est))
    o = oracle_fit(dur, off, ocost, ctxj, wj, est, (40, 9))
    for x, y, z in zip(single, sharded, o):
        assert np.array_equal(x, y) and np.array_equal(x, z)
    # every sample is counted exactly once over the ranks
    assert int(acc[-1]) == 0


def test_invalid_samples_void_the_table(ct, ctx):
    rng = np.random.default_rng(3)
    F = 5
    dur, off = random_csr(rng, F, 50_000)
    bad_idx = rng.choice(len(dur), 7, replace=False)
    dur_bad = dur.copy()
    dur_bad[bad_idx] = -rng.integers(1, 2**31 - 1, 7)
    cp, ocost, ctxj, wj = params(ct, 128, 50_000, 4)
    est = cf.Estimator()
    arg, pap, st, nbad = host(ct.ct_fit_ttl(ctx, torch.from_numpy(dur_bad).cuda(), off, cp, est,
                                            want_invalid=True))
    assert int(nbad[0]) == 7
    assert np.all(arg == TTL_INVALID) and np.all(pap == TTL_INVALID) and np.all(st == 0)
    # unsorted layout: out-of-range tool ids are invalid samples too
    tool = rng.integers(0, F, len(dur)).astype(np.uint8)
    tool[:3] = F + 1
    arg, pap, st, nbad = host(ct.ct_fit_ttl(ctx, torch.from_numpy(dur).cuda(), None, cp, est,
                                            tool_u8=torch.from_numpy(tool).cuda(), n_tools=F,
                                            want_invalid=True))
    assert int(nbad[0]) == 3 and np.all(arg == TTL_INVALID)
    # the next valid calls are unaffected (the accumulator halves are cleaned in-kernel)
    for _ in range(3):
        g = host(ct.ct_fit_ttl(ctx, torch.from_numpy(dur).cuda(), off, cp, est, want_invalid=True))
        assert int(g[3][0]) == 0
        o = oracle_fit(dur, off, ocost, ctxj, wj, est)
        for x, y in zip(g[:3], o):
            assert np.array_equal(x, y)


def test_alternating_shapes_reuse_the_double_buffer(ct, ctx):
    """Consecutive calls with different (F, K) on one context: each call's in-kernel zeroing of
    the other accumulator half must cover the next call's extent (host bookkeeping)."""
    rng = np.random.default_rng(11)
    shapes = [(3, 64), (30, 512), (2, 16), (30, 512), (64, 256), (1, 1), (64, 256)]
    est = cf.Estimator()
    for F, K in shapes:
        dur, off = random_csr(rng, F, 30_000)
        cp, ocost, ctxj, wj = params(ct, K, 25_000, 3)
        g = host(ct.ct_fit_ttl(ctx, torch.from_numpy(dur).cuda(), off, cp, est))
        o = oracle_fit(dur, off, ocost, ctxj, wj, est)
        for x, y in zip(g, o):
            assert np.array_equal(x, y), (F, K)


@pytest.mark.parametrize("K", [899, 900, 1024])
def test_large_grid_lane_replicas(ct, ctx, K):
    """K = 899 is the largest grid whose 32-replica histogram ((K+1) x 256 B) fits in shared
    memory; 900 and 1024 run the 16-replica layout (two lanes per replica)."""
    rng = np.random.default_rng(K)
    dur, off = random_csr(rng, 4, 120_000)
    point = np.full(50_000, 3_000_000, np.int32)  # a point mass: every lane hits one bucket
    dur = np.concatenate([dur, point])
    off = np.concatenate([off, [off[-1] + len(point)]]).astype(np.int64)
    cp, ocost, ctxj, wj = params(ct, K, 20_000, 2)
    est = cf.Estimator()
    g = host(ct.ct_fit_ttl(ctx, torch.from_numpy(dur).cuda(), off, cp, est))
    o = oracle_fit(dur, off, ocost, ctxj, wj, est)
    for x, y in zip(g, o):
        assert np.array_equal(x, y)
