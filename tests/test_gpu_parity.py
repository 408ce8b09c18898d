"""GPU parity: libcontinuum (through the C ABI) vs the CPU oracle, byte for byte.

Every replica's 128-B summary and every per-program JCT must be identical (integer
arithmetic end to end).  Sizes span several warps/CTAs, every
slots-per-lane variant (P <= 32, 64, 128, 256), ragged tails, edge cases, and — in the
launch configuration bench.py times — sampled replicas of the full BASELINE configs.
"""
import random
from dataclasses import replace

import numpy as np
import pytest
import torch

from ctgen import configs as cf
from ctgen import traces
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_2511_02230_b200 import build
    build.build()
    import paper_2511_02230_b200 as ct
    return ct.Context(0)


def gpu_run(ctx, tr, sw, eng, rb=0, re=None, jct=True):
    import paper_2511_02230_b200 as ct
    dt = ct.DeviceTrace(tr)
    s, j = ct.ct_simulate_batch(ctx, dt, sw, eng, rb, re, jct=jct)
    torch.cuda.synchronize()
    return s.cpu().numpy(), (j.cpu().numpy() if j is not None else None)


def assert_same(gs, gj, os_, oj):
    bad = np.nonzero(np.any(gs != os_, axis=1))[0]
    assert bad.size == 0, "summary mismatch at replicas %s:\nGPU %s\nORA %s" % (
        bad[:5], gs[bad[:2]], os_[bad[:2]])
    if gj is not None:
        badj = np.nonzero(np.any(gj != oj, axis=1))[0]
        assert badj.size == 0, "jct mismatch at %s" % badj[:5]


UNIT = cf.Engine(c0_ps=10**6, c_pf_ps=10**6, c_kv_ps=0, c_h2d_ps=5 * 10**5, bs=1, max_batch=256,
                 dram_blocks=1000)


def test_goldens(ctx):
    G1 = traces.tiny([(0, [(10, 2, 0, 5), (3, 1, -1, 0)])])
    sw = cf.Sweep(1, [1 << 20], [100], [cf.ttl_grid(5), cf.ttl_grid(4), cf.PROG_FCFS, cf.VLLM,
                                        cf.VLLM_LMCACHE])
    gs, gj = gpu_run(ctx, G1, sw, UNIT)
    assert list(gj[:, 0]) == [21, 33, 33, 33, 27]
    os_, oj = O.simulate(G1, sw, UNIT)
    assert_same(gs, gj, os_, oj)
    G2 = traces.tiny([(0, [(10, 2, 0, 20), (2, 1, -1, 0)]), (1, [(10, 5, -1, 0)])])
    sw = cf.Sweep(1, [1 << 20], [30, 20], [cf.ttl_grid(100), cf.PROG_FCFS])
    gs, gj = gpu_run(ctx, G2, sw, UNIT)
    assert [list(x) for x in gj] == [[45, 25], [57, 25], [47, 26], [47, 26]]


def random_tiny_set(rng, n_seeds, P=3, n_tools=2):
    progs = []
    for _ in range(n_seeds):
        arr = sorted(rng.randint(0, 20) for _ in range(P))
        for p in range(P):
            T = rng.randint(1, 3)
            ts = [(rng.randint(0, 6), rng.randint(1, 4), rng.randint(0, n_tools - 1), rng.randint(1, 30))
                  for _ in range(T)]
            ts[-1] = (ts[-1][0], ts[-1][1], -1, 0)
            progs.append((arr[p], ts))
    tr = traces.tiny(progs, n_tools=n_tools)
    tr.n_seeds, tr.n_programs = n_seeds, P
    return tr


def random_policies(rng, n):
    out = []
    for _ in range(n):
        out.append(cf.Policy(priority=rng.choice([0, 0, 1, 2]),
                             pause=rng.choice([0, 1, 1, 2, 3, 4]), dram=rng.choice([0, 1]),
                             flags=rng.choice([0, 0, 1, 2, 3]), t_pin_us=rng.randint(0, 30),
                             t_thresh_us=rng.choice([cf.ALWAYS, rng.randint(1, 30)])))
    return out


@pytest.mark.parametrize("seed", range(6))
def test_random_tiny_instances(ctx, seed):
    rng = random.Random(1000 + seed)
    tr = random_tiny_set(rng, 300)
    eng = cf.Engine(c0_ps=rng.randint(1, 3 * 10**6), c_pf_ps=rng.choice([0, 5 * 10**5, 10**6]),
                    c_kv_ps=rng.choice([0, 10**4, 2 * 10**5]), c_h2d_ps=rng.randint(1, 2 * 10**6),
                    bs=rng.choice([1, 2, 4]), max_batch=rng.choice([1, 2, 256]),
                    dram_blocks=rng.randint(0, 12), max_iters=rng.choice([10**6, 40]))
    est = cf.Estimator(b_us=rng.choice([5, 40]), t_def_us=rng.randint(1, 40), n_min=rng.randint(1, 3),
                       a_num=rng.randint(0, 2), a_den=rng.choice([1, 3]), ttl_max_us=rng.choice([0, 25]))
    fitted = np.array([[rng.randint(0, 30) for _ in range(3)] for _ in range(2)], np.int64)
    sw = cf.Sweep(300, [1 << 20, 3 << 19], [6, 11, 18], random_policies(rng, 6), est, fitted)
    gs, gj = gpu_run(ctx, tr, sw, eng)
    os_, oj = O.simulate(tr, sw, eng, n_threads=8)
    assert_same(gs, gj, os_, oj)


ALL_POLICIES = [cf.VLLM, cf.VLLM_LMCACHE, cf.PROG_FCFS, cf.CONTINUUM, cf.ttl_grid(500_000),
                cf.ttl_grid(30_000_000), cf.simplified(5_000_000, 1_000_000),
                cf.Policy(cf.PRIO_PROG_FCFS, cf.PAUSE_PAPER, dram=1),
                cf.Policy(cf.PRIO_PROG_FCFS, cf.PAUSE_PAPER, flags=cf.FLAG_STEP_EXPIRY),
                cf.Policy(cf.PRIO_PROG_FCFS, cf.PAUSE_FIXED, flags=cf.FLAG_VICTIMS_ANY,
                          t_pin_us=20_000_000),
                cf.Policy(cf.PRIO_REQ_FCFS, cf.PAUSE_FITTED, dram=1),
                cf.Policy(cf.PRIO_PROG_FCFS, cf.PAUSE_FITTED, flags=cf.FLAG_STEP_EXPIRY),
                cf.AUTELLIX, cf.INFERCEPT,
                cf.Policy(cf.PRIO_PLAS, cf.PAUSE_PAPER, dram=1),
                cf.Policy(cf.PRIO_PROG_FCFS, cf.PAUSE_INFERCEPT, flags=cf.FLAG_STEP_EXPIRY)]


@pytest.mark.parametrize("P", [1, 7, 32, 33, 64, 70, 100, 128, 150, 180, 200, 256])
def test_workloads_all_policies(ctx, P):
    n_seeds = 6 if P <= 64 else 2
    tr = traces.generate(n_seeds, P, mix="mix", ctx_cap=8192, stream=P)
    fitted = np.tile(np.array([[0, 200_000, 3_000_000, 60_000_000]], np.int64), (tr.n_tools, 1))
    eng = cf.Engine(**{**cf.ENGINE_8B.__dict__, "dram_blocks": 40 * P})
    sw = cf.Sweep(n_seeds, [200_000, 3_000_000], [600, 20 * P + 600], ALL_POLICIES, fitted=fitted)
    gs, gj = gpu_run(ctx, tr, sw, eng)
    os_, oj = O.simulate(tr, sw, eng, n_threads=8)
    assert_same(gs, gj, os_, oj)
    assert np.mean((gs[:, 0] & 0xFFFFFFFF) == 0) > 0.8


def test_sharding_and_host_path(ctx):
    import paper_2511_02230_b200 as ct
    tr = traces.generate(8, 32, n_bfcl=16, mix="mix", ctx_cap=8192 * 16, stream=5)
    sw = cf.Sweep(8, cf.rate_axis(4), [8192], [cf.ttl_grid(t) for t in cf.ttl_axis(8)])
    full, fj = gpu_run(ctx, tr, sw, cf.ENGINE_8B)
    R = sw.n_replicas
    parts = [gpu_run(ctx, tr, sw, cf.ENGINE_8B, a, b) for a, b in [(0, 37), (37, 38), (38, R)]]
    assert np.array_equal(full, np.concatenate([p[0] for p in parts]))
    assert np.array_equal(fj, np.concatenate([p[1] for p in parts]))
    hs = torch.empty((R, 16), dtype=torch.int64).pin_memory()
    hj = torch.empty((R, 32), dtype=torch.int64).pin_memory()
    ct.ct_simulate_batch_host(ctx, tr, sw, cf.ENGINE_8B, 0, R, hs, hj)
    assert np.array_equal(hs.numpy(), full) and np.array_equal(hj.numpy(), fj)
    # empty range is a no-op
    s, _ = ct.ct_simulate_batch(ctx, ct.DeviceTrace(tr), sw, cf.ENGINE_8B, 5, 5, jct=False)
    assert s.shape[0] == 0


def test_edge_statuses(ctx):
    tr = traces.tiny([(0, [(100, 1, -1, 0)]), (5, [(1, 50, -1, 0)])])
    sw = cf.Sweep(1, [1 << 20], [50, 200], [cf.PROG_FCFS])
    eng = cf.Engine(**{**UNIT.__dict__, "max_iters": 20})
    gs, gj = gpu_run(ctx, tr, sw, eng)
    os_, oj = O.simulate(tr, sw, eng)
    assert_same(gs, gj, os_, oj)
    assert list(gs[:, 0] & 0xFFFFFFFF) == [cf.STATUS_UNSCHEDULABLE, cf.STATUS_EVENT_BUDGET]


def test_invalid_arguments_rejected(ctx):
    import paper_2511_02230_b200 as ct
    from paper_2511_02230_b200 import _lib
    tr = traces.tiny([(0, [(1, 1, -1, 0)])])
    sw = cf.Sweep(1, [1 << 20], [10], [cf.Policy(pause=cf.PAUSE_FITTED)])  # FITTED without table
    with pytest.raises(_lib.CtError):
        ct.ct_simulate_batch(ctx, ct.DeviceTrace(tr), sw, UNIT)
    bad = cf.Engine(**{**UNIT.__dict__, "c0_ps": 0})
    with pytest.raises(_lib.CtError):
        ct.ct_simulate_batch(ctx, ct.DeviceTrace(tr), cf.Sweep(1, [1], [10], [cf.PROG_FCFS]), bad)


# ---- TTL fit ----------------------------------------------------------------------------------
def fit_both(ctx, dur, off, K, step, J, c_pf, c_pin, est, avg=(0, 0), a=(1, 10)):
    import paper_2511_02230_b200 as ct
    ctxj = [int(500 * 2**j) % 200_000 + 16 for j in range(J)]
    wj = [j + 1 for j in range(J)]
    cp = ct.cost_params(c_pf, c_pin, 16, a[0], a[1], step, K, ctxj, wj, avg)
    d = torch.from_numpy(np.ascontiguousarray(dur, np.int32)).cuda()
    ga, gp, gst = ct.ct_fit_ttl(ctx, d, off, cp, est)
    torch.cuda.synchronize()
    oa, op, ost = O.fit(dur, off, [c_pf, c_pin, 16, a[0], a[1], step, K, J], ctxj, wj,
                        est.as_array(), avg)
    return (ga.cpu().numpy(), gp.cpu().numpy(), gst.cpu().numpy()), (oa, op, ost)


@pytest.mark.parametrize("seed", range(8))
def test_fit_parity_random(ctx, seed):
    rng = np.random.default_rng(seed)
    F = int(rng.integers(1, 12))
    sizes = rng.integers(0, 3000, size=F)
    sizes[rng.integers(0, F)] = int(rng.integers(0, 5))  # a tool below N
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    n = int(off[-1])
    dur = np.clip(rng.lognormal(np.log(rng.uniform(5e4, 5e6)), rng.uniform(0.1, 1.5), n), 0, 2**31 - 1).astype(np.int32)
    dur[rng.random(n) < 0.05] = 0
    K = int(rng.choice([1, 2, 17, 64, 256, 1024]))
    step = int(rng.choice([1, 999, 50_000, 250_000]))
    J = int(rng.integers(1, 9))
    est = cf.Estimator(n_min=int(rng.integers(1, 8)))
    g, o = fit_both(ctx, dur, off, K, step, J, 13_400_000, int(rng.integers(0, 3000)), est,
                    avg=(int(rng.integers(0, 500)), int(rng.integers(0, 50))))
    for name, x, y in zip(("ttl_argmax", "ttl_paper", "stats"), g, o):
        assert np.array_equal(x, y), (name, K, step, J, x, y)


def test_fit_point_mass_and_alignment(ctx):
    # misaligned CSR segments (head/tail paths), point mass (cd-like) and duplicates
    sizes = [1, 3, 5, 7, 4096 + 3, 70_001]
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    dur = np.full(int(off[-1]), 100_000, np.int32)
    dur[: off[4]] = np.arange(int(off[4])) * 7919 % 3_000_000
    g, o = fit_both(ctx, dur, off, 256, 50_000, 4, 13_400_000, 50, cf.Estimator())
    for x, y in zip(g, o):
        assert np.array_equal(x, y)


def test_jct_stats_parity(ctx):
    import paper_2511_02230_b200 as ct
    tr = traces.generate(16, 32, n_bfcl=16, mix="mix", ctx_cap=8192 * 16, stream=9)
    sw = cf.Sweep(16, cf.rate_axis(3), [8192, 2000], [cf.ttl_grid(t) for t in cf.ttl_axis(4)])
    s, _ = ct.ct_simulate_batch(ctx, ct.DeviceTrace(tr), sw, cf.ENGINE_8B, jct=False)
    cs = ct.ct_jct_stats(ctx, s, sw.n_cells).cpu().numpy()
    ocs = O.jct_stats(s.cpu().numpy(), sw.n_cells)
    assert np.array_equal(cs, ocs)


@pytest.mark.parametrize("K", [300, 512, 1024])
def test_fit_large_grids(ctx, K):
    """Grids of up to 899 points keep the 32-replica CTA histogram; K 1024 runs the 16-replica
    layout (tests/test_gpu_fit.py covers the boundary)."""
    rng = np.random.default_rng(K)
    sizes = [5, 100_003, 7, 250_000, 1]
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    dur = rng.integers(0, 60_000_000, int(off[-1])).astype(np.int32)
    g, o = fit_both(ctx, dur, off, K, 50_000, 3, 13_400_000, 40, cf.Estimator())
    for x, y in zip(g, o):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("case", range(6))
def test_fit_estimator_extremes(ctx, case):
    """Bernstein / CalcTTL at the validated extremes (b, T_default up to 2^40 - 1, delta down to
    1e-9, tiny and large n, large alpha and AvgTurns): the 128-bit divisions take both the
    double-estimate fast path and the generic path, and must stay exact."""
    rng = np.random.default_rng(100 + case)
    F = 6
    sizes = [1, 2, 3, int(rng.integers(5, 50)), int(rng.integers(1000, 5000)), 20_000]
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    n = int(off[-1])
    hi = [2**31 - 1, 2**28, 5_000_000][case % 3]
    dur = rng.integers(0, hi, n).astype(np.int32)
    dur[: 3] = 2**31 - 1
    big, b31 = 2**40 - 1, 2**31 - 1  # validated maxima: T_default, ttl_max < 2^40; b < 2^31 (fit)
    est = [cf.Estimator(delta=1e-9, b_us=b31, t_def_us=big, n_min=1, a_num=1000, a_den=1, ttl_max_us=big),
           cf.Estimator(delta=0.999, b_us=b31, t_def_us=7, n_min=2, a_num=0, a_den=3, ttl_max_us=0),
           cf.Estimator(delta=1e-6, b_us=2**30, t_def_us=10**12, n_min=1, a_num=7, a_den=9, ttl_max_us=big),
           cf.Estimator(delta=0.05, b_us=60_000_000, t_def_us=10_000_000, n_min=5, ttl_max_us=0),
           cf.Estimator(delta=1e-9, b_us=1, t_def_us=big, n_min=3, a_num=5, a_den=1, ttl_max_us=big),
           cf.Estimator(delta=0.3, b_us=b31, t_def_us=2**39, n_min=1, a_num=1, a_den=10**6, ttl_max_us=big)][case]
    avg = [(10**6, 3), (0, 0), (2**31, 1), (500, 40), (7, 7), (1, 2**20)][case]
    g, o = fit_both(ctx, dur, off, 64, 250_000, 2, 13_400_000, 40, est, avg=avg)
    for name, x, y in zip(("ttl_argmax", "ttl_paper", "stats"), g, o):
        assert np.array_equal(x, y), (name, case, x, y)


@pytest.mark.parametrize("kind", ["grid", "prog"])
@pytest.mark.parametrize("P", [1, 17, 32, 33, 70, 100, 130, 180, 200, 256])
def test_ttl_grid_32bit_horizon(ctx, P, kind):
    """TTL-grid-only and program-FCFS-only sweeps run the 32-bit-time kernels (P <= 32: MODE 1 / 3;
    P > 32: MODE 4 plus the list-driven 64-bit launch).  Long inter-arrival gaps (up to 2^30 µs),
    TTLs up to 2^40 µs and slow engines push replica horizons past 2^32 µs, where the replica
    must fall back to the 64-bit path: both must agree with the oracle byte for byte, as must the
    per-program bubble output (always the 64-bit path) and EVENT_BUDGET replicas."""
    import paper_2511_02230_b200 as ct
    n_seeds = 4 if P <= 32 else 2
    tr = traces.generate(n_seeds, P, n_bfcl=P // 2, mix="mix", ctx_cap=1500 * 16, stream=40 + P)
    gaps = [1 << 20, 300_000_000, (1 << 30) - 1]
    pols = [cf.ttl_grid(t) for t in (0, 1, 2_000_000, 600_000_000, 1 << 40)] + [cf.PROG_FCFS]
    fitted = None
    if kind == "prog":  # program-FCFS class with the estimator (32-bit kernel MODE 3)
        fitted = np.tile(np.array([[0, 200_000, 3_000_000, 1 << 40]], np.int64), (tr.n_tools, 1))
        pols = [cf.CONTINUUM, cf.simplified(5_000_000, 2_000_000), cf.simplified(1 << 40, 10**9),
                cf.CONTINUUM_FITTED, cf.ttl_grid(2_000_000), cf.PROG_FCFS]
        # request FCFS is in the simple class too (P <= 32: MODE 3; P > 32: MODE 4 with the
        # generic 64-bit kernel as the fallback launch)
        pols += [cf.VLLM, cf.Policy(cf.PRIO_REQ_FCFS, cf.PAUSE_PAPER)]
    span, budget = 0, False
    for eng in (cf.ENGINE_8B, cf.Engine(**{**cf.ENGINE_8B.__dict__, "c0_ps": 4 * 10**11}),
                cf.Engine(**{**cf.ENGINE_8B.__dict__, "max_iters": 2000 if P == 1 else 20000})):
        sw = cf.Sweep(n_seeds, gaps, [4096 if P <= 32 else 30 * P, 1600], pols, fitted=fitted)
        os_, oj, ob = O.simulate(tr, sw, eng, n_threads=8, want_bubble=True)
        # without the bubble output: the 32-bit kernel (and its fallback); with it: 64-bit path
        s, j = ct.ct_simulate_batch(ctx, ct.DeviceTrace(tr), sw, eng, jct=True)
        torch.cuda.synchronize()
        assert_same(s.cpu().numpy(), j.cpu().numpy(), os_, oj)
        li = ctx.last_launch()  # the specialised 32-bit kernel ran (DESIGN.md §8 MODE)
        # (P <= 32 "prog": TTL-grid policies run MODE 1 and the others MODE 3 in a second
        # launch over their policy subset: kernel_mode 13)
        assert li["kernel_mode"] == ((4 if kind == "grid" else 5) if P > 32 else
                                     1 if kind == "grid" else 13), li
        assert li["launches"] == (1 if P <= 32 and kind == "grid" else 2) + 1  # + trace check
        R = sw.n_replicas  # a shard: fallback replicas are indexed relative to replica_begin
        s, j = ct.ct_simulate_batch(ctx, ct.DeviceTrace(tr), sw, eng, R // 3, 2 * R // 3, jct=True)
        torch.cuda.synchronize()
        assert_same(s.cpu().numpy(), j.cpu().numpy(), os_[R // 3: 2 * R // 3], oj[R // 3: 2 * R // 3])
        s, j, b = ct.ct_simulate_batch(ctx, ct.DeviceTrace(tr), sw, eng, jct=True, bubble=True)
        torch.cuda.synchronize()
        assert_same(s.cpu().numpy(), j.cpu().numpy(), os_, oj)
        assert np.array_equal(b.cpu().numpy(), ob)
        span = max(span, int(np.max(os_[:, 7])))
        budget |= bool(np.any(os_[:, 0] == 2))
    assert budget and (P == 1 or span > 2**32)  # both the fallback and EVENT_BUDGET were exercised


EXT_POLICIES = [cf.VLLM, cf.VLLM_LMCACHE, cf.Policy(cf.PRIO_PROG_FCFS, cf.PAUSE_EVICT, dram=1),
                cf.Policy(cf.PRIO_PROG_FCFS, cf.PAUSE_PAPER, dram=1),
                cf.Policy(cf.PRIO_PROG_FCFS, cf.PAUSE_FITTED, dram=1), cf.AUTELLIX, cf.INFERCEPT,
                cf.Policy(cf.PRIO_PLAS, cf.PAUSE_PAPER, dram=1),
                cf.Policy(cf.PRIO_PLAS, cf.PAUSE_INFERCEPT, dram=0),
                cf.Policy(cf.PRIO_PROG_FCFS, cf.PAUSE_INFERCEPT, dram=1),
                cf.Policy(cf.PRIO_PROG_FCFS, cf.PAUSE_FIXED, dram=1, t_pin_us=2_000_000),
                cf.Policy(cf.PRIO_REQ_FCFS, cf.PAUSE_FIXED, dram=1, t_pin_us=5_000_000,
                          t_thresh_us=1_000_000)]


@pytest.mark.parametrize("P", [1, 7, 17, 32])
def test_extended_class_32bit(ctx, P):
    """Sweeps whose policies are all in the extended class (DRAM tier, PLAS, InferCept; flags 0)
    run the 32-bit P <= 32 kernel (MODE 6) with the 64-bit fallback past the 2^32 µs horizon
    (long gaps, a slow engine, slow H2D loads) and EVENT_BUDGET replicas: byte equality."""
    import paper_2511_02230_b200 as ct
    n_seeds = 4
    tr = traces.generate(n_seeds, P, n_bfcl=P // 2, mix="mix", ctx_cap=1500 * 16, stream=60 + P)
    fitted = np.tile(np.array([[0, 200_000, 3_000_000, 1 << 40]], np.int64), (tr.n_tools, 1))
    gaps = [1 << 20, 300_000_000, (1 << 30) - 1]
    engines = [cf.Engine(**{**cf.ENGINE_8B.__dict__, "dram_blocks": 30 * P}),
               cf.Engine(**{**cf.ENGINE_8B.__dict__, "dram_blocks": 3000, "c_h2d_ps": 4 * 10**11}),
               cf.Engine(**{**cf.ENGINE_8B.__dict__, "c0_ps": 4 * 10**11, "dram_blocks": 500}),
               cf.Engine(**{**cf.ENGINE_8B.__dict__, "dram_blocks": 800,
                            "max_iters": 2000 if P == 1 else 20000})]
    reloads = 0
    for eng in engines:
        sw = cf.Sweep(n_seeds, gaps, [1600, 4096], EXT_POLICIES, fitted=fitted)
        s, j = ct.ct_simulate_batch(ctx, ct.DeviceTrace(tr), sw, eng, jct=True)
        torch.cuda.synchronize()
        os_, oj = O.simulate(tr, sw, eng, n_threads=8)
        assert_same(s.cpu().numpy(), j.cpu().numpy(), os_, oj)
        assert ctx.last_launch()["kernel_mode"] == 6
        reloads += int(os_[:, 15].sum())
    assert reloads > 0  # DRAM reloads happened


@pytest.mark.parametrize("seed", range(4))
def test_random_tiny_extended_class(ctx, seed):
    rng = random.Random(2000 + seed)
    tr = random_tiny_set(rng, 300)
    eng = cf.Engine(c0_ps=rng.randint(1, 3 * 10**6), c_pf_ps=rng.choice([0, 5 * 10**5, 10**6]),
                    c_kv_ps=rng.choice([0, 10**4, 2 * 10**5]), c_h2d_ps=rng.randint(1, 2 * 10**6),
                    bs=rng.choice([1, 2, 4]), max_batch=rng.choice([1, 2, 256]),
                    dram_blocks=rng.randint(0, 12), max_iters=rng.choice([10**6, 40]))
    est = cf.Estimator(b_us=rng.choice([5, 40]), t_def_us=rng.randint(1, 40), n_min=rng.randint(1, 3),
                       a_num=rng.randint(0, 2), a_den=rng.choice([1, 3]), ttl_max_us=rng.choice([0, 25]))
    fitted = np.array([[rng.randint(0, 30) for _ in range(3)] for _ in range(2)], np.int64)
    pols = [replace(p, flags=0) for p in random_policies(rng, 8)] + [cf.AUTELLIX]
    sw = cf.Sweep(300, [1 << 20, 3 << 19], [6, 11, 18], pols, est, fitted)
    gs, gj = gpu_run(ctx, tr, sw, eng)
    assert ctx.last_launch()["kernel_mode"] in (6, 16)  # 16: TTL-grid policies split off
    os_, oj = O.simulate(tr, sw, eng, n_threads=8)
    assert_same(gs, gj, os_, oj)
