"""GPU parity for NEXT-2 (vLLM-style KV growth with recompute preemption, R27-R30)
and the per-program bubble output (NEXT-3), through ct_simulate_batch_ex, byte for byte
against the oracle.  Growth runs the shared-memory replay path for every P (also P <= 32)."""
import random

import numpy as np
import pytest
import torch

from ctgen import configs as cf
from ctgen import traces
from oracle import oracle as O
from tests.test_gpu_parity import ALL_POLICIES, UNIT, random_policies

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_2511_02230_b200 import build
    build.build()
    import paper_2511_02230_b200 as ct
    return ct.Context(0)


def gpu_run(ctx, tr, sw, eng):
    import paper_2511_02230_b200 as ct
    s, j, b = ct.ct_simulate_batch(ctx, ct.DeviceTrace(tr), sw, eng, jct=True, bubble=True)
    torch.cuda.synchronize()
    return s.cpu().numpy(), j.cpu().numpy(), b.cpu().numpy()


def check(ctx, tr, sw, eng):
    g = gpu_run(ctx, tr, sw, eng)
    o = O.simulate(tr, sw, eng, n_threads=8, want_bubble=True)
    for name, x, y in zip(("summary", "jct", "bubble"), g, o):
        bad = np.nonzero(np.any(x != y, axis=1))[0]
        assert bad.size == 0, "%s mismatch at replicas %s:\nGPU %s\nORA %s" % (
            name, bad[:5], x[bad[:2]], y[bad[:2]])
    return g


GROW_UNIT = cf.Engine(**{**UNIT.__dict__, "kv_growth": 1})


def test_growth_hand_traces(ctx):
    tr = traces.tiny([(0, [(2, 4, -1, 0)]), (1, [(2, 4, -1, 0)])])
    s, j, b = check(ctx, tr, cf.Sweep(1, [1 << 20], [7], [cf.PROG_FCFS]), GROW_UNIT)
    assert list(j[0]) == [8, 13] and list(b[0]) == [0, 4] and s[0][11] == 3
    tr = traces.tiny([(0, [(1, 4, -1, 0)]), (0, [(1, 4, -1, 0)]), (1, [(3, 1, -1, 0)])])
    s, j, b = check(ctx, tr, cf.Sweep(1, [1 << 20], [6], [cf.VLLM]), GROW_UNIT)
    assert list(j[0]) == [6, 11, 14] and list(b[0]) == [0, 2, 10]


def random_growth_set(rng, n_seeds, P=3, n_tools=2):
    progs = []
    for _ in range(n_seeds):
        arr = sorted(rng.randint(0, 3) for _ in range(P))
        for p in range(P):
            T = rng.randint(1, 2)
            ts = [(rng.randint(1, 4), rng.randint(2, 8), rng.randint(0, n_tools - 1),
                   rng.randint(1, 30)) for _ in range(T)]
            ts[-1] = (ts[-1][0], ts[-1][1], -1, 0)
            progs.append((arr[p], ts))
    tr = traces.tiny(progs, n_tools=n_tools)
    tr.n_seeds, tr.n_programs = n_seeds, P
    return tr


@pytest.mark.parametrize("seed", range(6))
def test_growth_random_tiny(ctx, seed):
    rng = random.Random(2000 + seed)
    tr = random_growth_set(rng, 300)
    eng = cf.Engine(c0_ps=rng.randint(1, 3 * 10**6), c_pf_ps=rng.choice([0, 5 * 10**5, 10**6]),
                    c_kv_ps=rng.choice([0, 10**4, 2 * 10**5]), c_h2d_ps=rng.randint(1, 2 * 10**6),
                    bs=rng.choice([1, 2, 4]), max_batch=rng.choice([2, 256]),
                    dram_blocks=rng.randint(0, 12), max_iters=rng.choice([10**6, 40]), kv_growth=1)
    est = cf.Estimator(b_us=rng.choice([5, 40]), t_def_us=rng.randint(1, 40), n_min=rng.randint(1, 3),
                       a_num=rng.randint(0, 2), a_den=rng.choice([1, 3]), ttl_max_us=rng.choice([0, 25]))
    fitted = np.array([[rng.randint(0, 30) for _ in range(3)] for _ in range(2)], np.int64)
    sw = cf.Sweep(300, [1 << 20, 3 << 19], [8, 12, 16], random_policies(rng, 6), est, fitted)
    s, _, _ = check(ctx, tr, sw, eng)
    assert np.mean((s[:, 0] & 0xFFFFFFFF) == 0) > 0.2


@pytest.mark.parametrize("P", [1, 7, 32, 33, 64, 100, 200, 256])
def test_growth_workloads_all_policies(ctx, P):
    """Pools from tight (frequent preemption) to ample, every policy variant, DRAM on/off."""
    n_seeds = 4 if P <= 64 else 2
    tr = traces.generate(n_seeds, P, mix="mix", ctx_cap=8192, stream=100 + P)
    fitted = np.tile(np.array([[0, 200_000, 3_000_000, 60_000_000]], np.int64), (tr.n_tools, 1))
    eng = cf.Engine(**{**cf.ENGINE_8B.__dict__, "dram_blocks": 40 * P, "kv_growth": 1})
    sw = cf.Sweep(n_seeds, [200_000, 3_000_000], [700, 8 * P + 700, 40 * P + 700], ALL_POLICIES,
                  fitted=fitted)
    s, _, _ = check(ctx, tr, sw, eng)
    assert np.mean((s[:, 0] & 0xFFFFFFFF) == 0) > 0.8


@pytest.mark.parametrize("P", [7, 32, 70, 200])
def test_bubble_series_reserve_mode(ctx, P):
    """The per-program bubble output on the default engine (both replay paths)."""
    tr = traces.generate(3, P, mix="mix", ctx_cap=8192, stream=200 + P)
    eng = cf.Engine(**{**cf.ENGINE_8B.__dict__, "dram_blocks": 40 * P})
    sw = cf.Sweep(3, [200_000, 3_000_000], [600, 20 * P + 600], ALL_POLICIES[:8])
    s, _, b = check(ctx, tr, sw, eng)
    ok = (s[:, 0] & 0xFFFFFFFF) == 0
    assert np.array_equal(b[ok].sum(axis=1), s[ok, 6])  # per-program series sums to the total


# ---- chunked prefill (NEXT-2, R31-R32) ---------------------------------------------------------
def test_chunked_hand_trace(ctx):
    tr = traces.tiny([(0, [(6, 2, -1, 0)]), (0, [(3, 1, -1, 0)])])
    eng = cf.Engine(**{**UNIT.__dict__, "max_batch": 2, "prefill_chunk": 4})
    s, j, b = check(ctx, tr, cf.Sweep(1, [1 << 20], [100], [cf.PROG_FCFS]), eng)
    assert list(j[0]) == [12, 12] and list(b[0]) == [0, 5]


@pytest.mark.parametrize("seed", range(4))
def test_chunked_random_tiny(ctx, seed):
    rng = random.Random(3000 + seed)
    tr = random_growth_set(rng, 300)
    mb = rng.choice([1, 2, 3])
    eng = cf.Engine(c0_ps=rng.randint(1, 3 * 10**6), c_pf_ps=rng.choice([0, 5 * 10**5, 10**6]),
                    c_kv_ps=rng.choice([0, 10**4, 2 * 10**5]), c_h2d_ps=rng.randint(1, 2 * 10**6),
                    bs=rng.choice([1, 2, 4]), max_batch=mb, dram_blocks=rng.randint(0, 12),
                    max_iters=rng.choice([10**6, 40]), prefill_chunk=rng.choice([mb, 3, 5]) + mb)
    est = cf.Estimator(b_us=rng.choice([5, 40]), t_def_us=rng.randint(1, 40), n_min=rng.randint(1, 3))
    fitted = np.array([[rng.randint(0, 30) for _ in range(3)] for _ in range(2)], np.int64)
    sw = cf.Sweep(300, [1 << 20, 3 << 19], [12, 20, 40], random_policies(rng, 6), est, fitted)
    s, _, _ = check(ctx, tr, sw, eng)
    assert np.mean((s[:, 0] & 0xFFFFFFFF) == 0) > 0.3


@pytest.mark.parametrize("P", [1, 7, 32, 33, 100, 200])
def test_chunked_workloads_all_policies(ctx, P):
    """Token budgets from tight (prompts span several iterations) to ample."""
    n_seeds = 4 if P <= 64 else 2
    tr = traces.generate(n_seeds, P, mix="mix", ctx_cap=8192, stream=300 + P)
    fitted = np.tile(np.array([[0, 200_000, 3_000_000, 60_000_000]], np.int64), (tr.n_tools, 1))
    for budget in (512, 2048):
        eng = cf.Engine(**{**cf.ENGINE_8B.__dict__, "dram_blocks": 40 * P, "prefill_chunk": budget})
        sw = cf.Sweep(n_seeds, [200_000, 3_000_000], [700, 20 * P + 700], ALL_POLICIES,
                      fitted=fitted)
        s, _, _ = check(ctx, tr, sw, eng)
        assert np.mean((s[:, 0] & 0xFFFFFFFF) == 0) > 0.8


def test_chunked_invalid_combinations(ctx):
    import paper_2511_02230_b200 as ct
    from paper_2511_02230_b200 import _lib
    tr = traces.tiny([(0, [(1, 1, -1, 0)])])
    sw = cf.Sweep(1, [1 << 20], [10], [cf.PROG_FCFS])
    for bad in ({"prefill_chunk": 4, "max_batch": 8}, {"prefill_chunk": 64, "kv_growth": 1},
                {"prefill_chunk": -1}):
        with pytest.raises(_lib.CtError):
            ct.ct_simulate_batch(ctx, ct.DeviceTrace(tr), sw, cf.Engine(**{**UNIT.__dict__, **bad}))
