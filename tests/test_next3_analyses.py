"""NEXT-3 analyses: the turn-scaling workload transform of the robustness
study and estimator convergence (Fig. mean_estimate_both).

The transform is input generation (ctgen); the analyses run the oracle here and the CUDA path in
the GPU test, which must agree byte for byte.
"""
import numpy as np
import pytest

from ctgen import configs as cf
from ctgen import traces
from oracle import oracle as O


def test_turn_scaling_shapes():
    tr = traces.generate(2, 6, n_bfcl=3, mix="mix", ctx_cap=8192 * 16, stream=4)
    for k in (1, 2, 3, 5):
        t2 = traces.turn_scaling(tr, k)
        assert np.array_equal(t2.programs["nturns"], tr.programs["nturns"] * k)
        # token volume preserved within rounding (±1 per turn and field)
        v0 = tr.turns[:, 0].astype(np.int64).sum() + tr.turns[:, 1].astype(np.int64).sum()
        v1 = t2.turns[:, 0].astype(np.int64).sum() + t2.turns[:, 1].astype(np.int64).sum()
        assert abs(v1 - v0) <= 2 * k * tr.turns.shape[0]
        # exactly one final turn (no tool) per program; every other turn calls a tool
        last = t2.programs["turn0"] + t2.programs["nturns"] - 1
        assert np.all(t2.turns[last, 2] == -1)
        assert (t2.turns[:, 2] == -1).sum() == len(t2.programs)
        assert np.all(t2.turns[t2.turns[:, 2] >= 0, 3] >= 1)


def test_turn_scaling_pinning_gain_grows_with_turns():
    """'Each additional turn is a potential idle bubble if the program is not pinned'
    (PAPER.md:505-507): Continuum's JCT advantage over program-FCFS grows with k."""
    tr = traces.generate(4, 16, n_bfcl=8, mix="mix", ctx_cap=8192 * 16, stream=3)
    gains = []
    for k in (1, 2, 3, 4, 5):
        t2 = traces.turn_scaling(tr, k)
        sw = cf.Sweep(4, [cf.gap_from_jps(0.13)], [8192], [cf.PROG_FCFS, cf.CONTINUUM])
        s, _ = O.simulate(t2, sw, cf.ENGINE_8B, n_threads=8, want_jct=False)
        assert np.all((s[:, 0] & 0xFFFFFFFF) == 0)
        gains.append(int(s[0::2, 2].sum() - s[1::2, 2].sum()))
    assert all(g > 0 for g in gains)
    assert all(a < b for a, b in zip(gains, gains[1:]))


def test_estimator_convergence_two_point():
    """SPEC.md:657 (AC12) analog: two-point tool {0.1 s, 1.9 s} (sigma 0.9 s).  SPEC's "within
    5 % after 200 samples in >= 95 % of seeds" is statistically impossible here (sd of the mean
    = 64 ms, so P(|err| <= 50 ms) ~ 0.56); the pinned properties are the 3-sigma band
    (>= 95 % of 100 seeds, expected 99.7 %) and the bound's width B - mean shrinking with n."""
    rng = np.random.default_rng(12)
    lq = cf.lq_from_delta(0.05)
    b = 10_000_000
    ok = 0
    widths = {10: [], 50: [], 200: []}
    for _ in range(100):
        xs = np.where(rng.random(200) < 0.5, 100_000, 1_900_000)
        for n in widths:
            r = O.stats_row(xs[:n])
            s2 = int(np.uint64(r[2])) + (int(np.uint64(r[3])) << 64)
            widths[n].append(O.bernstein(n, int(r[1]), s2, lq, b) - int(r[1]) // n)
        ok += abs(xs.mean() - 1_000_000) <= 3 * 900_000 / np.sqrt(200)
    assert ok >= 95
    m = [np.mean(widths[n]) for n in (10, 50, 200)]
    assert m[0] > m[1] > m[2] > 0


@pytest.mark.gpu
def test_turn_scaling_gpu_parity():
    import torch
    import paper_2511_02230_b200 as ct
    ctx = ct.Context(0)
    tr = traces.generate(8, 16, n_bfcl=8, mix="mix", ctx_cap=8192 * 16, stream=3)
    for k in (1, 3, 5):
        t2 = traces.turn_scaling(tr, k)
        sw = cf.Sweep(8, cf.rate_axis(4, 0.05, 0.5), [8192],
                      [cf.PROG_FCFS, cf.CONTINUUM, cf.AUTELLIX, cf.INFERCEPT])
        g, gj = ct.ct_simulate_batch(ctx, ct.DeviceTrace(t2), sw, cf.ENGINE_8B, jct=True)
        torch.cuda.synchronize()
        o, oj = O.simulate(t2, sw, cf.ENGINE_8B, n_threads=8)
        assert np.array_equal(g.cpu().numpy(), o) and np.array_equal(gj.cpu().numpy(), oj)
