"""NEXT-4: integer-only trace synthesis (ctgen/synth.py) and its on-device twin
(ct_synthesize_traces), which must write the same bytes; replay of synthesised traces against
the oracle."""
import numpy as np
import pytest

from ctgen import configs as cf
from ctgen import synth, traces
from oracle import oracle as O


def test_synth_shapes_match_generate():
    """Same workload shapes as traces.generate (turns per program, token and duration means,
    class mix, context cap) within sampling error."""
    sp = synth.params(ctx_cap=8192 * 16, n_bfcl=16)
    a = synth.synthesize(sp, 0, 256, 32)
    b = traces.generate(256, 32, n_bfcl=16, mix="mix", ctx_cap=8192 * 16)
    for x in (a, b):
        assert x.pclass.reshape(256, 32).sum(axis=1).tolist() == [16] * 256
    ta, tb = a.turns, b.turns
    assert abs(len(ta) / len(tb) - 1) < 0.05
    for col in (0, 1):
        assert abs(ta[:, col].mean() / tb[:, col].mean() - 1) < 0.05
    da, db = ta[ta[:, 2] >= 0, 3], tb[tb[:, 2] >= 0, 3]
    assert abs(np.median(da) / np.median(db) - 1) < 0.1
    # structure: one final turn per program, context cap respected, arrivals non-decreasing
    assert (ta[:, 2] == -1).sum() == len(a.programs)
    for i in range(0, len(a.programs), 97):
        t0, nt = a.programs["turn0"][i], a.programs["nturns"][i]
        assert ta[t0:t0 + nt, :2].sum() <= sp.ctx_cap
    arr = a.programs["arr_q"].reshape(256, 32)
    assert np.all(np.diff(arr, axis=1) >= 0)


def test_synth_quantile_tables_pin_distributions():
    """The 16-bit interpolated quantile map reproduces the table's distribution: the empirical
    median of 2^16 draws from the SWE decode table equals the lognormal median (200)."""
    sp = synth.params()
    h = traces._key(5, np.arange(1 << 16, dtype=np.uint64), 15)
    x = synth._quantile_rows(sp.dec, np.zeros(1 << 16, np.int64), h)
    assert abs(np.median(x) - 200) <= 3
    assert x.min() >= 16 and x.max() <= 2048
    # exponential gaps: mean 1 (in Q20) within 2 %
    g = synth._quantile_rows(sp.exp[None, :], np.zeros(1 << 16, np.int64), h)
    assert abs(g.mean() / 2**20 - 1) < 0.02


def test_synth_replay_on_oracle():
    """Synthesised traces are ordinary trace sets for the oracle."""
    sp = synth.params(ctx_cap=8192 * 16, n_bfcl=4)
    tr = synth.synthesize(sp, 10, 3, 8)
    sw = cf.Sweep(3, [cf.gap_from_jps(0.2)], [8192], [cf.PROG_FCFS, cf.CONTINUUM])
    s, _ = O.simulate(tr, sw, cf.ENGINE_8B)
    assert np.all((s[:, 0] & 0xFFFFFFFF) == 0)


@pytest.mark.gpu
@pytest.mark.parametrize("P,S,nb,cap", [(32, 300, 16, 8192 * 16), (1, 40, 0, 8192), (200, 20, 0, 16384 * 16),
                                        (77, 33, 77, 20000), (256, 4, 100, 131072)])
def test_synth_device_bytes(P, S, nb, cap):
    import torch
    import paper_2511_02230_b200 as ct
    ctx = ct.Context(0)
    sp = synth.params(stream=3, ctx_cap=cap, n_bfcl=nb)
    g = ct.ct_synthesize_traces(ctx, sp, 1000, S, P)
    torch.cuda.synchronize()
    ref = synth.synthesize(sp, 1000, S, P)
    assert np.array_equal(g.programs.cpu().numpy(), np.ascontiguousarray(ref.programs).view(np.uint8))
    assert np.array_equal(g.turns.cpu().numpy(), ref.turns)


@pytest.mark.gpu
def test_synth_device_replay_parity():
    """Replay straight from synthesised HBM traces == oracle on the reference bytes."""
    import torch
    import paper_2511_02230_b200 as ct
    ctx = ct.Context(0)
    sp = synth.params(ctx_cap=8192 * 16, n_bfcl=16)
    g = ct.ct_synthesize_traces(ctx, sp, 0, 16, 32)
    sw = cf.Sweep(16, cf.rate_axis(3), [8192], [cf.PROG_FCFS, cf.CONTINUUM, cf.ttl_grid(2_000_000)])
    s, j = ct.ct_simulate_batch(ctx, g, sw, cf.ENGINE_8B, jct=True)
    torch.cuda.synchronize()
    os_, oj = O.simulate(synth.synthesize(sp, 0, 16, 32), sw, cf.ENGINE_8B, n_threads=8)
    assert np.array_equal(s.cpu().numpy(), os_) and np.array_equal(j.cpu().numpy(), oj)


@pytest.mark.gpu
def test_synth_turns_cap_too_small():
    import paper_2511_02230_b200 as ct
    from paper_2511_02230_b200 import _lib
    ctx = ct.Context(0)
    with pytest.raises(_lib.CtError):
        ct.ct_synthesize_traces(ctx, synth.params(), 0, 8, 32, turns_cap=10)
