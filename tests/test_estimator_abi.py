"""The estimator calls of the C ABI (include/continuum.h: ct_bernstein / ct_calc_ttl_batch on
the device, ct_bernstein_ref / ct_calc_ttl_ref on the host) against the paper's worked examples
(tests/golden/spec_estimator_examples.txt: SPEC.md:263, 283-285) and against the oracle.

The host references are the library's own fixed-point helpers compiled for the host, so the
CPU tests here check the hot path's arithmetic without a GPU; the -m gpu tests run the same
examples through the device kernels.
"""
import math
import random
from dataclasses import replace

import numpy as np
import pytest

from ctgen import configs as cf
from oracle import oracle as O

S = 1_000_000
INVALID = -1


@pytest.fixture(scope="module")
def ct():
    from paper_2511_02230_b200 import build
    build.build()
    from paper_2511_02230_b200 import api
    return api


def stat(xs, b=None):
    """(n, s1, s2) of samples clamped to b."""
    xs = [min(int(x), b) if b is not None else int(x) for x in xs]
    return (len(xs), sum(xs), sum(x * x for x in xs))


def point_mass_row(value_us, n):
    return (n, n * value_us, n * value_us * value_us)


def spec_cases():
    """(name, g, f, est, n_done, turns_done, expected µs) from the golden file's CalcTTL lines;
    B_f = 5 s exactly: 2^30 samples of 5 s (sigma = 0; range term floor(3 b L_q / (n 2^32)) = 0
    with b = 5 s)."""
    five = point_mass_row(5 * S, 1 << 30)
    e40 = cf.Estimator(t_def_us=10 * S, a_num=1, a_den=10, ttl_max_us=0, b_us=5 * S, n_min=5)
    e30 = cf.Estimator(t_def_us=10 * S, a_num=1, a_den=10, ttl_max_us=30 * S, b_us=5 * S, n_min=5)
    e110 = cf.Estimator(t_def_us=10 * S, a_num=0, a_den=1, ttl_max_us=0)
    return [("calc_ttl_110", (0, 0, 0), (0, 0, 0), e110, 0, 0, 10 * S),  # expiry = now + 10 s
            ("calc_ttl_40", five, five, e40, 1, 10, 40 * S),
            ("calc_ttl_40_avg", five, five, e40, 3, 30, 40 * S),
            ("calc_ttl_clamp", five, five, e30, 1, 10, 30 * S),
            ("calc_ttl_no_done", five, five, e40, 0, 0, 20 * S)]


def test_golden_file_lists_the_cases():
    names = [l.split("|")[0].strip() for l in open("tests/golden/spec_estimator_examples.txt")
             if l.strip() and not l.startswith("#")]
    assert {"bernstein_n1", "calc_ttl_110", "calc_ttl_40", "calc_ttl_clamp"} <= set(names)


def test_host_ref_spec_examples(ct):
    # n = 1, mu = 2 s, b = 10 s, delta = .05 -> 124,830,336 µs (2 + 30 ln 60 s)
    e = cf.Estimator(b_us=10 * S)
    assert ct.ct_bernstein_ref(stat([2 * S]), e) == 124_830_336
    for name, g, f, est, d, td, want in spec_cases():
        assert ct.ct_calc_ttl_ref(g, f, est, d, td) == want, name


def test_host_ref_equals_oracle_random(ct):
    rng = random.Random(5)
    for _ in range(3000):
        b = rng.choice([10 * S, 60 * S, 2**31 - 1, 2**40 - 1])
        e = cf.Estimator(delta=rng.choice([0.05, 1e-9, 0.5]), b_us=b,
                         t_def_us=rng.choice([1, 10 * S, 2**40 - 1]), n_min=rng.randint(1, 6),
                         a_num=rng.randint(0, 2**20 - 1), a_den=rng.randint(1, 2**20 - 1),
                         ttl_max_us=rng.choice([0, 50 * S, 2**40 - 1]))
        xs = [rng.choice([0, b, rng.randint(0, b)]) for _ in range(rng.randint(0, 9))]
        g = stat(xs, b)
        f = stat(xs[: rng.randint(0, len(xs))], b)
        d = rng.randint(0, 256)
        td = rng.randint(0, 256 * 65536)
        ea = e.as_array()
        orow = lambda r: [r[0], r[1], int(np.uint64(r[2] & (2**64 - 1)).astype(np.int64)),  # noqa: E731
                          r[2] >> 64]
        assert ct.ct_calc_ttl_ref(g, f, e, d, td) == O.calc_ttl(orow(g), orow(f), ea, d, td)
        if g[0] >= 1:
            assert ct.ct_bernstein_ref(g, e) == O.bernstein(g[0], g[1], g[2], ea[0], b)


def test_host_ref_rejects_invalid_rows(ct):
    e = cf.Estimator(b_us=10 * S)
    assert ct.ct_bernstein_ref((0, 0, 0), e) == INVALID                 # n = 0
    assert ct.ct_bernstein_ref((1, 11 * S, (11 * S) ** 2), e) == INVALID  # sample above b
    assert ct.ct_bernstein_ref((2, 2, 1), e) == INVALID                 # n s2 < s1^2
    assert ct.ct_calc_ttl_ref((1, 1, 1), (1, 1, 1), e, 257, 0) == INVALID  # n_done > 256
    bad = cf.Estimator(a_den=1 << 20)                                    # alpha bound (R36 note)
    assert ct.ct_calc_ttl_ref((1, 1, 1), (1, 1, 1), bad, 1, 1) == INVALID


@pytest.mark.gpu
def test_device_spec_examples_and_random(ct):
    import torch
    ctx = ct.Context(0)
    e = cf.Estimator(b_us=10 * S)

    def rows(rs):
        return torch.tensor([[r[0], r[1], np.int64(np.uint64(r[2] & (2**64 - 1))),
                              np.int64(np.uint64(r[2] >> 64))] for r in rs], dtype=torch.int64).cuda()

    out = ct.ct_bernstein(ctx, rows([stat([2 * S]), stat([S, 2 * S, 3 * S]), (0, 0, 0)]), e)
    assert out.cpu().tolist()[0] == 124_830_336 and out.cpu().tolist()[2] == INVALID
    for name, g, f, est, d, td, want in spec_cases():
        got = ct.ct_calc_ttl_batch(ctx, rows([g]), rows([f]), torch.tensor([d]).cuda(),
                                   torch.tensor([td]).cuda(), est)
        assert int(got.cpu()[0]) == want, name
    # a batch of random queries: device == host reference == oracle
    rng = random.Random(9)
    e = cf.Estimator(delta=1e-9, b_us=2**31 - 1, t_def_us=10 * S, n_min=3, a_num=7, a_den=9,
                     ttl_max_us=0)
    G, Fr, D, TD = [], [], [], []
    for _ in range(5000):
        xs = [rng.choice([0, 2**31 - 1, rng.randint(0, 2**31 - 1)]) for _ in range(rng.randint(0, 8))]
        G.append(stat(xs))
        Fr.append(stat(xs[: rng.randint(0, len(xs))]))
        D.append(rng.randint(0, 256))
        TD.append(rng.randint(0, 10**6))
    got = ct.ct_calc_ttl_batch(ctx, rows(G), rows(Fr), torch.tensor(D).cuda(),
                               torch.tensor(TD).cuda(), e).cpu().tolist()
    bern = ct.ct_bernstein(ctx, rows(G), e).cpu().tolist()
    for i in range(len(G)):
        assert got[i] == ct.ct_calc_ttl_ref(G[i], Fr[i], e, D[i], TD[i])
        if G[i][0] >= 1:
            assert bern[i] == ct.ct_bernstein_ref(G[i], e)


@pytest.mark.gpu
def test_device_calc_ttl_clamp_shortcut_exact(ct):
    """The device CalcTTL (the replay's helper) returns ttl_max without the exact evaluation
    when a single-precision upper bound of the Bernstein bound proves the clamp.  It must equal
    the exact host reference (and the oracle) everywhere, in particular with ttl_max within a
    few µs of the unclamped value, where a too-loose or too-tight bound would show."""
    import torch
    ctx = ct.Context(0)
    rng = np.random.default_rng(11)
    L = O.lib()

    def rows(rs):
        return torch.tensor([[r[0], r[1], np.int64(np.uint64(r[2] & (2**64 - 1))),
                              np.int64(np.uint64(r[2] >> 64))] for r in rs], dtype=torch.int64).cuda()

    cases = []
    for i in range(240):
        b = int(rng.choice([60 * S, 2**31 - 1, 5 * S]))
        n = int(rng.choice([1, 2, 3, 5, 17, 100, 1000, 20000]))
        mu = float(rng.choice([1e3, 1e5, 2e6, 8e6]))
        xs = np.minimum(rng.lognormal(np.log(mu), float(rng.choice([0.0, 0.3, 1.0, 2.0])), n), 2**31 - 1)
        fs = stat(xs.astype(np.int64).tolist(), b)
        gs = stat((xs.astype(np.int64).tolist() * 2)[: n + 3], b)
        d = int(rng.integers(0, 257))
        td = int(rng.integers(d, 50 * d + 1)) if d else 0
        e0 = cf.Estimator(b_us=b, t_def_us=int(rng.choice([10 * S, 3 * S, 60 * S])), n_min=5,
                          a_num=1, a_den=10, ttl_max_us=0)
        free = ct.ct_calc_ttl_ref(gs, fs, e0, d, td)  # unclamped offset
        assert free >= 0
        for off in (-3, -1, 0, 1, 2) if free > 4 else (1, 2):
            cases.append((gs, fs, d, td, e0, max(free + off, 1)))
    for gs, fs, d, td, e0, tmax in cases:
        e = replace(e0, ttl_max_us=tmax)
        got = int(ct.ct_calc_ttl_batch(ctx, rows([gs]), rows([fs]), torch.tensor([d]).cuda(),
                                       torch.tensor([td]).cuda(), e).cpu()[0])
        want = ct.ct_calc_ttl_ref(gs, fs, e, d, td)
        assert got == want, (gs, fs, d, td, tmax)
        orow = lambda r: [r[0], r[1], int(np.uint64(r[2] & (2**64 - 1)).astype(np.int64)),  # noqa: E731
                          r[2] >> 64]
        assert want == O.calc_ttl(orow(gs), orow(fs), e.as_array(), d, td)
