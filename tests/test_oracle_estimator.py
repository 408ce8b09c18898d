"""Pins for the oracle's estimator / CalcTTL / simplified decision (§4.2-4.5).

Each pin is independent of the oracle's integer arithmetic: worked examples
(tests/golden/spec_estimator_examples.txt), the paper formula evaluated in double
precision within the fixed-point error bound, library routines (math.isqrt), and
properties the paper states (B >= mean, coverage >= 1 - delta).
"""
import math
import random

import numpy as np
import pytest

from ctgen import configs as cf
from oracle import oracle as O

S = 1_000_000  # µs per second
LQ05 = cf.lq_from_delta(0.05)


def est(**kw):
    e = cf.Estimator(**kw)
    return e.as_array()


def float_bound(samples_us, delta, b_us):
    """B(delta) of PAPER.md:469-474 in double precision, sigma with (n-1) normalisation."""
    n = len(samples_us)
    mu = sum(samples_us) / n
    var = 0.0 if n == 1 else sum((t - mu) ** 2 for t in samples_us) / (n - 1)
    L = math.log(3.0 / delta)
    return mu + math.sqrt(2.0 * var * L / n) + 3.0 * b_us * L / n


def row(samples, b=None):
    return O.stats_row(samples, b)


def test_lq_encoding():
    assert LQ05 == 17_585_075_993
    assert abs(LQ05 / 2**32 - math.log(60.0)) < 2**-32


def test_isqrt_matches_library():
    rng = random.Random(1)
    vals = [0, 1, 2, 3, 4, 15, 16, 17, 2**62, 2**64 - 1, (2**32 - 1) ** 2, (2**32 - 1) ** 2 - 1]
    vals += [rng.randrange(2**64) for _ in range(3000)] + [rng.randrange(10**6) for _ in range(1000)]
    vals += [2**64, 2**64 + 1, 2**128 - 1, (2**64 - 1) ** 2, (2**64 - 1) ** 2 - 1]
    vals += [rng.randrange(2**128) for _ in range(2000)] + [rng.randrange(2**70) for _ in range(1000)]
    for v in vals:
        assert O.isqrt(v) == math.isqrt(v)


def test_bernstein_spec_example():
    # n=1, mu=2 s, b=10 s, delta=0.05 -> 2 + 30 ln 60 = 124.830336.. s
    B = O.bernstein(1, 2 * S, (2 * S) ** 2, LQ05, 10 * S)
    assert B == 124_830_336
    assert abs(B - (2 * S + 30 * S * math.log(60))) < 1.0


def test_sample_std_example():
    # {1,2,3} s -> mu = 2 s, sigma = 1 s; B then follows PAPER.md:469-474
    r = row([1 * S, 2 * S, 3 * S])
    n, s1, s2 = 3, 6 * S, 14 * S * S
    assert list(r[:2]) == [n, s1]
    B = O.bernstein(n, s1, s2, LQ05, 10 * S)
    exact = 2 * S + math.sqrt(2 * (1 * S) ** 2 * math.log(60) / 3) + 30 * S * math.log(60) / 3
    assert abs(B - exact) <= 3
    # sigma = 0 at n = 1: only the range term remains
    assert O.bernstein(1, 5 * S, 25 * S * S, LQ05, 10 * S) == 5 * S + (3 * 10 * S * LQ05) // 2**32


@pytest.mark.parametrize("seed", range(4))
def test_bernstein_vs_double_formula(seed):
    """Fixed point B within 3 µs of the double-precision paper formula (3 floors + L_q rounding)."""
    rng = random.Random(seed)
    for _ in range(500):
        n = rng.choice([1, 2, 3, 5, 10, 50, 400])
        b = rng.choice([10 * S, 60 * S, 120 * S])
        delta = rng.choice([0.05, 0.1, 0.01, 1e-6])
        kind = rng.random()
        if kind < 0.3:
            xs = [rng.randint(1, b) for _ in range(n)]
        elif kind < 0.6:
            xs = [int(rng.lognormvariate(math.log(2 * S), 1.0)) % b + 1 for _ in range(n)]
        else:
            c = rng.randint(1, b)
            xs = [c] * n
        r = row(xs)
        B = O.bernstein(n, int(r[1]), int(np.uint64(r[2])) + (int(np.uint64(r[3])) << 64),
                        cf.lq_from_delta(delta), b)
        assert abs(B - float_bound(xs, delta, b)) <= 3.0, (xs, delta, b)
        assert B >= sum(xs) // n  # B >= mean


def test_bernstein_vs_double_wide_samples():
    """The square-root argument 2 v L_q / (n 2^32) exceeds 2^64 for a few samples spread over
    [0, 2^31) with a small delta: the whole 128-bit value must enter the root.
    Relative tolerance: the double formula itself rounds at ~2^-52 of B."""
    rng = random.Random(77)
    big = 0
    for _ in range(400):
        n = rng.choice([2, 3, 4, 7])
        b = 2**31 - 1
        delta = rng.choice([1e-9, 1e-7, 1e-4])
        xs = [rng.choice([0, b, rng.randint(0, b)]) for _ in range(n)]
        r = row(xs)
        lq = cf.lq_from_delta(delta)
        s2 = int(np.uint64(r[2])) + (int(np.uint64(r[3])) << 64)
        B = O.bernstein(n, int(r[1]), s2, lq, b)
        want = float_bound(xs, delta, b)
        assert abs(B - want) <= 3.0 + want * 1e-13, (xs, delta, B, want)
        var = (n * s2 - int(r[1]) ** 2) // (n * (n - 1))
        big += (2 * var * lq) // (n << 32) >= 2**64
    assert big > 30  # the > 2^64 region is exercised


def test_bernstein_nonincreasing_in_n():
    # Fixed mu and sigma, growing n (two-point sample 1 s / 3 s, n even) -> B non-increasing
    prev = None
    for half in range(1, 400):
        xs = [1 * S] * half + [3 * S] * half
        r = row(xs)
        B = O.bernstein(2 * half, int(r[1]), int(np.uint64(r[2])) + (int(np.uint64(r[3])) << 64),
                        LQ05, 10 * S)
        # sigma_hat with (n-1) normalisation shrinks toward 1 s as n grows; both terms shrink
        if prev is not None:
            assert B <= prev
        prev = B


def test_bernstein_coverage():
    """SPEC.md:647 (AC2): uniform [0, b], b = 10 s, delta = 0.1; over 1000 streams of length 50
    the true mean (5 s) is <= B at every prefix in >= 90% of streams."""
    rng = np.random.default_rng(7)
    b = 10 * S
    lq = cf.lq_from_delta(0.1)
    ok = 0
    for _ in range(1000):
        xs = rng.integers(0, b + 1, size=50)
        good = True
        n = s1 = s2 = 0
        for x in xs:
            x = int(x)
            n += 1
            s1 += x
            s2 += x * x
            if O.bernstein(n, s1, s2, lq, b) < b // 2:
                good = False
                break
        ok += good
    assert ok >= 900


def test_select_bound_cases():
    e = est(n_min=5, t_def_us=10 * S, b_us=10 * S)
    g0 = row([])
    assert O.select_bound(g0, g0, e) == 10 * S
    g = row([S] * 20)
    f2 = row([2 * S] * 2)
    f7 = row([3 * S] * 7)
    Bg = O.bernstein(20, 20 * S, 20 * S * S, int(e[0]), 10 * S)
    Bf = O.bernstein(7, 21 * S, 63 * S * S, int(e[0]), 10 * S)
    assert O.select_bound(g, f2, e) == Bg
    assert O.select_bound(g, f7, e) == Bf
    assert Bf != Bg


def test_calc_ttl_spec_examples():
    # T_default = 10, B = 10 (|S| < N -> B = T_default), alpha = 0 -> TTL 10 s
    e = est(t_def_us=10 * S, a_num=0, a_den=1, ttl_max_us=0)
    g0 = row([])
    assert O.calc_ttl(g0, g0, e, 0, 0) == 10 * S
    # B = 5 s, alpha = 0.1, AvgTurns = 10 -> 10^2/5 * (1 + 1) = 40 s.
    # B_f = 5 s exactly: 16 identical samples of 5 s (sigma = 0) with b = 1 µs (range term 0).
    f = row([5 * S] * 16)
    e = est(t_def_us=10 * S, a_num=1, a_den=10, ttl_max_us=0, b_us=1, n_min=5)
    assert O.select_bound(f, f, e) == 5 * S
    assert O.calc_ttl(f, f, e, 1, 10) == 40 * S
    assert O.calc_ttl(f, f, e, 3, 30) == 40 * S  # AvgTurns = 30/3 = 10 as well
    # clamp to ttl_max = 30 s
    e2 = est(t_def_us=10 * S, a_num=1, a_den=10, ttl_max_us=30 * S, b_us=1, n_min=5)
    assert O.calc_ttl(f, f, e2, 1, 10) == 30 * S
    # no completed program yet: AvgTurns factor is 1 (reading R7)
    assert O.calc_ttl(f, f, e, 0, 0) == 20 * S


def test_calc_ttl_vs_double():
    rng = random.Random(3)
    for _ in range(2000):
        T = rng.choice([1, 5, 10, 30]) * S
        e = est(t_def_us=T, a_num=rng.randint(0, 5), a_den=rng.choice([1, 10, 100]), ttl_max_us=0,
                b_us=rng.choice([10, 60]) * S, n_min=rng.choice([1, 5, 20]))
        xs = [rng.randint(1, 20 * S) for _ in range(rng.randint(0, 40))]
        g = row(xs, int(e[1]))
        f = row(xs[: rng.randint(0, len(xs))], int(e[1]))
        D = rng.randint(0, 50)
        td = D * rng.randint(1, 40)
        B = O.select_bound(g, f, e)
        want = T * T / B * (1 + (e[4] / e[5]) * (td / D if D else 0.0))
        got = O.calc_ttl(g, f, e, D, td)
        assert abs(got - want) <= 1.0 + want * 1e-12
        # monotone: decreasing in B, increasing in AvgTurns
        if D:
            assert O.calc_ttl(g, f, e, D, td + D) >= got


def test_simplified_examples():
    e = est(n_min=5)
    g = row([S // 2] * 6)
    assert O.simplified(g, g, e, 5 * S, 2 * S) == 5 * S
    g3 = row([3 * S] * 6)
    assert O.simplified(g3, g3, e, 5 * S, 2 * S) == 0
    g0 = row([])
    assert O.simplified(g0, g0, e, 5 * S, 2 * S) == 0
    assert O.simplified(g0, g0, e, 5 * S, cf.ALWAYS) == 5 * S  # TTL-grid sentinel (R9)
    # per-tool mean when |S_f| >= N, else global mean
    f_few = row([10 * S] * 2)
    assert O.simplified(g, f_few, e, 7, 2 * S) == 7
    f_many = row([10 * S] * 5)
    assert O.simplified(g, f_many, e, 7, 2 * S) == 0
