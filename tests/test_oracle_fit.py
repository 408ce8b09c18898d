"""Pins for the oracle's TTL fit (extension C-4 of DESIGN.md; paper mode = C-2).

Closed forms fixed by the mathematics of n*U(k) = V*cnt_le(k) - C*sum_i min(d_i, tau_k):
  * point mass d: tau* = ceil(d/step)*step iff V > C*d, else 0;
  * uniform lattice {step..M*step}: U convex in k -> tau* = M*step iff V > C*E[D], else 0;
  * C = 0, V > 0: smallest tau covering every sample <= tau_{K-1};
  * V = 0: tau* = 0;
  * tau* non-increasing in C (Topkis: decreasing differences);
  * tools with fewer than N samples take the pooled row (PAPER.md:492-494 ladder);
  * ttl_paper row == CalcTTL of the row's statistics (pinned in test_oracle_estimator).
"""
import math
import random

import numpy as np

from ctgen import configs as cf
from oracle import oracle as O

S = 1_000_000


def csr(groups):
    dur = np.concatenate([np.asarray(g, np.int32) for g in groups]) if groups else np.zeros(0, np.int32)
    off = np.concatenate([[0], np.cumsum([len(g) for g in groups])]).astype(np.int64)
    return dur, off


def cost(c_pf=10_000, c_pin=1, bs=16, a_num=0, a_den=1, step=50_000, K=64, J=1):
    return [c_pf, c_pin, bs, a_num, a_den, step, K, J]


def est(N=1):
    return cf.Estimator(n_min=N).as_array()


def fit1(samples, V, C, step=50_000, K=64, N=1):
    """Single tool, J=1, ctx chosen so that V and C come out exactly as requested."""
    # V = c_pf*ctx*(a_den + a_num*w)/a_den with ctx=16, a_num=0 -> V = 16*c_pf; C = c_pin*ceil(16/16)
    assert V % 16 == 0
    dur, off = csr([samples])
    arg, pap, st = O.fit(dur, off, cost(c_pf=V // 16, c_pin=C, step=step, K=K), [16], [0], est(N))
    return int(arg[0, 0]), int(arg[1, 0])


def test_point_mass_closed_form():
    rng = random.Random(0)
    for _ in range(300):
        step = rng.choice([1, 7, 50_000])
        K = rng.choice([2, 8, 64])
        d = rng.randint(0, step * (K + 2))
        n = rng.randint(1, 20)
        C = rng.randint(0, 50)
        V = 16 * rng.randint(0, 200) * max(1, d // 16 + 1)
        got, _ = fit1([d] * n, V, C, step, K)
        k = -(-d // step)
        want = max(k, 1) * step if (V > C * d and max(k, 1) <= K - 1) else 0
        assert got == want, (d, step, K, V, C)


def test_cd_like_example():
    # SURVEY/DESIGN example: cd = 100 ms constant, step 50 ms -> tau* = 100 ms iff V > C*1e5
    assert fit1([100_000] * 10, V=16 * 10**6, C=100)[0] == 100_000   # 1.6e7 > 1e7
    assert fit1([100_000] * 10, V=16 * 6250, C=10)[0] == 0            # 1e5 == 10*1e4 -> tie -> 0


def test_uniform_lattice_bang_bang():
    rng = random.Random(1)
    for _ in range(200):
        step = rng.choice([3, 1000, 50_000])
        M = rng.randint(1, 30)
        m = rng.randint(1, 4)
        samples = [k * step for k in range(1, M + 1)] * m
        C = rng.randint(1, 20)
        mean2 = step * (M + 1)  # 2*E[D]
        V = 16 * rng.randint(1, (C * mean2) // 16 * 2 + 2)
        got, _ = fit1(samples, V, C, step, K=64)
        want = M * step if 2 * V > C * mean2 else 0
        assert got == want


def test_c_zero_covers_all():
    rng = random.Random(2)
    for _ in range(100):
        step, K = 1000, 40
        xs = [rng.randint(1, 45_000) for _ in range(rng.randint(1, 30))]
        got, _ = fit1(xs, V=16 * 5, C=0, step=step, K=K)
        inside = [x for x in xs if x <= (K - 1) * step]
        want = max(1, -(-max(inside) // step)) * step if inside else step
        assert got == want


def test_v_zero_never_pins():
    xs = [random.Random(3).randint(1, 10**7) for _ in range(50)]
    assert fit1(xs, V=0, C=5)[0] == 0
    assert fit1(xs, V=0, C=0)[0] == 0


def test_monotone_in_cost():
    rng = np.random.default_rng(4)
    xs = list(np.clip(rng.lognormal(np.log(2e6), 1.0, 200), 1, 6e7).astype(int))
    prev = None
    for C in [0, 1, 2, 5, 10, 20, 50, 100, 1000]:
        got, _ = fit1(xs, V=16 * 10**8, C=C, step=250_000, K=256)
        if prev is not None:
            assert got <= prev
        prev = got


def test_fallback_and_turn_buckets():
    rng = random.Random(5)
    a = [rng.randint(1, 300_000) for _ in range(40)]
    b = [rng.randint(5 * S, 9 * S) for _ in range(3)]  # fewer than N=5 samples
    dur, off = csr([a, b])
    J = 4
    ctx = [500, 2000, 8000, 32000]
    w = [1, 2, 3, 4]
    arg, pap, st = O.fit(dur, off, [13_400_000, 20, 16, 1, 10, 50_000, 256, J], ctx, w,
                         est(N=5), avg=(40, 4))
    assert list(arg[1]) == list(arg[2])          # tool 1 falls back to the pooled row
    assert st[0, 0] == 40 and st[1, 0] == 3 and st[2, 0] == 43
    assert st[2, 1] == sum(a) + sum(b)
    # turn weight (1 + alpha*w) and ctx both raise V/C -> tau* non-decreasing in j here
    assert all(arg[0, j] <= arg[0, j + 1] for j in range(J - 1))
    # paper mode: each row is CalcTTL of (global, row) statistics with the caller's AvgTurns
    e = est(N=5)
    for r in range(3):
        assert pap[r] == O.calc_ttl(st[2], st[r], e, 4, 40)


def test_paper_stats_clamp_at_b():
    b = cf.Estimator().b_us
    dur, off = csr([[10, b + 5, 3 * b]])
    _, _, st = O.fit(dur, off, cost(), [16], [0], est())
    assert st[0, 1] == 10 + b + b
    assert int(np.uint64(st[0, 2])) + (int(np.uint64(st[0, 3])) << 64) == 100 + 2 * b * b


def test_point_mass_rational_turn_factor_and_block_ceiling():
    """V_j = floor(c_pf ctx_j (a_den + a_num w_j) / a_den) and C_j = c_pin ceil(ctx_j / bs)
    (C-4) with a_den > 1, a_num > 0 and ctx_j % bs != 0, on point masses placed at
    d = floor(V/C) + {-1, 0, +1}: tau* = ceil(d/step) step iff V > C d.  The expected V and C
    use Fraction arithmetic (exact rationals, then floor / ceiling), so the pin fails if the
    oracle drops /a_den, floors ceil(ctx/bs), or rounds V up."""
    from fractions import Fraction
    rng = random.Random(6)
    flips = {"a_den": 0, "ceil": 0, "round": 0}
    for i in range(600):
        exact = i % 3 == 0  # a third of the cases sit exactly on V = C d with V's floor active
        while True:
            bs = rng.randint(2, 32)
            ctx = rng.randint(1, 6) * bs + rng.randint(1, bs - 1)        # ctx % bs != 0
            a_den, a_num, w = rng.randint(2, 9), rng.randint(1, 5), rng.randint(1, 8)
            c_pf, c_pin = rng.randint(1, 3000), rng.randint(1, 40)
            Vq = Fraction(c_pf * ctx * (a_den + a_num * w), a_den)
            V = math.floor(Vq)
            nb = math.ceil(Fraction(ctx, bs))
            C = c_pin * nb
            if not exact or (V % C == 0 and Vq.denominator != 1):
                break
        d = max(1, V // C + (0 if exact else rng.choice([-1, 0, 1])))
        step = max(1, -(-(d + 1) // 500))
        dur, off = csr([[d] * rng.randint(1, 5)])
        arg, _, _ = O.fit(dur, off, [c_pf, c_pin, bs, a_num, a_den, step, 1024, 1], [ctx], [w],
                          est(1))
        want = -(-d // step) * step if V > C * d else 0
        assert int(arg[0, 0]) == want, (bs, ctx, a_den, a_num, w, c_pf, c_pin, d)
        # the cases below would change under the named mistake
        flips["a_den"] += (c_pf * ctx * (a_den + a_num * w) > C * d) != (V > C * d)
        flips["ceil"] += (V > c_pin * (ctx // bs) * d) != (V > C * d)
        flips["round"] += (math.ceil(Vq) > C * d) != (V > C * d)
    assert min(flips.values()) >= 5, flips
