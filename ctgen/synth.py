"""Integer-only trace synthesis (NEXT-4): the same workload shapes as `traces.generate`, drawn
with arithmetic that a GPU reproduces bit for bit, so traces can be synthesised in HBM
(`ct_synthesize_traces`) instead of being generated on the host and copied.

This is input generation, shared by both sides like `traces`: the CPU oracle replays the traces
this module builds, the library's synthesis kernel must write the same bytes.  It holds none of
the method's arithmetic.

Definition (every step is integer; `key` is the SplitMix64 fold of `traces._key`):
  u(h)            = h >> 32                                    (32-bit uniform)
  uniform(h, n)   = (u(h) * n) >> 32                           (0 <= . < n)
  quantile(T, h)  = T[i] + (((T[i+1] - T[i]) * f) >> 16),  i = u >> 22, f = (u >> 6) & 0xFFFF
                    for a monotone int64 table T[0..1024] of the distribution's quantiles at
                    p = i / 1024 (the tables are inputs; floats are used only to build them).
  class (mix)     : program p of seed s is BFCL iff the rank of key(stream,s,p,0xC1A55) among
                    the seed's keys (ties: index) is < n_bfcl.
  turns           : SWE quantile(TURNS, key(s,p,1)); BFCL 2 + uniform(key(s,p,3), 9).
  turn 0 prompt   : SWE 1500 + uniform(key(s,p,0,10), 2501); BFCL (2 (1000 + uniform(.., 2001))) / 5.
  turn t>0 new    : quantile(OBS_class, key(s,p,t,11)).
  decode          : quantile(DEC_class, key(s,p,t,15)).
  tool            : first j of the class's tools with u(key(s,p,t,20)) < CDF_j (u32 thresholds);
                    duration quantile(DUR_tool, key(s,p,t,21)); the final turn has tool -1, dur 0.
  ctx cap (R24)   : a program keeps its leading turns whose cumulative new + decode <= ctx_cap.
  arrivals        : arr_q = prefix sum over the seed of quantile(EXP, key(s,p,30)).
Layout: programs back to back per seed; a seed's turns are contiguous, seeds in order.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
from scipy.special import ndtri

from .traces import BFCL, N_TOOLS, PROG_DTYPE, Q20, SWE, TOOLS, TraceSet, _key

TABLE = 1025  # quantile points i / 1024, i = 0..1024
MIX_KEY = 0xC1A55


def _p():
    p = np.arange(TABLE, dtype=np.float64) / 1024.0
    return np.clip(p, 2.0 ** -20, 1.0 - 2.0 ** -20)


def lognormal_table(median: float, sigma: float, lo: int, hi: int, scale: float = 1.0) -> np.ndarray:
    """Quantiles of clip(round(scale * median * exp(sigma z)), lo, hi)."""
    q = np.rint(scale * median * np.exp(sigma * ndtri(_p())))
    return np.clip(q, lo, hi).astype(np.int64)


def exp_table() -> np.ndarray:
    """Quantiles of round(min(-ln(1 - p), 8) * 2^20) (unit-rate Poisson gaps in Q20)."""
    g = np.minimum(-np.log1p(-_p()), 8.0)
    return np.rint(g * Q20).astype(np.int64)


@dataclass
class SynthParams:
    """All inputs of the synthesis (tables are int64[1025] quantile tables)."""
    stream: int
    ctx_cap: int
    max_turns: int
    n_bfcl: int              # BFCL programs per seed ("mix"); 0 = all SWE, P = all BFCL
    turns_swe: np.ndarray
    obs: np.ndarray          # [2, 1025] (SWE, BFCL)
    dec: np.ndarray          # [2, 1025]
    dur: np.ndarray          # [N_TOOLS, 1025]
    exp: np.ndarray          # [1025]
    tool_cdf: np.ndarray     # uint32 [N_TOOLS]: cumulative threshold within the tool's class
    tool_class: np.ndarray   # int32 [N_TOOLS]


def params(stream: int = 0, ctx_cap: int = 131072, max_turns: int = 50, n_bfcl: int = 0) -> SynthParams:
    if ctx_cap < 8192:
        raise ValueError("ctx_cap >= 8192 keeps every first turn (prompt <= 4000, decode <= 2048)")
    if not 2 <= max_turns <= 1024:
        raise ValueError("max_turns in [2, 1024]")
    obs = np.stack([lognormal_table(400, 0.8, 20, 8000), lognormal_table(1500, 0.6, 8, 8000, 0.4)])
    dec = np.stack([lognormal_table(200, 0.7, 16, 2048), lognormal_table(120, 0.5, 8, 1024)])
    dur = np.stack([lognormal_table(t[3], t[4], 1, t[5]) for t in TOOLS])
    cdf = np.zeros(N_TOOLS, np.uint32)
    cls = np.array([SWE if t[1] == "swe" else BFCL for t in TOOLS], np.int32)
    for c in (SWE, BFCL):
        ids = [i for i in range(N_TOOLS) if cls[i] == c]
        w = np.array([TOOLS[i][2] for i in ids])
        cum = np.cumsum(w) / w.sum()
        th = np.minimum(np.rint(cum * 2.0 ** 32), 2.0 ** 32 - 1).astype(np.uint64)
        th[-1] = 2 ** 32 - 1  # the last tool takes the rest (u <= 2^32 - 1)
        cdf[ids] = th.astype(np.uint32)
    return SynthParams(stream, ctx_cap, max_turns, n_bfcl,
                       lognormal_table(20, 0.6, 2, max_turns), obs, dec, dur, exp_table(), cdf, cls)


def _u(h):
    return h >> np.uint64(32)


def _uniform(h, n):
    return ((_u(h) * np.uint64(n)) >> np.uint64(32)).astype(np.int64)


def _quantile_rows(T2, row, h):
    """Per-element table row (class or tool)."""
    u = _u(h)
    i = (u >> np.uint64(22)).astype(np.int64)
    f = ((u >> np.uint64(6)) & np.uint64(0xFFFF)).astype(np.int64)
    a = T2[row, i]
    b = T2[row, i + 1]
    return a + (((b - a) * f) >> 16)


def synthesize(sp: SynthParams, seed0: int, n_seeds: int, P: int) -> TraceSet:
    """The reference synthesis (numpy, vectorised); the CUDA kernel writes the same bytes."""
    S = int(n_seeds)
    st = np.uint64(sp.stream)
    seeds = np.arange(seed0, seed0 + S, dtype=np.uint64)
    sidx = np.repeat(seeds, P)
    pidx = np.tile(np.arange(P, dtype=np.uint64), S)
    # class
    k = _key(st, sidx, pidx, MIX_KEY).reshape(S, P)
    order = np.argsort(k, axis=1, kind="stable")
    rank = np.empty_like(order)
    rank[np.arange(S)[:, None], order] = np.arange(P)[None, :]
    cls = (rank.reshape(-1) < sp.n_bfcl).astype(np.int64)  # 1 = BFCL
    # turn counts
    nt = np.where(cls == 1, 2 + _uniform(_key(st, sidx, pidx, 3), 9),
                  _quantile_rows(sp.turns_swe[None, :], np.zeros(S * P, np.int64), _key(st, sidx, pidx, 1)))
    nt = np.minimum(nt, sp.max_turns)
    TM = int(nt.max())
    tix = np.arange(TM, dtype=np.uint64)[None, :]
    S2, P2, C2 = sidx[:, None], pidx[:, None], np.broadcast_to(cls[:, None], (S * P, TM))
    h10 = _key(st, S2, P2, tix, 10)
    prompt = np.where(C2 == 1, (2 * (1000 + _uniform(h10, 2001))) // 5, 1500 + _uniform(h10, 2501))
    obs = _quantile_rows(sp.obs, C2, _key(st, S2, P2, tix, 11))
    new = np.where(tix == 0, prompt, obs)
    dec = _quantile_rows(sp.dec, C2, _key(st, S2, P2, tix, 15))
    u20 = _u(_key(st, S2, P2, tix, 20)).astype(np.int64)
    tool = np.full((S * P, TM), -1, np.int64)
    for c in (SWE, BFCL):
        ids = [i for i in range(N_TOOLS) if sp.tool_class[i] == c]
        t_c = np.full((S * P, TM), ids[-1], np.int64)
        for j in reversed(ids):  # first j with u < CDF_j
            t_c = np.where(u20 < int(sp.tool_cdf[j]), j, t_c)
        tool = np.where(C2 == (1 if c == BFCL else 0), t_c, tool)
    dur = _quantile_rows(sp.dur, tool, _key(st, S2, P2, tix, 21))
    # ctx cap (R24): leading turns whose cumulative new + decode fits
    valid = tix.astype(np.int64) < nt[:, None]
    cum = np.cumsum(np.where(valid, new + dec, 0), axis=1)
    ok = valid & (cum <= sp.ctx_cap)
    nt2 = np.argmin(np.concatenate([ok, np.zeros((S * P, 1), bool)], axis=1), axis=1).astype(np.int64)
    assert np.all(nt2 >= 1)
    last = tix.astype(np.int64) == (nt2[:, None] - 1)
    tool = np.where(last, -1, tool)
    dur = np.where(last, 0, dur)
    keep = tix.astype(np.int64) < nt2[:, None]
    turns = np.stack([new[keep], dec[keep], tool[keep], dur[keep]], axis=1).astype(np.int32)
    # arrivals
    gq = _quantile_rows(sp.exp[None, :], np.zeros(S * P, np.int64), _key(st, sidx, pidx, 30))
    arr = np.cumsum(gq.reshape(S, P), axis=1).reshape(-1)
    progs = np.zeros(S * P, dtype=PROG_DTYPE)
    progs["arr_q"] = arr
    progs["turn0"] = np.concatenate([[0], np.cumsum(nt2)[:-1]]).astype(np.int32)
    progs["nturns"] = nt2.astype(np.int32)
    return TraceSet(progs, np.ascontiguousarray(turns), S, P, N_TOOLS, cls.astype(np.uint8))
