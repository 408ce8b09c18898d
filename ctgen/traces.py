"""Seeded synthetic agent-workload traces (input generation only).

This module is shared by the CUDA path and the CPU oracle as the ONLY common
code.  It holds none of the method's arithmetic (no statistics, no TTL, no
scheduling): it draws integer trace records from a counter-based generator and
lays them out in the binary format both sides read.

Shapes follow the paper's qualitative workload facts:
  * SWE-Bench programs: up to 40+/50 turns (Fig. workload_char),
    short bash tools plus long-tailed python/pytest (Fig. 3).
  * BFCL programs: few turns, tokens scaled by 0.4.
  * Poisson program arrivals, stored as unit-rate cumulative
    Exp(1) gaps in Q20 so that the rate axis is an integer gap.

Binary layout (little-endian, both sides):
  programs: structured array PROG_DTYPE, one 16-B record per program,
            seeds back to back (program index = arrival order inside a seed).
  turns:    int32[T, 4] = (new_tokens, decode_tokens, tool, dur_us); tool = -1 and
            dur_us = 0 on a program's final turn.
Random numbers come from SplitMix64 keyed by (stream, seed, program, turn, field).
"""
from __future__ import annotations

import hashlib
from dataclasses import dataclass

import numpy as np

PROG_DTYPE = np.dtype([("arr_q", "<i8"), ("turn0", "<i4"), ("nturns", "<i4")])
Q20 = 1 << 20

# ---- tool catalog --------------------------------------------------------------
# (name, class, weight within class, median_us, sigma, max_us); sigma 0 = constant.
TOOLS = [
    ("cat", "swe", 0.25, 60_000, 0.30, 2_000_000),
    ("sed", "swe", 0.15, 80_000, 0.30, 2_000_000),
    ("grep", "swe", 0.10, 150_000, 0.50, 5_000_000),
    ("ls", "swe", 0.08, 50_000, 0.30, 2_000_000),
    ("find", "swe", 0.05, 400_000, 0.60, 10_000_000),
    ("cd", "swe", 0.05, 100_000, 0.0, 100_000),
    ("git", "swe", 0.05, 200_000, 0.50, 5_000_000),
    ("echo", "swe", 0.04, 50_000, 0.20, 1_000_000),
    ("python", "swe", 0.13, 2_000_000, 1.00, 60_000_000),
    ("pytest", "swe", 0.10, 8_000_000, 0.80, 120_000_000),
    ("web_search", "bfcl", 0.60, 1_500_000, 0.50, 20_000_000),
    ("fetch_url", "bfcl", 0.40, 3_000_000, 0.60, 20_000_000),
]
N_TOOLS = len(TOOLS)
SWE, BFCL = 0, 1

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _splitmix(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = (x + np.uint64(0x9E3779B97F4A7C15)) & _M64
        z = ((z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)) & _M64
        z = ((z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)) & _M64
        return z ^ (z >> np.uint64(31))


def _key(*parts) -> np.ndarray:
    """Counter-based key: fold each part through SplitMix64."""
    h = np.uint64(0x243F6A8885A308D3)
    for part in parts:
        p = np.asarray(part).astype(np.uint64)
        with np.errstate(over="ignore"):
            h = _splitmix(h ^ p)
    return h


def _u01(h: np.ndarray) -> np.ndarray:
    """uint64 -> float64 uniform in (0, 1)."""
    return ((h >> np.uint64(11)).astype(np.float64) + 0.5) * (1.0 / (1 << 53))


def _normal(h1: np.ndarray, h2: np.ndarray) -> np.ndarray:
    return np.sqrt(-2.0 * np.log(_u01(h1))) * np.cos(2.0 * np.pi * _u01(h2))


@dataclass
class TraceSet:
    programs: np.ndarray  # PROG_DTYPE [S*P]
    turns: np.ndarray     # int32 [T, 4]
    n_seeds: int
    n_programs: int       # P, programs per seed
    n_tools: int
    pclass: np.ndarray    # uint8 [S*P], 0 = SWE, 1 = BFCL

    @property
    def n_turns(self) -> int:
        return int(self.turns.shape[0])

    def digest(self) -> str:
        h = hashlib.sha256()
        h.update(self.programs.tobytes())
        h.update(self.turns.tobytes())
        return h.hexdigest()[:16]


def generate(n_seeds: int, n_programs: int, n_bfcl: int | None = None, *,
             stream: int = 0, seed0: int = 0, ctx_cap: int = 131072,
             max_turns: int = 50, mix: str = "swe") -> TraceSet:
    """Generate S independent traces of P programs each.

    mix: "swe" (all SWE-shaped), "bfcl" (all BFCL-shaped) or "mix" (n_bfcl BFCL
    programs placed at random positions, rest SWE).  ctx_cap bounds every
    program's final context (tokens) so it fits the smallest KV budget of a
    sweep (reading R24): the program is truncated before the first
    turn that would exceed it.
    """
    S, P = int(n_seeds), int(n_programs)
    seeds = np.arange(seed0, seed0 + S, dtype=np.uint64)
    sidx = np.repeat(seeds, P)
    pidx = np.tile(np.arange(P, dtype=np.uint64), S)

    # ---- program class -------------------------------------------------------
    if mix == "swe":
        pclass = np.zeros(S * P, dtype=np.uint8)
    elif mix == "bfcl":
        pclass = np.ones(S * P, dtype=np.uint8)
    elif mix == "mix":
        nb = P // 2 if n_bfcl is None else int(n_bfcl)
        r = _key(stream, sidx, pidx, 0xC1A55).reshape(S, P)
        order = np.argsort(r, axis=1, kind="stable")
        pcl = np.zeros((S, P), dtype=np.uint8)
        rows = np.arange(S)[:, None]
        pcl[rows, order[:, :nb]] = 1
        pclass = pcl.reshape(-1)
    else:
        raise ValueError(mix)
    is_b = pclass == 1

    # ---- turn counts -----------------------------------------------------------
    z = _normal(_key(stream, sidx, pidx, 1), _key(stream, sidx, pidx, 2))
    t_swe = np.clip(np.rint(20.0 * np.exp(0.6 * z)), 2, max_turns)
    t_bfcl = 2 + (_key(stream, sidx, pidx, 3) % np.uint64(9)).astype(np.float64)
    nt = np.where(is_b, t_bfcl, t_swe).astype(np.int64)
    TM = int(min(max_turns, nt.max()))

    tix = np.arange(TM, dtype=np.uint64)[None, :]
    S2 = sidx[:, None]
    P2 = pidx[:, None]

    def nrm(field):
        return _normal(_key(stream, S2, P2, tix, field), _key(stream, S2, P2, tix, field + 1))

    # ---- tokens -----------------------------------------------------------------
    u_p = _u01(_key(stream, S2, P2, tix, 10))
    prompt_swe = np.floor(1500 + u_p * 2501)
    prompt_bfcl = np.floor((1000 + u_p * 2001) * 0.4)
    obs_swe = np.clip(np.rint(400.0 * np.exp(0.8 * nrm(11))), 20, 8000)
    obs_bfcl = np.clip(np.rint(1500.0 * np.exp(0.6 * nrm(13)) * 0.4), 8, 8000)
    dec_swe = np.clip(np.rint(200.0 * np.exp(0.7 * nrm(15))), 16, 2048)
    dec_bfcl = np.clip(np.rint(120.0 * np.exp(0.5 * nrm(17))), 8, 1024)
    b2 = is_b[:, None]
    first = (tix == 0)
    new = np.where(first, np.where(b2, prompt_bfcl, prompt_swe),
                   np.where(b2, obs_bfcl, obs_swe)).astype(np.int64)
    dec = np.where(b2, dec_bfcl, dec_swe).astype(np.int64)

    # ---- tools & durations --------------------------------------------------------
    u_t = _u01(_key(stream, S2, P2, tix, 20))
    swe_ids = [i for i, t in enumerate(TOOLS) if t[1] == "swe"]
    bf_ids = [i for i, t in enumerate(TOOLS) if t[1] == "bfcl"]

    def pick(ids):
        w = np.array([TOOLS[i][2] for i in ids])
        cdf = np.cumsum(w) / w.sum()
        j = np.searchsorted(cdf, u_t, side="right")
        return np.asarray(ids)[np.minimum(j, len(ids) - 1)]

    tool = np.where(b2, pick(bf_ids), pick(swe_ids)).astype(np.int64)
    zd = nrm(21)
    med = np.array([t[3] for t in TOOLS], dtype=np.float64)[tool]
    sig = np.array([t[4] for t in TOOLS], dtype=np.float64)[tool]
    mx = np.array([t[5] for t in TOOLS], dtype=np.float64)[tool]
    dur = np.clip(np.rint(med * np.exp(sig * zd)), 1, mx).astype(np.int64)

    # ---- context cap truncation (reading R24) ---------------------------------------
    valid = tix < nt[:, None].astype(np.uint64)
    step = new + dec
    cum_after = np.cumsum(np.where(valid, step, 0), axis=1)
    fits = cum_after <= ctx_cap
    ok = valid & fits
    # number of leading turns that are valid and fit
    nt2 = np.argmin(np.concatenate([ok, np.zeros((S * P, 1), bool)], axis=1), axis=1)
    if np.any(nt2 < 1):
        raise ValueError("ctx_cap too small for a first turn")
    nt2 = nt2.astype(np.int64)

    last = (tix.astype(np.int64) == (nt2[:, None] - 1))
    tool = np.where(last, -1, tool)
    dur = np.where(last, 0, dur)

    keep = tix.astype(np.int64) < nt2[:, None]
    turns = np.stack([new[keep], dec[keep], tool[keep], dur[keep]], axis=1).astype(np.int32)

    # ---- arrivals: cumulative Exp(1) in Q20, per seed ------------------------------------
    g = -np.log(_u01(_key(stream, sidx, pidx, 30)))
    gq = np.rint(np.minimum(g, 8.0) * Q20).astype(np.int64)
    arr = np.cumsum(gq.reshape(S, P), axis=1).reshape(-1)

    progs = np.zeros(S * P, dtype=PROG_DTYPE)
    progs["arr_q"] = arr
    t0 = np.concatenate([[0], np.cumsum(nt2)[:-1]])
    if t0[-1] + nt2[-1] >= 2**31:
        raise ValueError("too many turns for int32 offsets")
    progs["turn0"] = t0.astype(np.int32)
    progs["nturns"] = nt2.astype(np.int32)
    return TraceSet(progs, np.ascontiguousarray(turns), S, P, N_TOOLS, pclass)


def tiny(programs: list[tuple[int, list[tuple[int, int, int, int]]]], n_tools: int = 1) -> TraceSet:
    """Hand-written trace (one seed): [(arr_q, [(new, dec, tool, dur_us), ...]), ...].

    arr_q is in Q20 units: arrival_us = floor(arr_q * gap_us / 2^20); with gap_us = 2^20
    arr_q is the arrival in microseconds.
    """
    progs = np.zeros(len(programs), dtype=PROG_DTYPE)
    rows = []
    for i, (aq, ts) in enumerate(programs):
        progs[i] = (aq, len(rows), len(ts))
        rows.extend(ts)
    turns = np.array(rows, dtype=np.int32).reshape(-1, 4)
    return TraceSet(progs, turns, 1, len(programs), n_tools, np.zeros(len(programs), np.uint8))


def tool_samples(tr: TraceSet) -> tuple[np.ndarray, np.ndarray]:
    """All (tool, dur_us) records of a trace set grouped by tool (CSR layout).

    Returns (dur int32[n], tool_off int64[F+1]); segment f is dur[off[f]:off[f+1]].
    """
    t = tr.turns
    m = t[:, 2] >= 0
    tool = t[m, 2].astype(np.int64)
    d = t[m, 3]
    order = np.argsort(tool, kind="stable")
    off = np.zeros(tr.n_tools + 1, dtype=np.int64)
    np.add.at(off, tool + 1, 1)
    return np.ascontiguousarray(d[order].astype(np.int32)), np.cumsum(off)


def synthetic_samples(n: int, n_tools: int, seed: int = 0) -> tuple[np.ndarray, np.ndarray]:
    """n duration samples over n_tools tools (CSR by tool) for the bandwidth run.

    Tool f reuses catalog entry f % 12 (median/sigma/cap); segment sizes follow the
    catalog weights.  Generated chunk-wise in float32 to bound host memory.
    """
    w = np.array([TOOLS[f % N_TOOLS][2] for f in range(n_tools)], dtype=np.float64)
    cnt = np.floor(w / w.sum() * n).astype(np.int64)
    cnt[0] += n - cnt.sum()
    off = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64)
    out = np.empty(n, dtype=np.int32)
    CH = 1 << 24
    for f in range(n_tools):
        med, sig, mx = TOOLS[f % N_TOOLS][3:6]
        for a in range(int(off[f]), int(off[f + 1]), CH):
            b = min(a + CH, int(off[f + 1]))
            idx = np.arange(a, b, dtype=np.uint64)
            z = _normal(_key(7, seed, f, idx, 1), _key(7, seed, f, idx, 2)).astype(np.float32)
            out[a:b] = np.clip(np.rint(np.float32(med) * np.exp(np.float32(sig) * z)), 1, mx).astype(np.int32)
    return out, off


def synthetic_samples_torch(log2n: int, n_tools: int = 32, seed: int = 1234, device="cuda"):
    """2^log2n duration samples (CSR by tool) generated on a torch device (bandwidth run).

    Tool f has weight and median of catalog entry f % 12, lognormal sigma 0.8, clamped to
    [1 µs, 120 s].  Returns (dur int32 tensor on `device`, tool_off int64 numpy [F+1]).
    """
    import torch
    n = 1 << log2n
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    w = torch.tensor([TOOLS[f % N_TOOLS][2] for f in range(n_tools)], dtype=torch.float64)
    cnt = (w / w.sum() * n).floor().long()
    cnt[0] += n - int(cnt.sum())
    off = np.concatenate([[0], np.cumsum(cnt.numpy())]).astype(np.int64)
    dur = torch.empty(n, dtype=torch.int32, device=device)
    for f in range(n_tools):
        a, b = int(off[f]), int(off[f + 1])
        z = torch.randn(b - a, generator=g, device=device)
        med = float(TOOLS[f % N_TOOLS][3])
        dur[a:b] = torch.clamp(med * torch.exp(0.8 * z), 1, 1.2e8).to(torch.int32)
    return dur, off


def turn_scaling(tr: TraceSet, k: int) -> TraceSet:
    """Turn-scaling transform of the robustness study.

    Every program's turn list is repeated k times and every token count is divided by k
    (integer division, minimum 1), so total token volume is kept within rounding.  Tool calls
    and durations repeat with their turns; the last turn of each non-final copy calls the
    program's first tool with its first duration (the original final turn has no tool).
    """
    if k < 1:
        raise ValueError("k >= 1")
    if k == 1:
        return tr
    progs = np.zeros_like(tr.programs)
    rows = []
    for i in range(len(tr.programs)):
        t0, nt = int(tr.programs["turn0"][i]), int(tr.programs["nturns"][i])
        base = tr.turns[t0:t0 + nt]
        first_tool = (int(base[0, 2]), int(base[0, 3])) if nt > 1 else (0, 100_000)
        progs[i] = (tr.programs["arr_q"][i], len(rows), nt * k)
        for c in range(k):
            for j in range(nt):
                new = max(int(base[j, 0]) // k, 1 if j == 0 else 0)
                dec = max(int(base[j, 1]) // k, 1)
                tool, dur = int(base[j, 2]), int(base[j, 3])
                if j == nt - 1 and c < k - 1:
                    tool, dur = first_tool
                rows.append((new, dec, tool, dur))
    turns = np.array(rows, dtype=np.int32).reshape(-1, 4)
    return TraceSet(progs, turns, tr.n_seeds, tr.n_programs, tr.n_tools, tr.pclass)


def to_jsonl(tr: TraceSet, path: str, seed: int = 0, messages: bool = False) -> None:
    """Write seed `seed` of a trace set as a JSONL trace (one program per line, SPEC.md:144-152
    field names) for the host ingest (NEXT-4).  Times are written as exact decimal seconds of
    the integer µs (arrival = arr_q µs, i.e. the trace's arrivals at gap_us = 2^20).  With
    `messages`, non-final turns carry a synthetic raw model output instead of tool_name, in
    the App. A formats, rotating over the turns."""
    import json

    def sec(us: int) -> str:
        return "%d.%06d" % divmod(int(us), 1_000_000)

    P = tr.n_programs
    with open(path, "w") as fh:
        for i in range(seed * P, (seed + 1) * P):
            t0, nt = int(tr.programs["turn0"][i]), int(tr.programs["nturns"][i])
            turns = []
            for j in range(nt):
                new, dec, tool, dur = (int(x) for x in tr.turns[t0 + j])
                t = {"new_prompt_tokens": new, "decode_tokens": dec}
                if j < nt - 1:
                    name = TOOLS[tool][0]
                    if messages:
                        t["message"] = _message(name, i + j)
                    else:
                        t["tool_name"] = name
                    t["tool_duration_s"] = "@" + sec(dur) + "@"
                turns.append(t)
            rec = {"program_id": "p%d" % i, "arrival_time_s": "@" + sec(tr.programs["arr_q"][i]) + "@",
                   "turns": turns}
            # numbers as exact decimal text (json.dumps would print a float)
            fh.write(json.dumps(rec).replace('"@', "").replace('@"', "") + "\n")


def _message(name: str, k: int) -> str:
    forms = [
        "```bash\n%s -la . && echo done\n```" % name,
        '{"id": "fc_%d", "call_id": "call_%d", "type": "function_call", "name": "%s", '
        '"arguments": {"q": "x"}}' % (k, k, name),
        '{"name": "%s", "arguments": {"q": "x"}}' % name,
        "%s(query=\"x\", n=3)" % name,
    ]
    return forms[k % len(forms)]
