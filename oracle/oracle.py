"""ctypes wrapper around oracle/libct_oracle.so (TEST INFRASTRUCTURE ONLY).

Builds the library on first use with g++ if it is missing (it is plain C++17,
single-threaded per replica, no dependency on the product tree).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libct_oracle.so")
SRC = os.path.join(HERE, "ct_oracle.cpp")

SUMMARY_FIELDS = ["status_ndone", "turns_done", "sum_jct", "max_jct", "p50_jct", "p99_jct",
                  "sum_bubble", "makespan", "iterations", "busy_us", "prefill_tokens",
                  "recompute_tokens", "pin_hits", "pin_expiries", "victims", "reloads"]


def build(force: bool = False) -> str:
    alt = os.environ.get("CT_ORACLE_LIB")  # tools/oracle_mutations.py: a mutated oracle build
    if alt:
        return alt
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        # build beside it and rename: a process that has the old library mapped keeps it
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-o", LIB + ".tmp",
                               SRC, "-lpthread"])
        os.replace(LIB + ".tmp", LIB)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        i64, u64, p = C.c_int64, C.c_uint64, C.c_void_p
        _lib.or_isqrt.restype = u64
        _lib.or_isqrt.argtypes = [u64, u64]
        _lib.or_bernstein.restype = i64
        _lib.or_bernstein.argtypes = [i64, i64, u64, u64, u64, i64]
        for f in ("or_select_bound",):
            getattr(_lib, f).restype = i64
            getattr(_lib, f).argtypes = [p, p, p]
        _lib.or_calc_ttl.restype = i64
        _lib.or_calc_ttl.argtypes = [p, p, p, i64, i64]
        _lib.or_simplified.restype = i64
        _lib.or_simplified.argtypes = [p, p, p, i64, i64]
        _lib.or_infercept_predict.restype = i64
        _lib.or_infercept_predict.argtypes = [p, p, p]
        _lib.or_infercept_swap_us.restype = i64
        _lib.or_infercept_swap_us.argtypes = [i64, i64, i64]
        _lib.or_fit.restype = C.c_int
        _lib.or_fit.argtypes = [p, p, C.c_int, p, p, p, p, p, p, p, p]
        _lib.or_simulate.restype = C.c_int
        _lib.or_simulate.argtypes = [p, p, i64, C.c_int, C.c_int, C.c_int, p, C.c_int, p, C.c_int,
                                     p, C.c_int, p, p, p, C.c_int, i64, i64, C.c_int, p, p, p]
        _lib.or_simulate_audit.restype = C.c_int
        _lib.or_simulate_audit.argtypes = [p, p, i64, C.c_int, C.c_int, C.c_int, p, C.c_int, p,
                                           C.c_int, p, C.c_int, p, p, p, C.c_int, i64, p, i64, p, p]
        _lib.or_jct_stats.restype = C.c_int
        _lib.or_jct_stats.argtypes = [p, i64, C.c_int, p]
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int64))


# ---- statistics rows: [n, s1, s2_lo, s2_hi] --------------------------------------
def stats_row(samples_us, b_us: int | None = None) -> np.ndarray:
    n, s1, s2 = 0, 0, 0
    for t in samples_us:
        t = int(t)
        if b_us is not None:
            t = min(t, b_us)
        n += 1
        s1 += t
        s2 += t * t
    return _i64([n, s1, np.int64(np.uint64(s2 & (2**64 - 1))), np.int64(np.uint64(s2 >> 64))])


def isqrt(x: int) -> int:
    """floor(sqrt(x)) for 0 <= x < 2^128."""
    return int(lib().or_isqrt(x & (2**64 - 1), x >> 64))


def bernstein(n: int, s1: int, s2: int, lq: int, b_us: int) -> int:
    return int(lib().or_bernstein(n, s1, s2 & (2**64 - 1), s2 >> 64, lq, b_us))


def select_bound(g, f, est) -> int:
    g, f, est = _i64(g), _i64(f), _i64(est)
    return int(lib().or_select_bound(_ptr(g), _ptr(f), _ptr(est)))


def calc_ttl(g, f, est, n_done: int, turns_done: int) -> int:
    g, f, est = _i64(g), _i64(f), _i64(est)
    return int(lib().or_calc_ttl(_ptr(g), _ptr(f), _ptr(est), n_done, turns_done))


def simplified(g, f, est, t_pin: int, t_thresh: int) -> int:
    g, f, est = _i64(g), _i64(f), _i64(est)
    return int(lib().or_simplified(_ptr(g), _ptr(f), _ptr(est), t_pin, t_thresh))


def infercept_predict(g, f, est) -> int:
    g, f, est = _i64(g), _i64(f), _i64(est)
    return int(lib().or_infercept_predict(_ptr(g), _ptr(f), _ptr(est)))


def infercept_swap_us(ctx: int, bs: int, c_h2d_ps: int) -> int:
    return int(lib().or_infercept_swap_us(ctx, bs, c_h2d_ps))


def fit(dur: np.ndarray, tool_off: np.ndarray, cost, ctx_j, w_j, est, avg=(0, 0)):
    """Returns (ttl_argmax[(F+1), J], ttl_paper[F+1], stats[(F+1), 4])."""
    dur = np.ascontiguousarray(dur, dtype=np.int32)
    off = _i64(tool_off)
    F = off.shape[0] - 1
    cost = _i64(cost)
    J = int(cost[7])
    ctx_j, w_j, est, avg = _i64(ctx_j), _i64(w_j), _i64(est), _i64(avg)
    arg = np.zeros((F + 1, J), np.int64)
    pap = np.zeros(F + 1, np.int64)
    st = np.zeros((F + 1, 4), np.int64)
    rc = lib().or_fit(_ptr(dur), _ptr(off), F, _ptr(cost), _ptr(ctx_j), _ptr(w_j), _ptr(est),
                      _ptr(avg), _ptr(arg), _ptr(pap), _ptr(st))
    if rc != 0:
        raise ValueError("or_fit rejected its input (%d)" % rc)
    return arg, pap, st


def simulate(trace, sweep, engine, r_begin: int = 0, r_end: int | None = None,
             n_threads: int = 1, want_jct: bool = True, want_bubble: bool = False):
    """Replay replicas [r_begin, r_end) of `sweep` over `trace` (ctgen types).

    Returns (summary int64[R,16], jct int64[R,P] or None), plus bubble int64[R,P] (each
    program's total waiting time) as a third element when want_bubble.
    """
    if r_end is None:
        r_end = sweep.n_replicas
    R = r_end - r_begin
    progs = np.ascontiguousarray(trace.programs)
    turns = np.ascontiguousarray(trace.turns, dtype=np.int32)
    gap = _i64(sweep.gap_us)
    kv = _i64(sweep.kv_blocks)
    pol = _i64(sweep.policy_array())
    est = _i64(sweep.estimator.as_array())
    eng = _i64(engine.as_array() if hasattr(engine, "as_array") else engine)
    if sweep.fitted is not None:
        fitted = _i64(sweep.fitted)
        J = int(fitted.shape[1])
    else:
        fitted = np.zeros((trace.n_tools, 1), np.int64)
        J = 1
    summ = np.zeros((R, 16), np.int64)
    jct = np.zeros((R, trace.n_programs), np.int64) if want_jct else None
    bub = np.zeros((R, trace.n_programs), np.int64) if want_bubble else None
    rc = lib().or_simulate(_ptr(progs), _ptr(turns), turns.shape[0], trace.n_seeds,
                           trace.n_programs, trace.n_tools, _ptr(gap), len(gap), _ptr(kv), len(kv),
                           _ptr(pol), len(sweep.policies), _ptr(est), _ptr(eng), _ptr(fitted), J,
                           r_begin, r_end, n_threads, _ptr(summ),
                           _ptr(jct) if jct is not None else None,
                           _ptr(bub) if bub is not None else None)
    if rc != 0:
        raise ValueError("or_simulate rejected its input (%d)" % rc)
    return (summ, jct, bub) if want_bubble else (summ, jct)


def audit(trace, sweep, engine, replica: int):
    """Per-decision audit log of one replica: (summary int64[16], [records])."""
    import json
    progs = np.ascontiguousarray(trace.programs)
    turns = np.ascontiguousarray(trace.turns, dtype=np.int32)
    gap, kv = _i64(sweep.gap_us), _i64(sweep.kv_blocks)
    pol, est = _i64(sweep.policy_array()), _i64(sweep.estimator.as_array())
    eng = _i64(engine.as_array() if hasattr(engine, "as_array") else engine)
    if sweep.fitted is not None:
        fitted = _i64(sweep.fitted)
        J = int(fitted.shape[1])
    else:
        fitted, J = np.zeros((trace.n_tools, 1), np.int64), 1
    summ = np.zeros(16, np.int64)
    n = C.c_int64(0)
    cap = 1 << 16
    while True:
        buf = C.create_string_buffer(cap)
        rc = lib().or_simulate_audit(_ptr(progs), _ptr(turns), turns.shape[0], trace.n_seeds,
                                     trace.n_programs, trace.n_tools, _ptr(gap), len(gap), _ptr(kv),
                                     len(kv), _ptr(pol), len(sweep.policies), _ptr(est), _ptr(eng),
                                     _ptr(fitted), J, int(replica), buf, cap, C.byref(n), _ptr(summ))
        if rc < 0:
            raise ValueError("or_simulate_audit rejected its input (%d)" % rc)
        if rc == 0:
            break
        cap = int(n.value) + 1
    text = buf.raw[: n.value].decode()
    return summ, [json.loads(l) for l in text.splitlines() if l]


def jct_stats(summary: np.ndarray, n_cells: int) -> np.ndarray:
    s = np.ascontiguousarray(summary, dtype=np.int64)
    out = np.zeros((n_cells, 8), np.int64)
    rc = lib().or_jct_stats(_ptr(s), s.shape[0], n_cells, _ptr(out))
    if rc != 0:
        raise ValueError("or_jct_stats rejected its input")
    return out


def status(summary_row) -> int:
    return int(np.int64(summary_row[0]) & 0xFFFFFFFF)


def n_done(summary_row) -> int:
    return int(np.int64(summary_row[0]) >> 32)
