"""Python binding of libcontinuum: same names as the C ABI, argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels; this module only turns
torch tensors (device memory), streams and the ctgen parameter objects into the C structs of
include/continuum.h.  There is no CPU fallback: without a CUDA device or without the built
library every call raises.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib as L

SUMMARY_FIELDS = ["status_ndone", "turns_done", "sum_jct", "max_jct", "p50_jct", "p99_jct",
                  "sum_bubble", "makespan", "iterations", "busy_us", "prefill_tokens",
                  "recompute_tokens", "pin_hits", "pin_expiries", "victims", "reloads"]


def _stream_ptr(stream) -> int | None:
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


class Context:
    """Owns a ct_ctx (scratch only) on one CUDA device."""

    def __init__(self, device: int | None = None):
        if not torch.cuda.is_available():
            raise L.CtError("libcontinuum needs a CUDA device (no CPU fallback)")
        self.device = torch.cuda.current_device() if device is None else int(device)
        self._h = C.c_void_p()
        with torch.cuda.device(self.device):
            L.check(L.lib().ct_ctx_create(self.device, C.byref(self._h)), "ct_ctx_create")

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                L.lib().ct_ctx_destroy(h)
            except Exception:
                pass
            self._h = None

    @property
    def handle(self):
        return self._h

    def set_timing(self, enable: bool = True) -> None:
        """Record CUDA events around the dominant kernel of each call (kernel-only times)."""
        L.check(L.lib().ct_ctx_set_timing(self._h, 1 if enable else 0), "ct_ctx_set_timing")

    def last_launch(self) -> dict:
        info = L.LaunchInfo()
        L.check(L.lib().ct_last_launch(self._h, C.byref(info)), "ct_last_launch")
        return {k: getattr(info, k) for k, _ in L.LaunchInfo._fields_}


# ---- parameter conversion -----------------------------------------------------------------
def estimator_params(est) -> L.EstimatorParams:
    a = [int(x) for x in est.as_array()]
    return L.EstimatorParams(a[0], a[1], a[2], a[3], a[4], a[5], a[6], 0)


def engine_params(eng) -> L.EngineParams:
    return L.EngineParams(*[int(x) for x in eng.as_array()])


class DeviceTrace:
    """A ctgen TraceSet resident in HBM (programs: 16-B records, turns: int32[T, 4])."""

    def __init__(self, trace, device=None):
        dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.trace = trace
        self.programs = torch.from_numpy(np.ascontiguousarray(trace.programs).view(np.uint8)).to(dev)
        self.turns = torch.from_numpy(np.ascontiguousarray(trace.turns, dtype=np.int32)).to(dev)
        self.n_seeds, self.n_programs, self.n_tools = trace.n_seeds, trace.n_programs, trace.n_tools

    @property
    def bytes(self) -> int:
        return self.programs.numel() + 4 * self.turns.numel()

    def struct(self) -> L.TraceSet:
        return L.TraceSet(self.programs.data_ptr(), self.turns.data_ptr(), int(self.turns.shape[0]),
                          self.n_seeds, self.n_programs, self.n_tools, 0)


class SynthesizedTrace(DeviceTrace):
    """A trace set written straight into HBM by ct_synthesize_traces (no host copy)."""

    def __init__(self, programs: torch.Tensor, turns: torch.Tensor, n_seeds: int, n_programs: int,
                 n_tools: int):
        self.trace = None
        self.programs, self.turns = programs, turns
        self.n_seeds, self.n_programs, self.n_tools = n_seeds, n_programs, n_tools


def ct_synthesize_traces(ctx: Context, sp, seed0: int, n_seeds: int, n_programs: int,
                         turns_cap: int | None = None, stream=None) -> SynthesizedTrace:
    """On-device trace synthesis (NEXT-4) of ctgen.synth's generator; `sp` is a
    ctgen.synth.SynthParams.  turns_cap defaults to n_seeds * P * max_turns."""
    dev = torch.device("cuda", ctx.device)
    tabs = [np.ascontiguousarray(x, dtype=np.int64) for x in (sp.turns_swe, sp.obs, sp.dec, sp.dur, sp.exp)]
    cdf = np.ascontiguousarray(sp.tool_cdf, dtype=np.uint32)
    cls = np.ascontiguousarray(sp.tool_class, dtype=np.int32)
    p = L.SynthParams(int(sp.stream), int(sp.ctx_cap), int(sp.max_turns), int(sp.n_bfcl), len(cdf), 0,
                      *[t.ctypes.data for t in tabs], cdf.ctypes.data, cls.ctypes.data)
    if turns_cap is None:
        turns_cap = n_seeds * n_programs * int(sp.max_turns)
    progs = torch.empty(16 * n_seeds * n_programs, dtype=torch.uint8, device=dev)
    turns = torch.empty((max(turns_cap, 1), 4), dtype=torch.int32, device=dev)
    nt = C.c_int64(0)
    rc = L.lib().ct_synthesize_traces(ctx.handle, C.byref(p), int(seed0), int(n_seeds),
                                      int(n_programs), progs.data_ptr(), turns.data_ptr(),
                                      int(turns_cap), C.byref(nt), _stream_ptr(stream))
    L.check(rc, "ct_synthesize_traces")
    return SynthesizedTrace(progs, turns[: nt.value], n_seeds, n_programs, len(cdf))


class _SweepStruct:
    """Keeps the host axis arrays alive for the duration of a call."""

    def __init__(self, sweep, fitted: torch.Tensor | None = None):
        self.gap = np.ascontiguousarray(sweep.gap_us, dtype=np.int64)
        self.kv = np.ascontiguousarray(sweep.kv_blocks, dtype=np.int64)
        pols = (L.Policy * len(sweep.policies))()
        for i, p in enumerate(sweep.policies):
            pols[i] = L.Policy(p.priority, p.pause, p.dram, p.flags, p.t_pin_us, p.t_thresh_us, (0, 0))
        self.pols = pols
        self.fitted = fitted
        fptr, fj, frows = 0, 0, 0
        if fitted is not None:
            assert fitted.is_cuda and fitted.dtype == torch.int64 and fitted.is_contiguous()
            fptr, fj, frows = fitted.data_ptr(), int(fitted.shape[1]), int(fitted.shape[0])
        self.s = L.Sweep(sweep.n_seeds, len(self.gap), len(self.kv), len(sweep.policies),
                         self.gap.ctypes.data, self.kv.ctypes.data, C.addressof(pols),
                         estimator_params(sweep.estimator), fptr, fj, frows)


def _fitted_tensor(sweep, device):
    if sweep.fitted is None:
        return None
    f = sweep.fitted
    if isinstance(f, torch.Tensor):
        return f.to(device=device, dtype=torch.int64).contiguous()
    return torch.from_numpy(np.ascontiguousarray(f, dtype=np.int64)).to(device)


# ---- the three calls ----------------------------------------------------------------------
def ct_simulate_batch(ctx: Context, trace: DeviceTrace, sweep, engine, replica_begin: int = 0,
                      replica_end: int | None = None, out: torch.Tensor | None = None,
                      jct: torch.Tensor | bool | None = None, stream=None,
                      bubble: torch.Tensor | bool | None = None):
    """Replay replicas [replica_begin, replica_end) on the GPU.

    Returns (summary int64[R, 16] device tensor, jct int64[R, P] device tensor or None), plus
    the per-program bubble int64[R, P] as a third element when `bubble` is given
    (ct_simulate_batch_ex).
    """
    if replica_end is None:
        replica_end = sweep.n_replicas
    R = replica_end - replica_begin
    dev = trace.turns.device
    if out is None:
        out = torch.empty((max(R, 0), 16), dtype=torch.int64, device=dev)
    if jct is True:
        jct = torch.empty((max(R, 0), trace.n_programs), dtype=torch.int64, device=dev)
    elif jct is False:
        jct = None
    sw = _SweepStruct(sweep, _fitted_tensor(sweep, dev))
    ts = trace.struct()
    eng = engine_params(engine)
    if bubble is None or bubble is False:
        rc = L.lib().ct_simulate_batch(ctx.handle, C.byref(ts), C.byref(sw.s), C.byref(eng),
                                       int(replica_begin), int(replica_end), out.data_ptr(),
                                       jct.data_ptr() if jct is not None else None,
                                       _stream_ptr(stream))
        L.check(rc, "ct_simulate_batch")
        return out, jct
    if bubble is True:
        bubble = torch.empty((max(R, 0), trace.n_programs), dtype=torch.int64, device=dev)
    o = L.ReplayOutputs(out.data_ptr(), jct.data_ptr() if jct is not None else None,
                        bubble.data_ptr())
    rc = L.lib().ct_simulate_batch_ex(ctx.handle, C.byref(ts), C.byref(sw.s), C.byref(eng),
                                      int(replica_begin), int(replica_end), C.byref(o),
                                      _stream_ptr(stream))
    L.check(rc, "ct_simulate_batch_ex")
    return out, jct, bubble


def ct_simulate_batch_host(ctx: Context, trace, sweep, engine, replica_begin: int = 0,
                           replica_end: int | None = None, out: torch.Tensor | None = None,
                           jct: torch.Tensor | None = None, stream=None,
                           programs: torch.Tensor | None = None, turns: torch.Tensor | None = None):
    """End-to-end call with HOST buffers (pinned torch tensors recommended).

    programs (uint8 [S*P*16]) and turns (int32 [T, 4]) default to pinned copies of `trace`;
    out (int64 [R, 16]) and jct (int64 [R, P] or None) are host tensors.  Synchronises.
    """
    if replica_end is None:
        replica_end = sweep.n_replicas
    R = replica_end - replica_begin
    if programs is None:
        programs = torch.from_numpy(np.ascontiguousarray(trace.programs).view(np.uint8)).pin_memory()
    if turns is None:
        turns = torch.from_numpy(np.ascontiguousarray(trace.turns, dtype=np.int32)).pin_memory()
    if out is None:
        out = torch.empty((R, 16), dtype=torch.int64).pin_memory()
    dev = torch.device("cuda", ctx.device)
    sw = _SweepStruct(sweep, _fitted_tensor(sweep, dev))
    ts = L.TraceSet(programs.data_ptr(), turns.data_ptr(), int(turns.shape[0]), trace.n_seeds,
                    trace.n_programs, trace.n_tools, 0)
    eng = engine_params(engine)
    rc = L.lib().ct_simulate_batch_host(ctx.handle, C.byref(ts), C.byref(sw.s), C.byref(eng),
                                        int(replica_begin), int(replica_end), out.data_ptr(),
                                        jct.data_ptr() if jct is not None else None,
                                        _stream_ptr(stream))
    L.check(rc, "ct_simulate_batch_host")
    return out, jct


def cost_params(c_pf_ps: int, c_pin_ps: int, bs: int, a_num: int, a_den: int, grid_step_us: int,
                K: int, ctx_tokens, turn_weight, avg_turns=(0, 0)) -> L.CostParams:
    J = len(ctx_tokens)
    assert J == len(turn_weight) and 1 <= J <= L.MAX_J
    cp = L.CostParams()
    cp.c_pf_ps, cp.c_pin_ps, cp.bs, cp.a_num, cp.a_den = c_pf_ps, c_pin_ps, bs, a_num, a_den
    cp.grid_step_us, cp.K, cp.J = grid_step_us, K, J
    for j in range(J):
        cp.ctx_tokens[j] = int(ctx_tokens[j])
        cp.turn_weight[j] = int(turn_weight[j])
    cp.avg_turns_num, cp.avg_turns_den = int(avg_turns[0]), int(avg_turns[1])
    return cp


def _samples(dur_us: torch.Tensor, tool_off, tool_u8: torch.Tensor | None, n_tools: int | None):
    assert dur_us.is_cuda and dur_us.dtype == torch.int32 and dur_us.is_contiguous()
    if tool_off is None:  # unsorted (dur, u8 tool) layout
        assert tool_u8 is not None and tool_u8.is_cuda and tool_u8.dtype == torch.uint8
        assert tool_u8.is_contiguous() and tool_u8.numel() == dur_us.numel() and n_tools
        return L.Samples(dur_us.data_ptr(), None, tool_u8.data_ptr(), int(dur_us.numel()),
                         int(n_tools), 0), int(n_tools), None
    off = np.ascontiguousarray(tool_off, dtype=np.int64)
    F = off.shape[0] - 1
    return L.Samples(dur_us.data_ptr(), off.ctypes.data, None, int(off[-1]), F, 0), F, off


def _table(F: int, J: int, dev, want_stats: bool):
    arg = torch.empty((F + 1, J), dtype=torch.int64, device=dev)
    pap = torch.empty(F + 1, dtype=torch.int64, device=dev)
    st = torch.empty((F + 1, 4), dtype=torch.int64, device=dev) if want_stats else None
    bad = torch.empty(1, dtype=torch.int64, device=dev)
    tab = L.TtlTable(arg.data_ptr(), pap.data_ptr(), st.data_ptr() if st is not None else None,
                     bad.data_ptr())
    return arg, pap, st, bad, tab


def ct_fit_ttl(ctx: Context, dur_us: torch.Tensor, tool_off, cost: L.CostParams, est, stream=None,
               want_stats: bool = True, tool_u8: torch.Tensor | None = None,
               n_tools: int | None = None, want_invalid: bool = False):
    """TTL fit over device samples.

    CSR layout: dur_us int32 device tensor [n] grouped by tool, tool_off host int64 [F+1].
    Unsorted layout: tool_off=None, tool_u8 uint8 device tensor [n], n_tools = F.
    Returns (ttl_argmax int64[F+1, J], ttl_paper int64[F+1], stats int64[F+1, 4] or None), plus
    n_invalid int64[1] (device) when want_invalid.
    """
    sm, F, _off = _samples(dur_us, tool_off, tool_u8, n_tools)
    arg, pap, st, bad, tab = _table(F, cost.J, dur_us.device, want_stats)
    e = estimator_params(est)
    rc = L.lib().ct_fit_ttl(ctx.handle, C.byref(sm), C.byref(cost), C.byref(e), C.byref(tab),
                            _stream_ptr(stream))
    L.check(rc, "ct_fit_ttl")
    return (arg, pap, st, bad) if want_invalid else (arg, pap, st)


def ct_fit_acc_words(n_tools: int, K: int) -> int:
    w = int(L.lib().ct_fit_acc_words(int(n_tools), int(K)))
    if w < 0:
        raise L.CtError("ct_fit_acc_words: n_tools / K out of range")
    return w


def ct_fit_ttl_partial(ctx: Context, dur_us: torch.Tensor, tool_off, cost: L.CostParams, est,
                       rank: int, world: int, acc: torch.Tensor | None = None, stream=None):
    """Accumulator (int64 [ct_fit_acc_words(F, K)], device) of this rank's slice of every tool
    segment; sum it over the ranks (all-reduce) and pass it to ct_fit_ttl_finish."""
    sm, F, _off = _samples(dur_us, tool_off, None, None)
    if acc is None:
        acc = torch.empty(ct_fit_acc_words(F, cost.K), dtype=torch.int64, device=dur_us.device)
    assert acc.is_cuda and acc.dtype == torch.int64 and acc.numel() >= ct_fit_acc_words(F, cost.K)
    e = estimator_params(est)
    rc = L.lib().ct_fit_ttl_partial(ctx.handle, C.byref(sm), C.byref(cost), C.byref(e), int(rank),
                                    int(world), acc.data_ptr(), _stream_ptr(stream))
    L.check(rc, "ct_fit_ttl_partial")
    return acc


def ct_fit_ttl_finish(ctx: Context, acc: torch.Tensor, n_tools: int, cost: L.CostParams, est,
                      stream=None, want_stats: bool = True, want_invalid: bool = False):
    """Tables from a (reduced) accumulator; same outputs as ct_fit_ttl."""
    assert acc.is_cuda and acc.dtype == torch.int64 and acc.is_contiguous()
    arg, pap, st, bad, tab = _table(int(n_tools), cost.J, acc.device, want_stats)
    e = estimator_params(est)
    rc = L.lib().ct_fit_ttl_finish(ctx.handle, acc.data_ptr(), int(n_tools), C.byref(cost),
                                   C.byref(e), C.byref(tab), _stream_ptr(stream))
    L.check(rc, "ct_fit_ttl_finish")
    return (arg, pap, st, bad) if want_invalid else (arg, pap, st)


def _stat_row(r) -> L.StatRow:
    """(n, s1, s2) with s2 a Python int, or (n, s1, s2_lo, s2_hi)."""
    r = [int(x) for x in r]
    if len(r) == 3:
        r = [r[0], r[1], r[2] & (2**64 - 1), r[2] >> 64]
    return L.StatRow(r[0], r[1], r[2] & (2**64 - 1), r[3] & (2**64 - 1))


def ct_bernstein(ctx: Context, rows: torch.Tensor, est, stream=None) -> torch.Tensor:
    """B(delta) per statistics row; rows int64 device tensor [n, 4] = {n, s1, s2_lo, s2_hi}."""
    assert rows.is_cuda and rows.dtype == torch.int64 and rows.shape[-1] == 4 and rows.is_contiguous()
    out = torch.empty(rows.shape[0], dtype=torch.int64, device=rows.device)
    e = estimator_params(est)
    rc = L.lib().ct_bernstein(ctx.handle, rows.data_ptr(), int(rows.shape[0]), C.byref(e),
                              out.data_ptr(), _stream_ptr(stream))
    L.check(rc, "ct_bernstein")
    return out


def ct_calc_ttl_batch(ctx: Context, g: torch.Tensor, f: torch.Tensor, n_done: torch.Tensor,
                      turns_done: torch.Tensor, est, stream=None) -> torch.Tensor:
    """CalcTTL offset per query (global row g[i], tool row f[i], D = n_done[i])."""
    n = int(g.shape[0])
    for t in (g, f, n_done, turns_done):
        assert t.is_cuda and t.dtype == torch.int64 and t.is_contiguous() and t.shape[0] == n
    out = torch.empty(n, dtype=torch.int64, device=g.device)
    e = estimator_params(est)
    rc = L.lib().ct_calc_ttl_batch(ctx.handle, g.data_ptr(), f.data_ptr(), n_done.data_ptr(),
                                   turns_done.data_ptr(), n, C.byref(e), out.data_ptr(),
                                   _stream_ptr(stream))
    L.check(rc, "ct_calc_ttl_batch")
    return out


def ct_bernstein_ref(row, est) -> int:
    e = estimator_params(est)
    r = _stat_row(row)
    return int(L.lib().ct_bernstein_ref(C.byref(r), C.byref(e)))


def ct_calc_ttl_ref(g, f, est, n_done: int, turns_done: int) -> int:
    e = estimator_params(est)
    gr, fr = _stat_row(g), _stat_row(f)
    return int(L.lib().ct_calc_ttl_ref(C.byref(gr), C.byref(fr), C.byref(e), int(n_done),
                                       int(turns_done)))


def ct_validate_trace_set(ctx: Context, trace: "DeviceTrace", sweep, replica_begin: int = 0,
                          replica_end: int | None = None, stream=None) -> None:
    """Synchronous check of a device trace set against ct_simulate_batch's preconditions;
    raises CtError naming the first invalid program."""
    sw = _SweepStruct(sweep, _fitted_tensor(sweep, trace.programs.device))
    re_ = sweep.n_replicas if replica_end is None else int(replica_end)
    rc = L.lib().ct_validate_trace_set(ctx.handle, C.byref(trace.struct()), C.byref(sw.s),
                                       int(replica_begin), re_, _stream_ptr(stream))
    L.check(rc, "ct_validate_trace_set")


def ct_jct_stats(ctx: Context, summary: torch.Tensor, n_cells: int, out: torch.Tensor | None = None,
                 stream=None) -> torch.Tensor:
    assert summary.is_cuda and summary.dtype == torch.int64 and summary.shape[1] == 16
    if out is None:
        out = torch.empty((n_cells, 8), dtype=torch.int64, device=summary.device)
    rc = L.lib().ct_jct_stats(ctx.handle, summary.data_ptr(), int(summary.shape[0]), int(n_cells),
                              out.data_ptr(), _stream_ptr(stream))
    L.check(rc, "ct_jct_stats")
    return out


def status(summary: torch.Tensor | np.ndarray):
    return summary[:, 0] & 0xFFFFFFFF


# ---- host-side trace ingest (NEXT-4; csrc/ingest.cpp) -------------------------------------------
TOOLFMT = {"auto": 0, "openai": 1, "name": 2, "pythonic": 3, "bash": 4, "terminal": 5}


def ct_parse_tool_name(msg, fmt: str | int = "auto") -> tuple[str | None, bool]:
    """Tool name of one model output message (App. A): (name or None,
    malformed)."""
    b = msg.encode() if isinstance(msg, str) else bytes(msg)
    f = TOOLFMT[fmt] if isinstance(fmt, str) else int(fmt)
    cap = len(b) + 1
    buf = C.create_string_buffer(cap)
    n, bad = C.c_int32(0), C.c_int32(0)
    L.check(L.lib().ct_parse_tool_name(b, len(b), f, buf, cap, C.byref(n), C.byref(bad)),
            "ct_parse_tool_name")
    return (buf.raw[: n.value].decode("utf-8", "surrogateescape") if n.value else None,
            bool(bad.value))


def ct_load_trace_jsonl(path: str, fmt: str | int = "auto", ctx_window: int = 0,
                        known_tools=()):
    """Load a JSONL agent trace (one program per line) into one seed of replay records.

    Returns (ctgen TraceSet with n_seeds = 1, tool names by id, malformed-message count).
    arr_q holds the recorded arrival in µs: replay it with gap_us = 2^20 for the recorded
    arrival process (any other gap rescales it)."""
    from ctgen.traces import PROG_DTYPE, TraceSet
    f = TOOLFMT[fmt] if isinstance(fmt, str) else int(fmt)
    names = C.create_string_buffer(64 * 64)
    for i, nm in enumerate(known_tools):
        e = nm.encode()
        names[64 * i: 64 * i + len(e)] = e
    counts = (C.c_int64 * 5)()
    p = path.encode()
    lib = L.lib()
    L.check(lib.ct_load_trace_jsonl(p, f, int(ctx_window), names, len(known_tools), None, 0, None,
                                    0, counts), "ct_load_trace_jsonl")
    n_p, n_t = int(counts[0]), int(counts[1])
    progs = np.zeros(n_p, dtype=PROG_DTYPE)
    turns = np.zeros((n_t, 4), dtype=np.int32)
    L.check(lib.ct_load_trace_jsonl(p, f, int(ctx_window), names, len(known_tools),
                                    progs.ctypes.data, n_p, turns.ctypes.data, n_t, counts),
            "ct_load_trace_jsonl")
    n_f = int(counts[2])
    tools = [names.raw[64 * i: 64 * (i + 1)].split(b"\0", 1)[0].decode() for i in range(n_f)]
    tr = TraceSet(progs, turns, 1, n_p, max(n_f, 1), np.zeros(n_p, np.uint8))
    return tr, tools, int(counts[3])
