"""ctypes view of include/continuum.h (argument marshalling only).

Loads the in-tree libcontinuum.so.  There is no fallback: if the library is missing the
import fails loudly (build it with `python -m paper_2511_02230_b200.build`).
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libcontinuum.so")

i32, i64, u64, vp = C.c_int32, C.c_int64, C.c_uint64, C.c_void_p

CT_OK, CT_EINVAL, CT_ENOMEM, CT_ECUDA, CT_EUNSUPPORTED = 0, -1, -2, -3, -4
MAX_J = 64

# every symbol include/continuum.h declares (checked by tests/test_abi.py)
EXPORTS = ["ct_version", "ct_last_error", "ct_ctx_create", "ct_ctx_destroy", "ct_fit_ttl",
           "ct_fit_acc_words", "ct_fit_ttl_partial", "ct_fit_ttl_finish", "ct_bernstein",
           "ct_calc_ttl_batch", "ct_bernstein_ref", "ct_calc_ttl_ref", "ct_validate_trace_set",
           "ct_simulate_batch", "ct_simulate_batch_ex", "ct_simulate_batch_host", "ct_jct_stats",
           "ct_last_launch", "ct_ctx_set_timing", "ct_synthesize_traces", "ct_parse_tool_name",
           "ct_load_trace_jsonl"]


class SynthParams(C.Structure):
    _fields_ = [("stream", i64), ("ctx_cap", i64), ("max_turns", i32), ("n_bfcl", i32),
                ("n_tools", i32), ("reserved", i32), ("turns_swe", vp), ("obs", vp), ("dec", vp),
                ("dur", vp), ("exp_q20", vp), ("tool_cdf", vp), ("tool_class", vp)]


class ReplayOutputs(C.Structure):
    _fields_ = [("summary", vp), ("jct_us", vp), ("bubble_us", vp)]


class TraceSet(C.Structure):
    _fields_ = [("programs", vp), ("turns", vp), ("n_turns", i64), ("n_seeds", i32),
                ("n_programs", i32), ("n_tools", i32), ("reserved", i32)]


class EstimatorParams(C.Structure):
    _fields_ = [("lq", u64), ("b_us", i64), ("t_default_us", i64), ("n_min", i64), ("a_num", i64),
                ("a_den", i64), ("ttl_max_us", i64), ("reserved", i64)]


class EngineParams(C.Structure):
    _fields_ = [("c0_ps", i64), ("c_pf_ps", i64), ("c_kv_ps", i64), ("c_h2d_ps", i64), ("bs", i64),
                ("max_batch", i64), ("dram_blocks", i64), ("max_iters", i64), ("kv_growth", i64),
                ("prefill_chunk", i64)]


class Policy(C.Structure):
    _fields_ = [("priority", i32), ("pause", i32), ("dram", i32), ("flags", i32), ("t_pin_us", i64),
                ("t_thresh_us", i64), ("reserved", i64 * 2)]


class Sweep(C.Structure):
    _fields_ = [("n_seeds", i32), ("n_rates", i32), ("n_kv", i32), ("n_policies", i32),
                ("gap_us", vp), ("kv_blocks", vp), ("policies", vp), ("est", EstimatorParams),
                ("fitted_ttl", vp), ("fitted_j", i32), ("fitted_rows", i32)]


class Samples(C.Structure):
    _fields_ = [("dur_us", vp), ("tool_off", vp), ("tool_u8", vp), ("n", i64), ("n_tools", i32),
                ("reserved", i32)]


class StatRow(C.Structure):
    _fields_ = [("n", i64), ("s1", i64), ("s2_lo", u64), ("s2_hi", u64)]


class CostParams(C.Structure):
    _fields_ = [("c_pf_ps", i64), ("c_pin_ps", i64), ("bs", i64), ("a_num", i64), ("a_den", i64),
                ("grid_step_us", i64), ("K", i32), ("J", i32), ("ctx_tokens", i64 * MAX_J),
                ("turn_weight", i64 * MAX_J), ("avg_turns_num", i64), ("avg_turns_den", i64)]


class TtlTable(C.Structure):
    _fields_ = [("ttl_argmax", vp), ("ttl_paper", vp), ("stats", vp), ("n_invalid", vp)]


class LaunchInfo(C.Structure):
    _fields_ = [("grid", i32), ("block", i32), ("warps_per_block", i32), ("slots_per_lane", i32),
                ("smem_per_block", i64), ("launches", i64), ("replay_ms", C.c_float),
                ("fit_hist_ms", C.c_float), ("kernel_mode", i32), ("reserved", i32)]


assert C.sizeof(Policy) == 48 and C.sizeof(EngineParams) == 80 and C.sizeof(EstimatorParams) == 64

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError("libcontinuum.so not built (%s); run `python -m paper_2511_02230_b200.build`"
                              % LIB_PATH)
        L = C.CDLL(LIB_PATH)
        L.ct_version.restype = C.c_int
        L.ct_last_error.restype = C.c_char_p
        L.ct_ctx_create.argtypes = [C.c_int, C.POINTER(vp)]
        L.ct_ctx_destroy.argtypes = [vp]
        L.ct_fit_ttl.argtypes = [vp, C.POINTER(Samples), C.POINTER(CostParams),
                                 C.POINTER(EstimatorParams), C.POINTER(TtlTable), vp]
        L.ct_fit_acc_words.restype = i64
        L.ct_fit_acc_words.argtypes = [i32, i32]
        L.ct_fit_ttl_partial.argtypes = [vp, C.POINTER(Samples), C.POINTER(CostParams),
                                         C.POINTER(EstimatorParams), i32, i32, vp, vp]
        L.ct_fit_ttl_finish.argtypes = [vp, vp, i32, C.POINTER(CostParams),
                                        C.POINTER(EstimatorParams), C.POINTER(TtlTable), vp]
        L.ct_bernstein.argtypes = [vp, vp, i64, C.POINTER(EstimatorParams), vp, vp]
        L.ct_calc_ttl_batch.argtypes = [vp, vp, vp, vp, vp, i64, C.POINTER(EstimatorParams), vp, vp]
        L.ct_bernstein_ref.restype = i64
        L.ct_bernstein_ref.argtypes = [C.POINTER(StatRow), C.POINTER(EstimatorParams)]
        L.ct_calc_ttl_ref.restype = i64
        L.ct_calc_ttl_ref.argtypes = [C.POINTER(StatRow), C.POINTER(StatRow),
                                      C.POINTER(EstimatorParams), i64, i64]
        L.ct_validate_trace_set.argtypes = [vp, C.POINTER(TraceSet), C.POINTER(Sweep), i64, i64, vp]
        L.ct_simulate_batch.argtypes = [vp, C.POINTER(TraceSet), C.POINTER(Sweep),
                                        C.POINTER(EngineParams), i64, i64, vp, vp, vp]
        L.ct_simulate_batch_ex.argtypes = [vp, C.POINTER(TraceSet), C.POINTER(Sweep),
                                           C.POINTER(EngineParams), i64, i64,
                                           C.POINTER(ReplayOutputs), vp]
        L.ct_simulate_batch_host.argtypes = [vp, C.POINTER(TraceSet), C.POINTER(Sweep),
                                             C.POINTER(EngineParams), i64, i64, vp, vp, vp]
        L.ct_jct_stats.argtypes = [vp, vp, i64, i32, vp, vp]
        L.ct_synthesize_traces.argtypes = [vp, C.POINTER(SynthParams), i64, i32, i32, vp, vp, i64,
                                           C.POINTER(i64), vp]
        L.ct_last_launch.argtypes = [vp, C.POINTER(LaunchInfo)]
        L.ct_ctx_set_timing.argtypes = [vp, C.c_int]
        L.ct_parse_tool_name.argtypes = [C.c_char_p, i64, i32, C.c_char_p, i32, C.POINTER(i32),
                                         C.POINTER(i32)]
        L.ct_load_trace_jsonl.argtypes = [C.c_char_p, i32, i64, vp, i32, vp, i64, vp, i64,
                                          C.POINTER(i64)]
        for f in ("ct_ctx_create", "ct_ctx_destroy", "ct_fit_ttl", "ct_fit_ttl_partial",
                  "ct_fit_ttl_finish", "ct_bernstein", "ct_calc_ttl_batch",
                  "ct_validate_trace_set", "ct_simulate_batch",
                  "ct_simulate_batch_ex", "ct_simulate_batch_host", "ct_synthesize_traces", "ct_jct_stats", "ct_last_launch", "ct_ctx_set_timing",
                  "ct_parse_tool_name", "ct_load_trace_jsonl"):
            getattr(L, f).restype = C.c_int
        _lib = L
    return _lib


class CtError(RuntimeError):
    pass


def check(rc: int, what: str) -> None:
    if rc != CT_OK:
        msg = lib().ct_last_error()
        raise CtError("%s failed (%d): %s" % (what, rc, msg.decode() if msg else ""))
