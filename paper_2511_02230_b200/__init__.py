"""libcontinuum: B200-native batched trace-replay of Continuum's KV-cache TTL scheduler.

Product path only: C ABI in include/continuum.h, CUDA kernels in csrc/, ctypes binding
in api.py.  No CPU fallback.
"""
from .api import (Context, DeviceTrace, SynthesizedTrace, ct_synthesize_traces,  # noqa: F401
                  ct_fit_ttl, ct_fit_acc_words, ct_fit_ttl_partial,  # noqa: F401
                  ct_fit_ttl_finish, ct_jct_stats, ct_simulate_batch,  # noqa: F401
                  ct_bernstein, ct_calc_ttl_batch, ct_bernstein_ref, ct_calc_ttl_ref,  # noqa: F401
                  ct_validate_trace_set,  # noqa: F401
                  ct_simulate_batch_host, cost_params, status, SUMMARY_FIELDS,  # noqa: F401
                  ct_parse_tool_name, ct_load_trace_jsonl)

__all__ = ["Context", "DeviceTrace", "SynthesizedTrace", "ct_synthesize_traces", "ct_fit_ttl",
           "ct_fit_acc_words", "ct_fit_ttl_partial", "ct_fit_ttl_finish", "ct_bernstein",
           "ct_calc_ttl_batch", "ct_bernstein_ref", "ct_calc_ttl_ref", "ct_validate_trace_set",
           "ct_jct_stats", "ct_simulate_batch",
           "ct_simulate_batch_host", "cost_params", "status", "SUMMARY_FIELDS",
           "ct_parse_tool_name", "ct_load_trace_jsonl"]
