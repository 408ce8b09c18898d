"""libcontinuum: B200-native batched trace-replay of Continuum's KV-cache TTL scheduler.

Product path only: C ABI in include/continuum.h, CUDA kernels in csrc/, ctypes binding
in api.py.  No CPU fallback.
"""
from .api import (Context, DeviceTrace, SynthesizedTrace, ct_synthesize_traces,  # noqa: F401
                  ct_fit_ttl, ct_jct_stats, ct_simulate_batch,  # noqa: F401
                  ct_simulate_batch_host, cost_params, status, SUMMARY_FIELDS,  # noqa: F401
                  ct_parse_tool_name, ct_load_trace_jsonl)

__all__ = ["Context", "DeviceTrace", "SynthesizedTrace", "ct_synthesize_traces", "ct_fit_ttl",
           "ct_jct_stats", "ct_simulate_batch",
           "ct_simulate_batch_host", "cost_params", "status", "SUMMARY_FIELDS",
           "ct_parse_tool_name", "ct_load_trace_jsonl"]
