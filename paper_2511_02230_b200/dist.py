"""Replica sharding across ranks and the single collective of the path.

Replicas are independent, so rank k of N owns the contiguous range
[R k / N, R (k+1) / N) — the mixed-radix sweep order puts every rate, KV budget and policy
inside each seed block, so contiguous ranges are balanced.  The only data-path collective is
one all-gather of the fixed-size 128-B summaries (NCCL over NVLink on B200; gloo in CPU
tests).  Integer summaries make the gathered bytes identical to a single-GPU run.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(R: int, rank: int, world: int) -> tuple[int, int]:
    return R * rank // world, R * (rank + 1) // world


def shard_capacity(R: int, world: int) -> int:
    """Rows per rank in the padded gather buffer."""
    return (R + world - 1) // world


def gather_summaries(summ_shard: torch.Tensor, R: int, world: int, out: torch.Tensor | None = None,
                     group=None) -> torch.Tensor:
    """All-gather each rank's [cap, 16] padded shard and return the [R, 16] sweep-ordered view."""
    cap = summ_shard.shape[0]
    assert cap == shard_capacity(R, world)
    if world == 1:
        return summ_shard[:R]
    if out is None:
        out = torch.empty((cap * world, summ_shard.shape[1]), dtype=summ_shard.dtype,
                          device=summ_shard.device)
    dist.all_gather_into_tensor(out, summ_shard, group=group)
    if R % world == 0:  # equal shards: the gathered buffer is already in sweep order
        return out[:R]
    parts = []
    for k in range(world):
        a, b = shard_range(R, k, world)
        parts.append(out[k * cap: k * cap + (b - a)])
    return torch.cat(parts)
