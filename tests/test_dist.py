"""World-size-2 gloo test of the multi-rank path on CPU: sharding + the summary all-gather.

The per-rank compute is stood in by the oracle (CPU); what is tested is the host logic the
GPU path uses (paper_2511_02230_b200.dist): shard ranges, padding, the collective and the
reassembly, which must reproduce the single-process result byte for byte.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2511_02230_b200 import dist as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, n_rates):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from ctgen import configs as cf
    from ctgen import traces
    from oracle import oracle as O
    tr = traces.generate(3, 8, n_bfcl=4, mix="mix", ctx_cap=8192 * 16, stream=11)
    sw = cf.Sweep(3, cf.rate_axis(n_rates), [8192], [cf.ttl_grid(t) for t in cf.ttl_axis(3)])
    R = sw.n_replicas  # 27: ragged over 2 ranks (reassembled); 36: equal shards (no copy)
    a, b = D.shard_range(R, rank, world)
    cap = D.shard_capacity(R, world)
    s, _ = O.simulate(tr, sw, cf.ENGINE_8B, a, b, want_jct=False)
    shard = torch.zeros((cap, 16), dtype=torch.int64)
    shard[: b - a] = torch.from_numpy(s)
    full = D.gather_summaries(shard, R, world)
    if rank == 0:
        ref, _ = O.simulate(tr, sw, cf.ENGINE_8B, 0, R, want_jct=False)
        q.put(bool(np.array_equal(full.numpy(), ref)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n_rates", [3, 4])
def test_gloo_world2_gather_equals_single_process(n_rates):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q, n_rates)) for r in range(2)]
    for p in ps:
        p.start()
    ok = q.get(timeout=300)
    for p in ps:
        p.join(timeout=120)
    assert ok
    assert all(p.exitcode == 0 for p in ps)


def test_shard_ranges_cover():
    for R in (1, 7, 64, 1 << 20):
        for w in (1, 2, 3, 8):
            rs = [D.shard_range(R, k, w) for k in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == R
            assert all(rs[k][1] == rs[k + 1][0] for k in range(w - 1))
            assert max(b - a for a, b in rs) <= D.shard_capacity(R, w)
