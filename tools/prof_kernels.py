"""Small driver for ncu captures: one kernel family per invocation.

  python tools/prof_kernels.py fit [log2n]        -> ct_fit_ttl on 2^log2n samples (3 calls)
  python tools/prof_kernels.py replay [cfg] [seeds] -> one ct_simulate_batch of a config
Prints timing from CUDA events (not a bench number when run under ncu).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_2511_02230_b200 as ct
from ctgen import configs as cf

if os.environ.get("AB_LIB"):  # tools/ab.sh: an experimental build of the library (A/B runs)
    from paper_2511_02230_b200 import _lib
    _lib.LIB_PATH = os.environ["AB_LIB"]
from ctgen import traces


def main():
    what = sys.argv[1]
    ctx = ct.Context(0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if what == "fit":
        log2n = int(sys.argv[2]) if len(sys.argv) > 2 else 28
        dur, off = traces.synthetic_samples_torch(log2n, 32, 1234, "cuda")
        cp = ct.cost_params(13_400_000, 200, 16, 1, 10, 50_000, 256,
                            [min(16 * 2**j, 120_000) for j in range(64)], list(range(1, 65)))
        est = cf.Estimator()
        n = 1 << log2n
        acc = torch.zeros(ct.ct_fit_acc_words(32, 256), dtype=torch.int64, device="cuda")

        def fused():
            ct.ct_fit_ttl(ctx, dur, off, cp, est, want_stats=False)

        def split():
            ct.ct_fit_ttl_partial(ctx, dur, off, cp, est, 0, 1, acc=acc)
            ct.ct_fit_ttl_finish(ctx, acc, 32, cp, est, want_stats=False)

        for name, fn in (("fused", fused), ("partial+finish", split)):
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            reps = 20
            e0.record()
            for _ in range(reps):
                fn()
            e1.record()
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1) / 1e3 / reps
            ctx.set_timing(True)
            ks = []
            for _ in range(reps):
                fn()
                ks.append(ctx.last_launch()["fit_hist_ms"])
            ctx.set_timing(False)
            k = sorted(ks)[reps // 2] / 1e3
            print("fit %s n=2^%d: call %.1f us (%.0f GB/s), kernel median %.1f us (%.0f GB/s)" % (
                name, log2n, t * 1e6, 4 * n / t / 1e9, k * 1e6, 4 * n / k / 1e9))
        for _ in range(2):
            dur.max()
        e0.record()
        for _ in range(20):
            dur.max()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 1e3 / 20
        print("read probe (torch max): %.1f us, %.0f GB/s" % (t * 1e6, 4 * n / t / 1e9))
    else:
        name = sys.argv[2] if len(sys.argv) > 2 else "cfg3"
        seeds = int(sys.argv[3]) if len(sys.argv) > 3 else 16
        if name == "cont":  # cfg3's workload under program-FCFS-class policies with the estimator
            w = cf.config3(n_seeds=seeds)
            pols = [cf.CONTINUUM, cf.simplified(5_000_000, 2_000_000), cf.PROG_FCFS] + \
                [cf.ttl_grid(t) for t in cf.ttl_axis(13, 100_000, 60_000_000)[1:]]
            w = cf.Workload("cont", w.trace, cf.Sweep(seeds, cf.rate_axis(16), [8192], pols),
                            w.engine, "cfg3 trace, 16 program-FCFS policies")
        else:
            w = {"cfg2": cf.config2, "cfg3": cf.config3, "cfg4": cf.config4,
                 "cfg5": cf.config5}[name](n_seeds=seeds)
            if name == "cfg4":  # the FITTED policy replays ct_fit_ttl's table (bench's cfg4 step)
                dur, off = traces.tool_samples(w.trace)
                p, c = cf.CFG4_FIT, cf.cfg4_fit_cost(w.engine)
                cp = ct.cost_params(*c[:7], p["ctx_j"], p["w_j"])
                w.sweep.fitted = ct.ct_fit_ttl(ctx, torch.from_numpy(dur).cuda(), off, cp,
                                               w.sweep.estimator)[0][:-1]
        dt = ct.DeviceTrace(w.trace)
        for i in range(2):
            e0.record()
            s, _ = ct.ct_simulate_batch(ctx, dt, w.sweep, w.engine, jct=False)
            e1.record()
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1) / 1e3
            turns = int(s[:, 1].sum())
            print("replay %s seeds=%d: %d replicas %d turns %.3f ms %.3e turns/s launch=%s" % (
                name, seeds, w.sweep.n_replicas, turns, t * 1e3, turns / t, ctx.last_launch()))


if __name__ == "__main__":
    main()
