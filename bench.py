#!/usr/bin/env python
"""bench.py — libcontinuum on B200: replica-turns/s of the TTL sweep (+ ttl_fit HBM GB/s).

One step = one pass of the whole hot path over one batch of synthetic input:
  A-2  ct_fit_ttl over the workload's tool-duration samples (TTL tables)
  A-1, A-3..A-8  ct_simulate_batch over this rank's contiguous replica shard
  A-9  all_gather_into_tensor of the 128-B summaries (N > 1, NCCL)
  A-8  ct_jct_stats per sweep cell
Inputs are resident in HBM before the timed region; L2 is flushed at the start of every step.
Default workload: BASELINE configs[2] (64 arrival rates x 64 TTLs x 256 seeds = 2^20 replicas on
a 16 BFCL + 16 SWE mix), the TTL sweep the metric names.  `--impl reference` times the CPU
oracle on the host cores instead (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "replica-turns/sec (TTL sweep, 1/2/4/8 B200) + HBM GB/s of ttl_fit vs peak"
UNIT = "replica-turns/s"
SM_COUNT = 148
ISSUE_PER_SM_CLK = 4  # warp schedulers per SM, 1 warp-instruction / clk each


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="libcontinuum", choices=["libcontinuum", "reference"])
    ap.add_argument("--workload", default="cfg3", choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
    ap.add_argument("--seeds", type=int, default=None, help="override seed count (smaller runs)")
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--fit-log2n", type=int, default=28)
    ap.add_argument("--no-fit-bandwidth", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def load_workload(name, seeds):
    from ctgen import configs as cf
    fn = {"cfg1": cf.config1, "cfg2": cf.config2, "cfg3": cf.config3, "cfg4": cf.config4,
          "cfg5": cf.config5}[name]
    if seeds is not None and name != "cfg1":
        return fn(n_seeds=seeds)
    return fn()


def fit_inputs(trace, J=8):
    """Turn-bucket context sizes and weights for the fit (input preparation, no method math)."""
    from ctgen import traces
    dur, off = traces.tool_samples(trace)
    progs, t = trace.programs, trace.turns
    ctxj = np.zeros(J, np.int64)
    cnt = np.zeros(J, np.int64)
    for i in range(0, len(progs), max(1, len(progs) // 512)):
        t0, nt = int(progs["turn0"][i]), int(progs["nturns"][i])
        c = 0
        for k in range(nt):
            c += int(t[t0 + k, 0]) + int(t[t0 + k, 1])
            j = min(k, J - 1)
            ctxj[j] += c
            cnt[j] += 1
    ctxj = np.maximum(ctxj // np.maximum(cnt, 1), 16)
    return dur, off, [int(x) for x in ctxj], [j + 1 for j in range(J)]


def fit_cost(w, ctxj):
    """The step fit's cost parameters as the oracle's vector [c_pf, c_pin, bs, a_num, a_den,
    grid_step, K, J] (the same values main() passes to ct.cost_params)."""
    e = w.sweep.estimator
    return [w.engine.c_pf_ps, 200, w.engine.bs, e.a_num, e.a_den, 50_000, 256, len(ctxj)]


# ---------------------------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            f = [x.strip() for x in l.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(max(mx)) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured"
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback (B200_PROFILING.md)"


def profile_constants():
    """ncu-derived per-unit constants committed under profiles/ (instructions per replica-turn,
    DRAM bytes per fit launch).  Missing file -> the fields are reported as null."""
    p = os.path.join(ROOT, "profiles", "ncu_constants.json")
    return json.load(open(p)) if os.path.exists(p) else {}


# ---------------------------------------------------------------------------------------------
def oracle_fitted(w, dur_np, off, cost, ctxj, wj):
    """The oracle's own TTL table for a FITTED policy (no input to the oracle comes from the
    CUDA path): or_fit on the same samples and cost parameters the step's ct_fit_ttl used."""
    from oracle import oracle as O
    if not any(p.pause == 3 for p in w.sweep.policies):
        return w.sweep
    arg, _, _ = O.fit(dur_np, off, cost, ctxj, wj, w.sweep.estimator.as_array())
    sw = type(w.sweep)(**{**w.sweep.__dict__, "fitted": arg[:-1]})
    return sw


def cpu_baseline(w, sweep, budget_s, n_threads, gpu_summ=None):
    """The oracle as it stands, on a bounded, strided sample of the same workload:
    (b) a thread pool over the sampled replicas (each replica single-threaded), and
    (a) one thread on a prefix of the every-256th-replica subset.
    With gpu_summ (the GPU's [R, 16] summaries of this step) every sampled replica is also
    compared byte for byte (parity)."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import oracle as O
    R = sweep.n_replicas
    t0 = time.time()
    probe = list(range(0, R, max(1, R // 16)))[:4]
    for r in probe:
        O.simulate(w.trace, sweep, w.engine, r, r + 1, n_threads=1, want_jct=False)
    per_rep = (time.time() - t0) / len(probe)
    n = int(max(n_threads, min(R, budget_s * n_threads / max(per_rep, 1e-6))))
    stride = max(1, R // n)
    reps = np.arange(0, R, stride)[:n]

    def one(r):
        s, _ = O.simulate(w.trace, sweep, w.engine, int(r), int(r) + 1, n_threads=1, want_jct=False)
        return s[0]

    t0 = time.time()
    with ThreadPoolExecutor(n_threads) as ex:
        rows = np.stack(list(ex.map(one, reps)))
    dt = time.time() - t0
    turns = int(rows[:, 1].sum())
    # (a) single thread, every 256th replica, bounded to ~budget/3 s
    t0 = time.time()
    t1_turns = t1_reps = 0
    for r in range(0, R, 256):
        t1_turns += int(one(r)[1])
        t1_reps += 1
        if time.time() - t0 > budget_s / 3:
            break
    t1 = time.time() - t0
    cpu = ""
    try:
        with open("/proc/cpuinfo") as fh:
            cpu = next((l.split(":", 1)[1].strip() for l in fh if l.startswith("model name")), "")
    except OSError:
        pass
    out = {"value": turns / dt, "unit": UNIT, "cores": n_threads, "kind": "oracle",
           "cpu_model": cpu, "compiler": "g++ -O2 -std=c++17",
           "est_turns_per_step": turns / len(reps) * R, "wall_s": dt,
           "sample": "%d of %d replicas (every %d-th), %d replica-turns, %.1f s wall on %d threads"
                     % (len(reps), R, stride, turns, dt, n_threads),
           "single_thread": {"value": t1_turns / t1, "unit": UNIT + " per core", "cores": 1,
                             "sample": "replicas 0, 256, ..., %d (%d of the every-256th subset, %d "
                                       "replica-turns, %.1f s)" % (256 * (t1_reps - 1), t1_reps,
                                                                   t1_turns, t1)}}
    if gpu_summ is not None:
        bad = np.nonzero(np.any(gpu_summ[reps] != rows, axis=1))[0]
        out["parity"] = {"checked": int(len(reps)), "mismatches": int(bad.size),
                         "compared": "128-B summary of every sampled replica, GPU step vs oracle",
                         "first_mismatch": int(reps[bad[0]]) if bad.size else None}
    return out


def cpu_fit_baseline(dur_np, off, cost, ctxj, wj, est, budget_s=5.0):
    """The oracle's TTL fit (plain O(n K) definition) on a bounded prefix of the samples."""
    from oracle import oracle as O
    n = len(dur_np)
    m = min(n, 1 << 16)
    while True:
        cut = np.minimum(off, m)
        t0 = time.time()
        O.fit(dur_np[:m], cut, cost, ctxj, wj, est.as_array())
        dt = time.time() - t0
        if dt > budget_s / 4 or m >= n:
            break
        m = min(n, m * 4)
    return {"value": m / dt, "unit": "samples/s", "gbs": 4.0 * m / dt / 1e9, "cores": 1,
            "kind": "oracle", "sample": "first %d of %d samples (K = %d), %.2f s" % (m, n, cost[6], dt)}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    w = load_workload(args.workload, args.seeds)
    sweep = w.sweep
    if any(p.pause == 3 for p in sweep.policies):
        dur_np, off, ctxj, wj = fit_inputs(w.trace)
        sweep = oracle_fitted(w, dur_np, off, fit_cost(w, ctxj), ctxj, wj)
    n_threads = os.cpu_count() or 1
    per_step = min(args.cpu_seconds, 150.0 / max(1, args.steps + args.warmup))
    vals, walls, turns = [], [], []
    last = None
    for i in range(args.warmup + args.steps):
        cb = cpu_baseline(w, sweep, per_step, n_threads)
        if i >= args.warmup:
            vals.append(cb["value"])
            walls.append(cb["wall_s"])
            last = cb
    v = float(np.sum([c * t for c, t in zip(vals, walls)]) / np.sum(walls))
    last["value"] = v
    est_full = last.pop("est_turns_per_step")
    last.pop("wall_s")
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": float(np.mean(walls)) * 1e3,
            "ms_per_step_basis": "timed wall time of one step = one bounded sample of the "
                                 "workload (cpu_baseline.sample) on all host cores",
            "ms_per_full_workload_est": est_full / v * 1e3,
            "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "int64", "data": "synthetic", "impl": "reference",
            "config": {"workload": w.name, "replicas": sweep.n_replicas,
                       "programs_per_replica": w.trace.n_programs, "description": w.description},
            "cpu_baseline": last,
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------------------
def fit_bandwidth(ctx, ct, cf, log2n, dev, peaks, consts):
    """ttl_fit HBM pass: 2^log2n int32 samples (CSR by tool, F = 32, K = 256, J = 64).

    kernel: CUDA events the library records around its single fused launch (per call, host
    synchronised to read them); call: 10 back-to-back ct_fit_ttl calls between two events on the
    stream, no host synchronisation in between.  Also a read-only HBM probe (torch int32 max over
    the same 1 GiB) as the read ceiling next to the measured copy peak."""
    import torch
    from ctgen import traces
    n = 1 << log2n
    K, J = 256, 64
    dur, off = traces.synthetic_samples_torch(log2n, 32, 1234, dev)
    cp = ct.cost_params(13_400_000, 200, 16, 1, 10, 50_000, K,
                        [min(16 * 2**j, 120_000) for j in range(J)], [j + 1 for j in range(J)])
    est = cf.Estimator()
    for _ in range(3):
        ct.ct_fit_ttl(ctx, dur, off, cp, est, want_stats=False)
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    reps = 20
    ctx.set_timing(True)
    kms = []
    for _ in range(reps):
        ct.ct_fit_ttl(ctx, dur, off, cp, est, want_stats=False)
        kms.append(ctx.last_launch()["fit_hist_ms"])  # waits for this launch's end event
    ctx.set_timing(False)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        ct.ct_fit_ttl(ctx, dur, off, cp, est, want_stats=False)
    e1.record(s)
    torch.cuda.synchronize()
    t_call = e0.elapsed_time(e1) / 1e3 / reps
    t = float(np.mean(kms)) / 1e3
    # read-only probe over the same bytes
    for _ in range(2):
        dur.max()
    e0.record(s)
    for _ in range(reps):
        dur.max()
    e1.record(s)
    torch.cuda.synchronize()
    t_read = e0.elapsed_time(e1) / 1e3 / reps
    gbs = 4.0 * n / t / 1e9
    peak = float(peaks["hbm_gbs"])
    tr = consts.get("fit_dram_bytes_per_sample")
    return {"bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s", "frac": gbs / peak,
            "traffic": tr * n if tr else None,
            "kernel": "fit_hist_kernel (the histogram pass; fit_finish_kernel follows as a "
                      "programmatic dependent launch; CUDA events inside the library)",
            "samples": n, "bytes_per_sample": 4, "ms_per_launch": t * 1e3,
            "call_ms": t_call * 1e3, "call_gbs": 4.0 * n / t_call / 1e9,
            "call_frac": 4.0 * n / t_call / 1e9 / peak,
            "read_probe_gbs": 4.0 * n / t_read / 1e9,
            "read_probe": "torch int32 max over the same 1 GiB (read-only HBM ceiling estimate)",
            "note": "call = back-to-back ct_fit_ttl calls, no host synchronisation"}


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    import paper_2511_02230_b200 as ct
    from ctgen import configs as cf
    from paper_2511_02230_b200 import dist as D

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    ctx = ct.Context(local)
    peaks, peak_kind = measured_peaks()
    consts = profile_constants()

    w = load_workload(args.workload, args.seeds)
    sw, eng, tr = w.sweep, w.engine, w.trace
    R = sw.n_replicas
    rb, re_ = D.shard_range(R, rank, world)
    shard = D.shard_capacity(R, world)
    dur_np, off, ctxj, wj = fit_inputs(tr)
    J = len(ctxj)
    F = tr.n_tools
    fc = fit_cost(w, ctxj)
    cp = ct.cost_params(fc[0], fc[1], fc[2], fc[3], fc[4], fc[5], fc[6], ctxj, wj, (0, 0))
    # ---- inputs resident in HBM before the timed region --------------------------------------
    dt = ct.DeviceTrace(tr)
    dur = torch.from_numpy(dur_np).to(dev)
    summ = torch.zeros((shard, 16), dtype=torch.int64, device=dev)
    gathered = torch.zeros((shard * world, 16), dtype=torch.int64, device=dev)
    acc = torch.zeros(ct.ct_fit_acc_words(F, fc[6]), dtype=torch.int64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    ev = {"fit": [], "replay": [], "gather": []}
    # a FITTED policy (cfg4) replays with this step's ct_fit_ttl table (per-tool rows)
    fitted_policy = any(p.pause == cf.PAUSE_FITTED for p in sw.policies)

    def fit():
        """A-2: one fused launch on 1 GPU; per-rank slices of every tool
        segment + an int64 all-reduce of the accumulator + the finish kernel on N GPUs."""
        if world == 1:
            return ct.ct_fit_ttl(ctx, dur, off, cp, sw.estimator, want_stats=False)[0], 1
        ct.ct_fit_ttl_partial(ctx, dur, off, cp, sw.estimator, rank, world, acc=acc)
        dist.all_reduce(acc)
        return ct.ct_fit_ttl_finish(ctx, acc, F, cp, sw.estimator, want_stats=False)[0], 2

    def mark(key, timed):
        if not timed:
            return None
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        ev[key].append([e])
        return e

    def close(key, timed):
        if timed:
            e = torch.cuda.Event(enable_timing=True)
            e.record(stream)
            ev[key][-1].append(e)

    fit_launches = [0]

    def step(timed):
        flush.zero_()  # L2 flush (256 MiB > 126 MB L2)
        mark("fit", timed)
        arg, fit_launches[0] = fit()
        close("fit", timed)
        if fitted_policy:
            sw.fitted = arg[:F]
        mark("replay", timed)
        ct.ct_simulate_batch(ctx, dt, sw, eng, rb, re_, out=summ[: re_ - rb], jct=False)
        close("replay", timed)
        mark("gather", timed)
        full = D.gather_summaries(summ, R, world, out=gathered)  # A-9: one NCCL all-gather
        close("gather", timed)
        cells = ct.ct_jct_stats(ctx, full, sw.n_cells)
        return cells, full

    for _ in range(args.warmup):
        step(False)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.3)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        cells, full = step(True)
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = clk.stop()
    t = e0.elapsed_time(e1) / 1e3

    def mean_ms(key):
        return sum(a.elapsed_time(b) for a, b in ev[key]) / len(ev[key])

    per_rank = torch.tensor([t, mean_ms("replay"), mean_ms("fit"), mean_ms("gather")],
                            dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(per_rank, op=dist.ReduceOp.MAX)
    t, k_ms, fit_ms, gather_ms = (float(x) for x in per_rank)
    k_t = k_ms / 1e3
    cells_np = cells.cpu().numpy()
    turns_step = int(cells_np[:, 3].sum())
    n_bad = int(cells_np[:, 1].sum())
    value = turns_step * args.steps / t
    launch = ctx.last_launch()
    full_np = full.cpu().numpy() if rank == 0 else None
    replay_launches = int(launch["launches"])  # the trace check + the replay kernel(s)

    # ---- e2e: host buffers through the C ABI, copies inside the timed region -------------------
    e2e = None
    if not args.no_e2e:
        h_prog = torch.from_numpy(np.ascontiguousarray(tr.programs).view(np.uint8)).pin_memory()
        h_turn = torch.from_numpy(np.ascontiguousarray(tr.turns)).pin_memory()
        h_dur = torch.from_numpy(dur_np).pin_memory()
        h_out = torch.empty((re_ - rb, 16), dtype=torch.int64).pin_memory()
        h_tab = torch.empty((F + 1, J), dtype=torch.int64).pin_memory()

        def e2e_step():
            d = h_dur.to(dev, non_blocking=True)
            arg, _, _ = ct.ct_fit_ttl(ctx, d, off, cp, sw.estimator, want_stats=False)
            h_tab.copy_(arg, non_blocking=True)
            if fitted_policy:
                sw.fitted = arg[:F]
            ct.ct_simulate_batch_host(ctx, tr, sw, eng, rb, re_, out=h_out, programs=h_prog,
                                      turns=h_turn)

        e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(args.steps):
            e2e_step()
        b.record(stream)
        torch.cuda.synchronize()
        te = torch.tensor([a.elapsed_time(b) / 1e3], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": turns_step * args.steps / float(te[0]), "unit": UNIT,
               "h2d_bytes_per_step": int(h_prog.numel() + 4 * h_turn.numel() + 4 * h_dur.numel()),
               "d2h_bytes_per_step": int(8 * h_out.numel() + 8 * h_tab.numel()),
               "api": "ct_fit_ttl + ct_simulate_batch_host (pinned host buffers)"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # ---- rooflines --------------------------------------------------------------------------------
    ipt = consts.get("replay_warp_inst_per_turn", {}).get(w.name) if consts else None
    clk_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    alu_peak = SM_COUNT * ISSUE_PER_SM_CLK * clk_mhz * 1e6 / 1e12  # T warp-inst/s
    turns_shard = turns_step * (re_ - rb) / R
    achieved = (ipt * turns_shard / k_t / 1e12) if ipt else None
    dram_pt = consts.get("replay_dram_bytes_per_turn", {}).get(w.name) if consts else None
    roofline = {"bound": "alu", "kernel": "replay_kernel", "unit": "Twarp-inst/s",
                "achieved": achieved, "peak": alu_peak,
                "frac": (achieved / alu_peak) if achieved else None,
                "traffic": dram_pt * turns_shard if dram_pt is not None else None,
                "warp_inst_per_replica_turn": ipt,
                "peak_basis": "148 SMs x 4 schedulers x 1 warp-inst/clk x %.0f MHz (max clock)" % clk_mhz,
                "achieved_basis": "ncu warp-inst per replica-turn (profiles/ncu_constants.json) x "
                                  "replica-turns per launch / CUDA-event launch time",
                "traffic_basis": "ncu dram bytes per replica-turn of a full-size capture "
                                 "(profiles/ncu_constants.json) x replica-turns per launch",
                "ms_per_launch": k_t * 1e3, "share_of_step": k_t / (t / args.steps),
                "replica_turns_per_s_kernel": turns_shard / k_t}
    rf = None
    if not args.no_fit_bandwidth:
        rf = fit_bandwidth(ctx, ct, cf, args.fit_log2n, dev, peaks, consts)
        rf["peak_kind"] = peak_kind
    cb = cbf = None
    if world == 1 and not args.no_cpu_baseline:
        osw = oracle_fitted(w, dur_np, off, fc, ctxj, wj)
        cb = cpu_baseline(w, osw, args.cpu_seconds, os.cpu_count() or 1, gpu_summ=full_np)
        cb.pop("est_turns_per_step")
        cb.pop("wall_s")
        cbf = cpu_fit_baseline(dur_np, off, fc, ctxj, wj, sw.estimator)

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t / args.steps * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": {"workload": w.name, "description": w.description, "replicas": R,
                       "programs_per_replica": tr.n_programs, "replica_turns_per_step": turns_step,
                       "non_ok_replicas": n_bad, "trace_bytes": dt.bytes,
                       "fit_samples_per_step": int(len(dur_np)),
                       "l2": "flushed every step (256 MiB write)",
                       "parallelism": ("replicas sharded (contiguous), fit sharded per tool "
                                       "segment + int64 all-reduce, all_gather of summaries")
                       if world > 1 else "1 GPU"},
            "roofline": roofline, "roofline_fit": rf, "cpu_baseline": cb, "cpu_baseline_fit": cbf,
            "e2e": e2e,
            # per step: the fit (1 fused launch, or partial + finish), the trace check + replay
            # kernel(s), jct_stats
            "gpu_launches": (fit_launches[0] + replay_launches + 1) * args.steps,
            "launch": launch,
            "per_step_ms_max_over_ranks": {"fit": fit_ms, "replay": k_ms, "gather": gather_ms},
            "clocks": clocks,
            "peaks": peak_kind}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
