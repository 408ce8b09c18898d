"""Full-size oracle digests for every-replica GPU parity (TEST INFRASTRUCTURE).

Imports only oracle/ and ctgen/ (the seeded input generators).  For each BASELINE config it
replays EVERY replica with the CPU oracle (all host cores) and records SHA-256 digests of the
summary bytes and the per-program JCT bytes, per block of replicas and for the whole sweep,
plus the per-cell statistics (or_jct_stats) and the trace digest the inputs came from.
tests/test_gpu_fullsize.py runs the same sweeps through ct_simulate_batch and compares the
digests block by block, so a mismatch is localised to a block and then to a replica.

    python tools/oracle_digests.py [cfg2 cfg4 cfg5 cfg3] [--threads N]

Progress is checkpointed per block under build/digests_partial/ (a killed run resumes).
The result is merged into tests/golden/fullsize_digests.json.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from ctgen import configs as cf  # noqa: E402
from ctgen import traces  # noqa: E402
from oracle import oracle as O  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "fullsize_digests.json")
PART = os.path.join(ROOT, "build", "digests_partial")

def workload(name):
    w = {"cfg2": cf.config2, "cfg3": cf.config3, "cfg4": cf.config4, "cfg5": cf.config5}[name]()
    extra = {}
    if name == "cfg4":
        dur, off = traces.tool_samples(w.trace)
        p = cf.CFG4_FIT
        arg, _, _ = O.fit(dur, off, cf.cfg4_fit_cost(w.engine), p["ctx_j"], p["w_j"],
                          w.sweep.estimator.as_array())
        w.sweep.fitted = arg[:-1]
        extra["fitted_sha256"] = hashlib.sha256(np.ascontiguousarray(arg).tobytes()).hexdigest()
    return w, extra


BLOCK = {"cfg2": 64, "cfg3": 4096, "cfg4": 512, "cfg5": 4096}


def h16(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()[:16]


def run(name, threads):
    t0 = time.time()
    w, extra = workload(name)
    R, B, P = w.sweep.n_replicas, BLOCK[name], w.trace.n_programs
    assert R % B == 0
    os.makedirs(PART, exist_ok=True)
    part = os.path.join(PART, "%s_%s.npz" % (name, w.trace.digest()))
    summ = np.zeros((R, 16), np.int64)
    bs_h, bj_h = [None] * (R // B), [None] * (R // B)
    done = 0
    if os.path.exists(part):
        z = np.load(part, allow_pickle=True)
        done = int(z["done"])
        summ[:done * B] = z["summ"][:done * B]
        bj_h[:done] = list(z["bj"][:done])
        print("%s: resuming at block %d/%d" % (name, done, R // B), flush=True)
    for b in range(done, R // B):
        s, j = O.simulate(w.trace, w.sweep, w.engine, b * B, (b + 1) * B, n_threads=threads)
        summ[b * B:(b + 1) * B] = s
        bj_h[b] = h16(np.ascontiguousarray(j).tobytes())
        if (b + 1) % 8 == 0 or b + 1 == R // B:
            np.savez(part + ".tmp.npz", done=b + 1, summ=summ[:(b + 1) * B], bj=np.array(bj_h[:b + 1]))
            os.replace(part + ".tmp.npz", part)
            el = time.time() - t0
            print("%s: block %d/%d  %.0f s" % (name, b + 1, R // B, el), flush=True)
    for b in range(R // B):
        bs_h[b] = h16(summ[b * B:(b + 1) * B].tobytes())
    st = summ[:, 0] & 0xFFFFFFFF
    n_cells = w.sweep.n_cells
    cells = O.jct_stats(summ, n_cells)
    rec = {"workload": w.name, "trace_digest": w.trace.digest(), "replicas": R, "programs": P,
           "block": B, "summary_sha256": hashlib.sha256(summ.tobytes()).hexdigest(),
           "block_summary": bs_h, "block_jct": bj_h,
           "cells_sha256": hashlib.sha256(cells.tobytes()).hexdigest(),
           "replica_turns": int(summ[st == 0, 1].sum()),
           "status_counts": {str(k): int((st == k).sum()) for k in np.unique(st)},
           "oracle_wall_s": round(time.time() - t0, 1), "oracle_threads": threads, **extra}
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["cfg2", "cfg4", "cfg5", "cfg3"])
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    a = ap.parse_args()
    for name in a.configs:
        rec = run(name, a.threads)
        cur = json.load(open(OUT)) if os.path.exists(OUT) else {}
        cur["_about"] = ("SHA-256 digests of the CPU oracle's summaries / per-program JCTs on "
                         "every replica of BASELINE configs 2-5, written by "
                         "tools/oracle_digests.py (oracle/ + ctgen/ only); block_* are the "
                         "first 16 hex digits of each block's digest")
        cur["oracle_src_sha256"] = hashlib.sha256(
            open(os.path.join(ROOT, "oracle", "ct_oracle.cpp"), "rb").read()).hexdigest()
        cur[name] = rec
        json.dump(cur, open(OUT, "w"), indent=1)
        print("%s: done, %d replicas, %s" % (name, rec["replicas"], rec["status_counts"]), flush=True)


if __name__ == "__main__":
    main()
