"""Throughput of on-device trace synthesis (NEXT-4) vs host generation + copy."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2511_02230_b200 as ct
from ctgen import synth

S = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
P = 32
ctx = ct.Context(0)
sp = synth.params(ctx_cap=8192 * 16, n_bfcl=16)
cap = S * P * 20
for _ in range(2):
    ct.ct_synthesize_traces(ctx, sp, 0, S, P, turns_cap=cap)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
g = ct.ct_synthesize_traces(ctx, sp, 0, S, P, turns_cap=cap)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
nt = g.turns.shape[0]
t = time.time()
ref = synth.synthesize(sp, 0, min(S, 4096), P)
host_s = (time.time() - t) * S / min(S, 4096)
print("device: %d seeds x %d programs, %d turn records (%.1f MB) in %.2f ms = %.2e turns/s; "
      "host numpy (extrapolated from 4096 seeds) %.2f s" % (S, P, nt, nt * 16 / 1e6, ms, nt / ms * 1e3, host_s))
