import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_02230_b200._lib as L
L.LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libcontinuum_dbg.so")
import numpy as np, torch
import paper_2511_02230_b200 as ct
from ctgen import configs as cf
ctx = ct.Context(0)
w = cf.config3(n_seeds=4)
s, _ = ct.ct_simulate_batch(ctx, ct.DeviceTrace(w.trace), w.sweep, w.engine)
s = s.cpu().numpy()
turns = s[:, 1].sum()
print("loops/turn %.2f sched/turn %.2f macro/turn %.2f mid/turn %.2f" % (s[:, 15].sum() / turns, s[:, 14].sum() / turns, s[:, 12].sum() / turns, s[:, 11].sum() / turns))
