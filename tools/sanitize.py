"""Small fit + replay + stats run for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2511_02230_b200 as ct
from ctgen import configs as cf, traces
ctx = ct.Context(0)
for P, mix in ((16, "mix"), (70, "mix")):
    tr = traces.generate(2, P, mix=mix, ctx_cap=8192, stream=P)
    fitted = np.tile(np.array([[0, 200_000, 3_000_000]], np.int64), (tr.n_tools, 1))
    eng = cf.Engine(**{**cf.ENGINE_8B.__dict__, "dram_blocks": 40 * P})
    pols = [cf.VLLM_LMCACHE, cf.CONTINUUM, cf.ttl_grid(500_000), cf.AUTELLIX, cf.INFERCEPT,
            cf.Policy(cf.PRIO_PROG_FCFS, cf.PAUSE_FITTED, flags=cf.FLAG_STEP_EXPIRY)]
    sw = cf.Sweep(2, [300_000], [600, 3000], pols, fitted=fitted)
    s, j = ct.ct_simulate_batch(ctx, ct.DeviceTrace(tr), sw, eng, jct=True)
    c = ct.ct_jct_stats(ctx, s, sw.n_cells)
# specialised kernels: TTL-grid class (32-bit times, with a horizon fallback at the long gap)
# and the program-FCFS class for P > 32
for P, pols in ((16, [cf.ttl_grid(0), cf.ttl_grid(2_000_000), cf.PROG_FCFS]),
                (70, [cf.CONTINUUM, cf.ttl_grid(500_000), cf.PROG_FCFS]),
                (70, [cf.VLLM, cf.CONTINUUM]), (16, [cf.VLLM, cf.CONTINUUM])):
    tr = traces.generate(2, P, mix="mix", ctx_cap=8192, stream=P + 1)
    sw = cf.Sweep(2, [300_000, (1 << 30) - 1], [3000], pols)
    s, j = ct.ct_simulate_batch(ctx, ct.DeviceTrace(tr), sw, cf.ENGINE_8B, jct=True)
# extended class (MODE 6: DRAM tier, PLAS, InferCept on 32-bit times) and an invalid trace set
tr = traces.generate(2, 16, mix="mix", ctx_cap=8192, stream=3)
eng = cf.Engine(**{**cf.ENGINE_8B.__dict__, "dram_blocks": 640})
sw = cf.Sweep(2, [300_000, (1 << 30) - 1], [600, 3000], [cf.VLLM_LMCACHE, cf.AUTELLIX, cf.INFERCEPT])
ct.ct_simulate_batch(ctx, ct.DeviceTrace(tr), sw, eng, jct=True)
bad = traces.TraceSet(tr.programs.copy(), tr.turns.copy(), tr.n_seeds, tr.n_programs, tr.n_tools, tr.pclass)
bad.turns[3, 2] = 99
ct.ct_simulate_batch(ctx, ct.DeviceTrace(bad), sw, eng, jct=True)
# fit: fused CSR launch, sharded partial + finish, unsorted pairs, invalid samples, estimator calls
dur, off = traces.tool_samples(tr)
cp = ct.cost_params(13_400_000, 200, 16, 1, 10, 50_000, 256, [2000, 8000], [1, 2])
d = torch.from_numpy(dur).cuda()
ct.ct_fit_ttl(ctx, d, off, cp, cf.Estimator())
acc = ct.ct_fit_ttl_partial(ctx, d, off, cp, cf.Estimator(), 1, 2)
ct.ct_fit_ttl_finish(ctx, acc, tr.n_tools, cp, cf.Estimator())
tool = torch.randint(0, tr.n_tools, (len(dur),), dtype=torch.uint8).cuda()
ct.ct_fit_ttl(ctx, d, None, cp, cf.Estimator(), tool_u8=tool, n_tools=tr.n_tools)
ct.ct_fit_ttl(ctx, -d, off, cp, cf.Estimator())
rows = torch.tensor([[3, 30, 300, 0], [1, 5, 25, 0]], dtype=torch.int64).cuda()
ct.ct_bernstein(ctx, rows, cf.Estimator())
nd = torch.tensor([1, 0], dtype=torch.int64).cuda()
ct.ct_calc_ttl_batch(ctx, rows, rows, nd, nd, cf.Estimator())
torch.cuda.synchronize()
print("sanitize run ok")
