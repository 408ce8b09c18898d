for v in ${VARIANTS:-15 17 15 17}; do echo "variant $v"; CT_FIT_VARIANT=$v python - <<'PY'
import torch, numpy as np, sys
sys.path.insert(0, '.')
import paper_2511_02230_b200 as ct
from ctgen import configs as cf, traces
ctx = ct.Context(0); ctx.set_timing(True)
dur, off = traces.synthetic_samples_torch(28, 32, 1234, "cuda")
cp = ct.cost_params(13_400_000, 200, 16, 1, 10, 50_000, 256, [min(16 * 2**j, 120_000) for j in range(64)], list(range(1, 65)))
ms = []
for i in range(12):
    ct.ct_fit_ttl(ctx, dur, off, cp, cf.Estimator()); ms.append(ctx.last_launch()["fit_hist_ms"])
m = np.median(ms[2:]); print("fit_hist %.1f us %.0f GB/s (min %.1f)" % (m*1e3, 4*2**28/(m*1e-3)/1e9, min(ms)*1e3))
PY
done
CT_FIT_VARIANT=${PVAR:-12} python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k fit 2>&1 | tail -1
