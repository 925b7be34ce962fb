import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import test_gpu_gated as T
from parity import normwise
worst = {}
for scale in (0.05, 1.0, 4.0):
    for idx in range(6):
        inp = T._case(2, 2, 1000, 128, 128, 64, "bf16", index=1200 + idx, scale=scale)
        rng = np.random.default_rng(idx)
        h0 = 0.3 * rng.standard_normal((2, 2, 128, 128)); dhT = 0.3 * rng.standard_normal((2, 2, 128, 128))
        got = T._gpu(inp, "bf16", 64, h0=h0, dhT=dhT); ref = T._ref(inp, h0=h0, dhT=dhT)
        e = {k: normwise(got[k], ref[k]) for k in ref}
        print(scale, idx, {k: f"{v:.2e}" for k, v in e.items()}, flush=True)
