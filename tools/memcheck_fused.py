"""compute-sanitizer memcheck driver for the fused tcgen05 kernels on small
shapes (plain, ragged, segmented, gated, compensated).  Profiling aid."""
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import synth  # noqa: E402
from parity import TOL, compare, run_gpu, run_oracle  # noqa: E402

import paper_2406_06484_b200 as dn  # noqa: E402

for B, H, L, extra in ((1, 2, 150, 0), (1, 1, 64 * 41 + 1, 0), (1, 2, 200, dn.DELTANET_COMPENSATED)):
    cfg = synth.custom_config(B, H, L, 128, 128, 64, "bf16", index=991 + L % 7)
    inp = synth.make_inputs(cfg)
    got = run_gpu(inp, "bf16", 64, extra_flags=extra)
    print(B, H, L, extra, compare(got, run_oracle(inp), TOL["bf16"]))
# gated
cfg = synth.custom_config(1, 2, 137, 128, 128, 64, "bf16", index=995)
inp = synth.make_inputs(cfg)
g = synth.make_gates(cfg, 1.0)
dev = lambda x, dt: torch.from_numpy(np.ascontiguousarray(x)).to(dt).cuda()
q, k, v, b, dO = (dev(inp[f], torch.bfloat16) for f in ("q", "k", "v", "beta", "dO"))
o, hT, ws = dn.deltanet_gated_fwd(q, k, v, b, dev(g, torch.float32))
r = dn.deltanet_gated_bwd(q, k, v, b, dev(g, torch.float32), dO, workspace=ws)
torch.cuda.synchronize()
print("gated ok")
