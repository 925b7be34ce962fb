"""Segmented fwd+bwd at BASELINE configs[2] (B=2 H=16 L=16384 d=128), a few
steps, for an ncu launch list (per-pass kernel times)."""
import sys

import torch

sys.path.insert(0, '.')
import paper_2406_06484_b200 as dn  # noqa: E402

B, H, L, D = 2, 16, 16384, 128
g = torch.Generator(device='cuda').manual_seed(0)
f = torch.nn.functional
mk = lambda: torch.randn((B, H, L, D), device='cuda', generator=g)
q, k = f.silu(mk()).bfloat16(), f.silu(mk()).bfloat16()
v, dO = mk().bfloat16(), mk().bfloat16()
b = torch.sigmoid(torch.randn((B, H, L), device='cuda', generator=g)).bfloat16()
o, hT, ws = dn.deltanet_fwd(q, k, v, b)
for _ in range(3):
    o, hT, ws = dn.deltanet_fwd(q, k, v, b, workspace=ws)
    dn.deltanet_bwd(q, k, v, b, dO, workspace=ws)
torch.cuda.synchronize()
print("launches fwd/bwd:", dn.deltanet_launch_count(dn.make_desc(B, H, L, D, D), 0),
      dn.deltanet_launch_count(dn.make_desc(B, H, L, D, D), 1))
