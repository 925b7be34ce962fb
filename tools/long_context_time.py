"""Segmented fwd+bwd at BASELINE configs[2] (B=2 H=16 L=16384 d=128), a few
steps (for an ncu launch list: per-pass kernel times), then the median of 20
event-timed steps."""
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

ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
tf, tb = [], []
for _ in range(20):
    ev[0].record()
    o, hT, ws = dn.deltanet_fwd(q, k, v, b, workspace=ws)
    ev[1].record()
    dn.deltanet_bwd(q, k, v, b, dO, workspace=ws)
    ev[2].record()
    torch.cuda.synchronize()
    tf.append(ev[0].elapsed_time(ev[1]))
    tb.append(ev[1].elapsed_time(ev[2]))
med = lambda x: sorted(x)[len(x) // 2]
print(f"B={B} H={H} L={L} d={D}: fwd {med(tf):.4f} ms, bwd {med(tb):.4f} ms, "
      f"step {med(tf) + med(tb):.4f} ms (median of 20, CUDA events)")
