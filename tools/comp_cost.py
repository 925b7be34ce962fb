"""Cost of DELTANET_COMPENSATED (R19) at the bench workload
(B=8 H=16 L=4096 d=128): fwd / bwd medians with and without the flag."""
import sys

import torch

sys.path.insert(0, '.')
import paper_2406_06484_b200 as dn  # noqa: E402


def run(flags, reps=30):
    B, H, L, D = 8, 16, 4096, 128
    g = torch.Generator(device='cuda').manual_seed(0)
    f = torch.nn.functional
    mk = lambda: torch.randn((B, H, L, D), device='cuda', generator=g)
    q, k = f.silu(mk()).bfloat16(), f.silu(mk()).bfloat16()
    v, dO = mk().bfloat16(), mk().bfloat16()
    b = torch.sigmoid(torch.randn((B, H, L), device='cuda', generator=g)).bfloat16()
    o, hT, ws = dn.deltanet_fwd(q, k, v, b, extra_flags=flags)
    dn.deltanet_bwd(q, k, v, b, dO, workspace=ws, extra_flags=flags)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    tf, tb = [], []
    for _ in range(reps):
        ev[0].record()
        dn.deltanet_fwd(q, k, v, b, workspace=ws, extra_flags=flags)
        ev[1].record()
        dn.deltanet_bwd(q, k, v, b, dO, workspace=ws, extra_flags=flags)
        ev[2].record()
        torch.cuda.synchronize()
        tf.append(ev[0].elapsed_time(ev[1]))
        tb.append(ev[1].elapsed_time(ev[2]))
    med = lambda x: sorted(x)[len(x) // 2]
    return med(tf), med(tb)


if __name__ == "__main__":
    f0, b0 = run(0)
    f1, b1 = run(dn.DELTANET_COMPENSATED)
    print(f"default      fwd {f0:.4f} ms  bwd {b0:.4f} ms  step {f0 + b0:.4f} ms")
    print(f"compensated  fwd {f1:.4f} ms  bwd {b1:.4f} ms  step {f1 + b1:.4f} ms  "
          f"(+{100 * ((f1 + b1) / (f0 + b0) - 1):.1f}% of the step)")
