#!/usr/bin/env python
"""B200 version of the paper's fig:kernel_speed: the
chunkwise-parallel forward (tcgen05 kernel) against the recurrent-form
forward (deltanet_recurrent_fwd), d_model = 2048 with d_head = 128 (H = 16),
batch x L = 16384 tokens, L = 512 ... 16384.  The paper's numbers (Triton,
GPU not stated for this figure) are printed beside ours.

    python tools/kernel_speed.py [--out profiles/r01_kernel_speed.json]
"""
import json
import sys

import os
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2406_06484_b200 as dn

# P:219-224 (d_head = 128): recurrent / chunkwise, unit not stated (ms)
PAPER = {512: (18.8856, 2.6611), 1024: (19.6152, 2.6409), 2048: (19.0975, 2.6484),
         4096: (31.2284, 2.9655), 8192: (60.9088, 3.8531), 16384: (191.4909, 5.8325)}


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    out = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else None
    H, D, T = 16, 128, 16384
    g = torch.Generator(device="cuda").manual_seed(0)
    rows = []
    for L in sorted(PAPER):
        B = T // L
        mk = lambda *s: torch.randn(*s, device="cuda", generator=g).to(torch.bfloat16)
        q, k, v = mk(B, H, L, D), mk(B, H, L, D), mk(B, H, L, D)
        beta = torch.rand(B, H, L, device="cuda", generator=g).to(torch.bfloat16)
        o = torch.empty_like(v)
        d = dn.make_desc(B, H, L, D, D, 64, torch.bfloat16, save_states=False)
        ws = dn.alloc_workspace(d, q.device)
        t_c = timed(lambda: dn.deltanet_fwd(q, k, v, beta, chunk=64, save_states=False,
                                            workspace=ws, want_hT=False, out=o))
        t_r = timed(lambda: dn.deltanet_recurrent_fwd(q, k, v, beta, want_hT=False, out=o))
        d1 = dn.make_desc(B, H, L, D, D, 64, torch.bfloat16, save_states=False, segments=False)
        ws1 = dn.alloc_workspace(d1, q.device)
        t_1 = timed(lambda: dn.deltanet_fwd(q, k, v, beta, chunk=64, save_states=False,
                                            workspace=ws1, want_hT=False, out=o,
                                            segments=False))
        pr, pc = PAPER[L]
        nseg_launches = dn.deltanet_launch_count(d, 0)
        rows.append({"L": L, "B": B, "recurrent_ms": t_r, "chunkwise_ms": t_c,
                     "chunkwise_one_cta_per_unit_ms": t_1, "segmented": nseg_launches == 3,
                     "speedup": t_r / t_c, "paper_recurrent": pr, "paper_chunkwise": pc,
                     "paper_speedup": pr / pc})
        print(f"L={L:6d} B={B:3d}  recurrent {t_r:8.3f} ms  chunkwise {t_c:7.3f} ms "
              f"(1 CTA/unit {t_1:7.3f} ms)  speed-up {t_r / t_c:6.2f}x   "
              f"(paper: {pr:.3f} / {pc:.3f} = {pr / pc:.2f}x)")
    if out:
        json.dump({"what": "fig:kernel_speed on B200, d_head=128, B*L=16384, forward, bf16",
                   "rows": rows}, open(out, "w"), indent=1)


if __name__ == "__main__":
    main()
