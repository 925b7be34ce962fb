#!/usr/bin/env python
"""B200 version of the paper's fig:kernel_speed: the
chunkwise-parallel forward (tcgen05 kernels: fused at d_head = 128, split at
64 and 256) against the recurrent-form forward (deltanet_recurrent_fwd),
d_model = 2048 (H = 2048 / d_head), batch x L = 16384 tokens, L = 512 ...
16384.  The paper's numbers (Triton, GPU not stated for this figure;
BASELINE.md §1) are printed beside ours.

    python tools/kernel_speed.py [--out profiles/r02_kernel_speed.json]
"""
import json
import sys

import os
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2406_06484_b200 as dn

# recurrent / chunkwise per head dim, unit not stated (ms)
PAPER = {
    64: {512: (10.7097, 2.6930), 1024: (10.9562, 2.4330), 2048: (14.0425, 2.4151),
         4096: (24.4682, 2.5787), 8192: (47.6885, 3.0478), 16384: (94.9672, 4.0006)},
    128: {512: (18.8856, 2.6611), 1024: (19.6152, 2.6409), 2048: (19.0975, 2.6484),
          4096: (31.2284, 2.9655), 8192: (60.9088, 3.8531), 16384: (191.4909, 5.8325)},
    256: {512: (47.2460, 4.6427), 1024: (47.4189, 4.6667), 2048: (47.8577, 4.6824),
          4096: (83.5260, 4.7730), 8192: (166.8563, 5.8201), 16384: (330.6606, 9.0348)},
}


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
    T = 16384
    g = torch.Generator(device="cuda").manual_seed(0)
    rows = []
    for D in (64, 128, 256):
        H = 2048 // D
        for L in sorted(PAPER[D]):
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
            pr, pc = PAPER[D][L]
            rows.append({"d_head": D, "H": H, "L": L, "B": B, "recurrent_ms": t_r,
                         "chunkwise_ms": t_c,
                         "chunkwise_path": {1: "tcgen05 fused", 2: "tcgen05 split"}.get(
                             dn.deltanet_path(d), "simt"),
                         "chunkwise_launches": dn.deltanet_launch_count(d, 0),
                         "speedup": t_r / t_c, "paper_recurrent": pr, "paper_chunkwise": pc,
                         "paper_speedup": pr / pc})
            print(f"d={D:3d} H={H:2d} L={L:6d} B={B:3d}  recurrent {t_r:8.3f} ms  "
                  f"chunkwise {t_c:7.3f} ms  speed-up {t_r / t_c:6.2f}x   "
                  f"(paper: {pr:.3f} / {pc:.3f} = {pr / pc:.2f}x)", flush=True)
            del q, k, v, beta, o, ws
    if out:
        json.dump({"what": "fig:kernel_speed on B200, d_model=2048, B*L=16384, forward, bf16",
                   "rows": rows}, open(out, "w"), indent=1)


if __name__ == "__main__":
    main()
