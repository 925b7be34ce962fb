#!/usr/bin/env python
"""Segment-parallel forward/backward on few-unit, long
sequences: fwd, bwd and fwd+bwd step times with and without segments, for the
BASELINE long-context config (B=2 H=16 L=16384) and B*L = 16384 shapes.

    python tools/seq_parallel.py [--out profiles/r01_seq_parallel.json]
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_06484_b200 as dn  # noqa: E402


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
    H, D = 16, 128
    g = torch.Generator(device="cuda").manual_seed(0)
    rows = []
    for B, L in ((2, 16384), (1, 16384), (2, 8192), (4, 4096), (8, 4096)):
        mk = lambda *s: torch.randn(*s, device="cuda", generator=g).to(torch.bfloat16)
        q, k, v, dO = (mk(B, H, L, D) for _ in range(4))
        beta = torch.rand(B, H, L, device="cuda", generator=g).to(torch.bfloat16)
        o = torch.empty_like(v)
        grads = (torch.empty_like(q), torch.empty_like(k), torch.empty_like(v),
                 torch.empty_like(beta))
        res = {"B": B, "L": L, "units": B * H}
        for seg in (True, False):
            d = dn.make_desc(B, H, L, D, D, 64, torch.bfloat16, segments=seg)
            ws = dn.alloc_workspace(d, q.device)
            f = lambda: dn.deltanet_fwd(q, k, v, beta, workspace=ws, want_hT=False, out=o,
                                        segments=seg)
            bw = lambda: dn.deltanet_bwd(q, k, v, beta, dO, workspace=ws, want_dh0=False,
                                         out=grads, segments=seg)
            tf = timed(f)
            f()
            tb = timed(bw)
            key = "seg" if seg else "serial"
            res[key] = {"fwd_ms": tf, "bwd_ms": tb, "step_ms": tf + tb,
                        "tokens_per_s": B * L / ((tf + tb) * 1e-3),
                        "launches": dn.deltanet_launch_count(d, 0) + dn.deltanet_launch_count(d, 1)}
        rows.append(res)
        print(f"B={B} L={L:6d} units={B * H:4d}: segmented fwd {res['seg']['fwd_ms']:.3f} "
              f"bwd {res['seg']['bwd_ms']:.3f} ms | one CTA/unit fwd {res['serial']['fwd_ms']:.3f} "
              f"bwd {res['serial']['bwd_ms']:.3f} ms | step speed-up "
              f"{res['serial']['step_ms'] / res['seg']['step_ms']:.2f}x")
    if out:
        json.dump({"what": "segment-parallel vs one CTA per unit, bf16, d=128, C=64",
                   "rows": rows}, open(out, "w"), indent=1)


if __name__ == "__main__":
    main()
