#!/usr/bin/env python
"""A/B timing of the layer prologue (fwd, bwd) across library builds (profiling aid).

    python tools/prologue_ab.py LIB_A.so LIB_B.so [...] [--rounds 3]
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(lib):
    sys.path.insert(0, ROOT)
    import torch
    import paper_2406_06484_b200 as dn
    dn.load_library(lib)
    B, H, L, D = 8, 16, 4096, 128
    g = torch.Generator(device="cuda").manual_seed(0)
    mk = lambda *s: torch.randn(s, device="cuda", generator=g)
    xq, xk, xv = (mk(B, L, H, D).bfloat16() for _ in range(3))
    xb = mk(B, L, H).bfloat16()
    wq, wk, wv = (mk(H * D, 4) * 0.5 for _ in range(3))
    q, k, v, b = dn.deltanet_prologue_fwd(xq, xk, xv, xb, wq, wk, wv)
    dq, dk, dv, db = (torch.randn_like(t) for t in (q, k, v, b))
    dn.deltanet_prologue_bwd(xq, xk, xv, xb, wq, wk, wv, dq, dk, dv, db)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    tf, tb = [], []
    for i in range(25):
        ev[0].record()
        dn.deltanet_prologue_fwd(xq, xk, xv, xb, wq, wk, wv)
        ev[1].record()
        dn.deltanet_prologue_bwd(xq, xk, xv, xb, wq, wk, wv, dq, dk, dv, db)
        ev[2].record()
        torch.cuda.synchronize()
        if i >= 5:
            tf.append(ev[0].elapsed_time(ev[1]))
            tb.append(ev[1].elapsed_time(ev[2]))
    med = lambda x: sorted(x)[len(x) // 2]
    print(json.dumps({"fwd": med(tf), "bwd": med(tb)}))


if __name__ == "__main__":
    if sys.argv[1] == "--child":
        child(sys.argv[2])
        sys.exit(0)
    libs = [a for a in sys.argv[1:] if a.endswith(".so")]
    for _ in range(2):
        for l in libs:
            out = subprocess.run([sys.executable, __file__, "--child", os.path.abspath(l)],
                                 capture_output=True, text=True)
            line = [x for x in out.stdout.splitlines() if x.startswith("{")]
            print(os.path.basename(l), line[-1] if line else out.stderr[-1500:])
