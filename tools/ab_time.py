#!/usr/bin/env python
"""A/B timing of library builds on the same GPU (profiling aid).

    python tools/ab_time.py LIB_A.so LIB_B.so [...] [--rounds 3] [--shape B,H,L]

Each library is timed in its own subprocess (ctypes can hold one
libdeltanet per process), alternating A, B, A, B ... so clock and thermal
drift hit every build alike; prints the median fwd / bwd / step per build
(CUDA events on the launching stream, 30 steps after 5 warm-up steps).
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(lib, B, H, L, gated=False):
    sys.path.insert(0, ROOT)
    import torch
    import paper_2406_06484_b200 as dn
    dn.load_library(lib)
    g = torch.Generator(device="cuda").manual_seed(0)
    mk = lambda: torch.randn((B, H, L, 128), device="cuda", generator=g)
    f = torch.nn.functional
    q, k = f.silu(mk()).bfloat16(), f.silu(mk()).bfloat16()
    v, dO = mk().bfloat16(), mk().bfloat16()
    b = torch.sigmoid(torch.randn((B, H, L), device="cuda", generator=g)).bfloat16()
    gt = -0.05 * f.softplus(torch.randn((B, H, L), device="cuda", generator=g))
    if gated:
        fwd = lambda ws=None: dn.deltanet_gated_fwd(q, k, v, b, gt, workspace=ws)
        bwd = lambda ws: dn.deltanet_gated_bwd(q, k, v, b, gt, dO, workspace=ws)
    else:
        fwd = lambda ws=None: dn.deltanet_fwd(q, k, v, b, workspace=ws)
        bwd = lambda ws: dn.deltanet_bwd(q, k, v, b, dO, workspace=ws)
    o, hT, ws = fwd()
    bwd(ws)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    tf, tb = [], []
    for i in range(35):
        ev[0].record()
        o, hT, ws = fwd(ws)
        ev[1].record()
        bwd(ws)
        ev[2].record()
        torch.cuda.synchronize()
        if i >= 5:
            tf.append(ev[0].elapsed_time(ev[1]))
            tb.append(ev[1].elapsed_time(ev[2]))
    med = lambda x: sorted(x)[len(x) // 2]
    print(json.dumps({"fwd": med(tf), "bwd": med(tb)}))


def main():
    args = sys.argv[1:]
    if args and args[0] == "--child":
        B, H, L = (int(x) for x in args[2].split(","))
        return child(args[1], B, H, L, len(args) > 3 and args[3] == "gated")
    rounds, shape, libs, mode = 3, "8,16,4096", [], []
    it = iter(args)
    for a in it:
        if a == "--rounds":
            rounds = int(next(it))
        elif a == "--shape":
            shape = next(it)
        elif a == "--gated":
            mode = ["gated"]
        else:
            libs.append(os.path.abspath(a))
    res = {l: [] for l in libs}
    for _ in range(rounds):
        for l in libs:
            out = subprocess.run([sys.executable, __file__, "--child", l, shape] + mode,
                                 capture_output=True, text=True)
            line = [x for x in out.stdout.splitlines() if x.startswith("{")]
            if not line:
                print(l, "FAILED", out.stderr[-2000:])
                continue
            res[l].append(json.loads(line[-1]))
    for l, rs in res.items():
        if not rs:
            continue
        f = sorted(r["fwd"] for r in rs)[len(rs) // 2]
        b = sorted(r["bwd"] for r in rs)[len(rs) // 2]
        print(f"{os.path.basename(l):28s} fwd {f:.4f} bwd {b:.4f} step {f + b:.4f}  "
              f"(fwd {[round(r['fwd'], 4) for r in rs]}, bwd {[round(r['bwd'], 4) for r in rs]})")


if __name__ == "__main__":
    main()
