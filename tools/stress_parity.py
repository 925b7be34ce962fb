#!/usr/bin/env python
"""Race / regression stress for the tcgen05 kernels (profiling aid, not a
test): random shapes on the bf16 d=128 path (ungated and gated) against the
fp64 oracle, and bitwise run-to-run determinism at the BASELINE target shape."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import oracle  # noqa: E402
import paper_2406_06484_b200 as dn  # noqa: E402
import synth  # noqa: E402
from parity import TOL, compare, run_gpu, run_oracle, to_dev  # noqa: E402


def main(n=12, seed=7):
    rng = np.random.default_rng(seed)
    worst = {}
    for it in range(n):
        B, H = int(rng.integers(1, 3)), int(rng.integers(1, 4))
        L = int(rng.integers(1, 2500))
        cfg = synth.custom_config(B, H, L, 128, 128, 64, "bf16", index=2000 + it)
        inp = synth.make_inputs(cfg)
        errs = compare(run_gpu(inp, "bf16", 64), run_oracle(inp), TOL["bf16"])
        worst = {k: max(worst.get(k, 0), v) for k, v in errs.items()}
        g = synth.make_gates(cfg, float(rng.choice([0.05, 1.0, 4.0])))
        td = torch.bfloat16
        q, k, v, b, dO = (to_dev(inp[f], td) for f in ("q", "k", "v", "beta", "dO"))
        gd = to_dev(g, torch.float32)
        o, hT, ws = dn.deltanet_gated_fwd(q, k, v, b, gd)
        grads = dn.deltanet_gated_bwd(q, k, v, b, gd, dO, workspace=ws)
        torch.cuda.synchronize()
        f = lambda t: t.float().cpu().numpy().astype(np.float64)
        ro, rhT = oracle.gated_fwd(inp["q"], inp["k"], inp["v"], inp["beta"], g)
        rg = oracle.gated_bwd(inp["q"], inp["k"], inp["v"], inp["beta"], g, inp["dO"])
        keys = ("dq", "dk", "dv", "dbeta", "dg", "dh0")
        ge = compare({"o": f(o), **{kk: f(t) for kk, t in zip(keys, grads)}},
                     {"o": ro, **dict(zip(keys, rg))}, TOL["bf16"])
        for a_, e_ in ge.items():
            worst["g_" + a_] = max(worst.get("g_" + a_, 0.0), e_)
        print(it, B, H, L, "ok", flush=True)
    print("worst", {k: f"{v:.2e}" for k, v in worst.items()})
    # determinism at the target shape (any race shows up as a bitwise difference)
    cfg = synth.CONFIGS["target"]
    inp = synth.make_inputs(cfg)
    outs = [run_gpu(inp, "bf16", 64) for _ in range(3)]
    for key in outs[0]:
        if outs[0][key] is None:
            continue
        for o2 in outs[1:]:
            assert np.array_equal(outs[0][key], o2[key]), f"non-deterministic {key}"
    print("deterministic over 3 runs at the target shape")
    # and at the long-context shape (segmented forward with prep records)
    cfg = synth.CONFIGS["long"]
    inp = synth.make_inputs(cfg)
    outs = [run_gpu(inp, "bf16", 64) for _ in range(2)]
    for key in outs[0]:
        if outs[0][key] is not None:
            assert np.array_equal(outs[0][key], outs[1][key]), f"non-deterministic {key} (long)"
    print("deterministic over 2 runs at the long-context shape")


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 12)
