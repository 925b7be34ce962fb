"""Shared helpers of the GPU parity tests: run the CUDA path through the
C ABI and the fp64 oracle on the SAME seeded inputs, compare normwise.

Tolerance (R16, BASELINE.json north_star): per output tensor,
err(x) = max|x - ref| / max|ref|; bar 1e-4 for fp32 I/O, 2e-2 for bf16 I/O.
"""
from __future__ import annotations

import os

import numpy as np
import torch

import oracle
import synth

TOL = {"fp32": 1e-4, "bf16": 2e-2}


def normwise(x, ref):
    x = np.asarray(x, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    den = np.abs(ref).max()
    num = np.abs(x - ref).max()
    if den == 0:
        return float(num)
    return float(num / den)


def torch_dtype(name):
    return {"bf16": torch.bfloat16, "fp32": torch.float32}[name]


def to_dev(a, dtype, dev="cuda"):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev).to(dtype).contiguous()


def run_gpu(inp, dtype, chunk, l2norm=True, h0=None, dhT=None, force_simt=False,
            save_states=True, segments=True, force_split=False, extra_flags=0):
    import paper_2406_06484_b200 as dn
    td = torch_dtype(dtype)
    q, k, v, b, dO = (to_dev(inp[f], td) for f in ("q", "k", "v", "beta", "dO"))
    h0t = None if h0 is None else to_dev(h0, torch.float32)
    dhTt = None if dhT is None else to_dev(dhT, torch.float32)
    o, hT, ws = dn.deltanet_fwd(q, k, v, b, chunk=chunk, l2norm=l2norm, h0=h0t,
                                save_states=save_states, force_simt=force_simt,
                                segments=segments, force_split=force_split,
                                extra_flags=extra_flags)
    g = dn.deltanet_bwd(q, k, v, b, dO, chunk=chunk, l2norm=l2norm, h0=h0t, dhT=dhTt,
                        workspace=ws if save_states else None,
                        states_saved=save_states, force_simt=force_simt,
                        segments=segments, force_split=force_split,
                        extra_flags=extra_flags)
    torch.cuda.synchronize()
    f = lambda t: None if t is None else t.float().cpu().numpy().astype(np.float64)
    return {"o": f(o), "hT": f(hT), "dq": f(g[0]), "dk": f(g[1]), "dv": f(g[2]),
            "dbeta": f(g[3]), "dh0": f(g[4])}


def run_oracle(inp, l2norm=True, h0=None, dhT=None):
    o, hT = oracle.recurrent_fwd(inp["q"], inp["k"], inp["v"], inp["beta"], h0=h0,
                                 l2norm=l2norm)
    dq, dk, dv, db, dh0 = oracle.recurrent_bwd(inp["q"], inp["k"], inp["v"], inp["beta"],
                                               inp["dO"], h0=h0, dhT=dhT, l2norm=l2norm)
    return {"o": o, "hT": hT, "dq": dq, "dk": dk, "dv": dv, "dbeta": db, "dh0": dh0}


def compare(got, ref, tol, keys=None):
    errs = {}
    for key in keys or ref.keys():
        if got.get(key) is None or ref.get(key) is None:
            continue
        assert got[key].shape == ref[key].shape, (key, got[key].shape, ref[key].shape)
        assert np.isfinite(got[key]).all(), f"{key} has non-finite values"
        errs[key] = normwise(got[key], ref[key])
    if os.environ.get("PARITY_VERBOSE") == "1":
        print("\n  normwise:", {k: f"{e:.2e}" for k, e in errs.items()}, f"(bar {tol})")
    bad = {k: e for k, e in errs.items() if not e <= tol}
    assert not bad, f"normwise errors above {tol}: {bad} (all: {errs})"
    return errs


def row_guard(got, ref, key, tol, rows=64):
    """Localised errors in low-magnitude stretches of a per-token output
    (dbeta, dg) are invisible in the tensor-max metric.  Per unit and per
    window of `rows` tokens: max|x - ref| / max(|ref| over the window, the
    unit's RMS) <= tol.  (The RMS floor keeps windows whose reference is
    accidentally ~0 from dividing by ~0.)"""
    x = np.asarray(got[key], np.float64)
    r = np.asarray(ref[key], np.float64)
    L = r.shape[-1]
    rms = np.sqrt((r ** 2).mean(axis=-1, keepdims=True))
    worst = 0.0
    for t0 in range(0, L, rows):
        xs, rs = x[..., t0:t0 + rows], r[..., t0:t0 + rows]
        den = np.maximum(np.abs(rs).max(axis=-1), rms[..., 0])
        worst = max(worst, float((np.abs(xs - rs).max(axis=-1) / den).max()))
    assert worst <= tol, f"{key}: per-window normwise error {worst:.3g} > {tol}"
    return worst
