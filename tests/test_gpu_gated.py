"""GPU parity of Gated DeltaNet (include/deltanet.h
deltanet_gated_fwd / _bwd / _recurrent_fwd; R23) against the fp64
oracle (oracle.gated_fwd / gated_bwd, pinned in tests/test_oracle_gated.py),
normwise (R16): 1e-4 for fp32 I/O, 2e-2 for bf16 I/O; dg is fp32
in both cases and held to the same bar as the other gradients."""
import numpy as np
import pytest
import torch

import oracle
import synth
from parity import TOL, compare, row_guard, to_dev, torch_dtype

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2406_06484_b200 import build
    build.build()


def _case(B, H, L, Dk, Dv, C, dtype, index, scale=0.05):
    cfg = synth.custom_config(B, H, L, Dk, Dv, C, dtype, index=index)
    inp = synth.make_inputs(cfg)
    inp["g"] = synth.make_gates(cfg, scale)
    return inp


def _np(t):
    return None if t is None else t.float().cpu().numpy().astype(np.float64)


def _gpu(inp, dtype, C, h0=None, dhT=None, l2norm=True, force_simt=False):
    import paper_2406_06484_b200 as dn
    td = torch_dtype(dtype)
    q, k, v, b, dO = (to_dev(inp[f], td) for f in ("q", "k", "v", "beta", "dO"))
    g = to_dev(inp["g"], torch.float32)
    h0t = None if h0 is None else to_dev(h0, torch.float32)
    dhTt = None if dhT is None else to_dev(dhT, torch.float32)
    o, hT, ws = dn.deltanet_gated_fwd(q, k, v, b, g, chunk=C, h0=h0t, l2norm=l2norm,
                                      force_simt=force_simt)
    dq, dk, dv, db, dg, dh0 = dn.deltanet_gated_bwd(q, k, v, b, g, dO, chunk=C, h0=h0t,
                                                    dhT=dhTt, workspace=ws, l2norm=l2norm,
                                                    force_simt=force_simt)
    torch.cuda.synchronize()
    return {"o": _np(o), "hT": _np(hT), "dq": _np(dq), "dk": _np(dk), "dv": _np(dv),
            "dbeta": _np(db), "dg": _np(dg), "dh0": _np(dh0)}


def _ref(inp, h0=None, dhT=None, l2norm=True):
    o, hT = oracle.gated_fwd(inp["q"], inp["k"], inp["v"], inp["beta"], inp["g"], h0=h0,
                             l2norm=l2norm)
    dq, dk, dv, db, dg, dh0 = oracle.gated_bwd(inp["q"], inp["k"], inp["v"], inp["beta"],
                                               inp["g"], inp["dO"], h0=h0, dhT=dhT,
                                               l2norm=l2norm)
    return {"o": o, "hT": hT, "dq": dq, "dk": dk, "dv": dv, "dbeta": db, "dg": dg, "dh0": dh0}


@pytest.mark.parametrize("Dk,Dv,C", [(16, 16, 16), (32, 64, 32), (64, 32, 16), (128, 128, 64)])
@pytest.mark.parametrize("scale", [0.05, 1.0])
def test_fp32_shapes(Dk, Dv, C, scale):
    inp = _case(2, 2, 3 * C + 5, Dk, Dv, C, "fp32", index=800 + Dk + Dv + C, scale=scale)
    rng = np.random.default_rng(Dk + Dv)
    h0 = 0.3 * rng.standard_normal((2, 2, Dk, Dv))
    dhT = 0.3 * rng.standard_normal((2, 2, Dk, Dv))
    compare(_gpu(inp, "fp32", C, h0=h0, dhT=dhT), _ref(inp, h0=h0, dhT=dhT), TOL["fp32"])


def test_fp32_no_l2norm():
    inp = _case(1, 2, 77, 32, 32, 16, "fp32", index=830)
    inp["k"] = 0.3 * inp["k"]
    compare(_gpu(inp, "fp32", 16, l2norm=False), _ref(inp, l2norm=False), TOL["fp32"])


@pytest.mark.parametrize("L", [64, 300])
def test_bf16_target_shape(L):
    inp = _case(2, 2, L, 128, 128, 64, "bf16", index=840 + L)
    compare(_gpu(inp, "bf16", 64), _ref(inp), TOL["bf16"])


def test_zero_gate_equals_ungated_kernel():
    """g = 0 through the gated entry points is the ungated SIMT computation, bit for bit."""
    import paper_2406_06484_b200 as dn
    inp = _case(2, 2, 150, 64, 64, 32, "fp32", index=850)
    inp["g"] = np.zeros_like(inp["g"])
    got = _gpu(inp, "fp32", 32)
    q, k, v, b, dO = (to_dev(inp[f], torch.float32) for f in ("q", "k", "v", "beta", "dO"))
    o, hT, ws = dn.deltanet_fwd(q, k, v, b, chunk=32, force_simt=True)
    dq, dk, dv, db, dh0 = dn.deltanet_bwd(q, k, v, b, dO, chunk=32, workspace=ws,
                                          force_simt=True)
    torch.cuda.synchronize()
    for key, t in (("o", o), ("hT", hT), ("dq", dq), ("dk", dk), ("dv", dv), ("dbeta", db),
                   ("dh0", dh0)):
        assert np.array_equal(got[key], _np(t)), key


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
@pytest.mark.parametrize("scale", [0.05, 1.0])
def test_recurrent_gated(dtype, scale):
    import paper_2406_06484_b200 as dn
    inp = _case(2, 3, 70, 128, 128, 64, dtype, index=860, scale=scale)
    td = torch_dtype(dtype)
    q, k, v, b = (to_dev(inp[f], td) for f in ("q", "k", "v", "beta"))
    g = to_dev(inp["g"], torch.float32)
    h0 = 0.3 * np.random.default_rng(2).standard_normal((2, 3, 128, 128))
    o, hT = dn.deltanet_gated_recurrent_fwd(q, k, v, b, g, h0=to_dev(h0, torch.float32))
    torch.cuda.synchronize()
    ro, rhT = oracle.gated_fwd(inp["q"], inp["k"], inp["v"], inp["beta"], inp["g"], h0=h0)
    compare({"o": _np(o), "hT": _np(hT)}, {"o": ro, "hT": rhT}, TOL[dtype])


def test_recurrent_gated_decode_loop():
    """One-token gated calls carrying the state in place equal one call over L."""
    import paper_2406_06484_b200 as dn
    inp = _case(1, 2, 24, 128, 128, 64, "bf16", index=870, scale=0.3)
    q, k, v, b = (to_dev(inp[f], torch.bfloat16) for f in ("q", "k", "v", "beta"))
    g = to_dev(inp["g"], torch.float32)
    o_ref, h_ref = dn.deltanet_gated_recurrent_fwd(q, k, v, b, g)
    state = torch.zeros((1, 2, 128, 128), dtype=torch.float32, device="cuda")
    outs = []
    for t in range(24):
        sl = lambda x: x[:, :, t:t + 1].contiguous()
        o, _ = dn.deltanet_gated_recurrent_fwd(sl(q), sl(k), sl(v), sl(b), sl(g), h0=state,
                                               hT=state)
        outs.append(o)
    torch.cuda.synchronize()
    assert torch.equal(torch.cat(outs, 2), o_ref)
    assert torch.equal(state, h_ref)


@pytest.mark.parametrize("scale", [0.05, 1.0, 4.0])
@pytest.mark.parametrize("L", [64, 1000])
def test_bf16_tcgen05_forward(L, scale):
    """The tcgen05 gated forward (include/deltanet.h: path 1 for bf16 d=128
    C=64) from a nonzero h0, slow to very fast decay (4.0: e^{-4 softplus}
    per token, in-chunk products far below fp32's range as ratios)."""
    import paper_2406_06484_b200 as dn
    assert dn.deltanet_path(dn.make_desc(2, 2, L, 128, 128, gated=True)) == 1
    inp = _case(2, 2, L, 128, 128, 64, "bf16", index=880 + L, scale=scale)
    q, k, v, b = (to_dev(inp[f], torch.bfloat16) for f in ("q", "k", "v", "beta"))
    g = to_dev(inp["g"], torch.float32)
    h0 = 0.3 * np.random.default_rng(4).standard_normal((2, 2, 128, 128))
    o, hT, _ = dn.deltanet_gated_fwd(q, k, v, b, g, h0=to_dev(h0, torch.float32))
    torch.cuda.synchronize()
    ro, rhT = oracle.gated_fwd(inp["q"], inp["k"], inp["v"], inp["beta"], inp["g"], h0=h0)
    compare({"o": _np(o), "hT": _np(hT)}, {"o": ro, "hT": rhT}, TOL["bf16"])


def test_bf16_gated_full_size_sampled_units():
    """BASELINE target shape (B=8 H=16 L=4096) gated forward in one launch;
    three sampled units against the oracle."""
    import paper_2406_06484_b200 as dn
    cfg = synth.CONFIGS["target"]
    inp = synth.make_inputs(cfg)
    gates = synth.make_gates(cfg)
    q, k, v, b = (to_dev(inp[f], torch.bfloat16) for f in ("q", "k", "v", "beta"))
    o, hT, _ = dn.deltanet_gated_fwd(q, k, v, b, to_dev(gates, torch.float32))
    torch.cuda.synchronize()
    o, hT = _np(o), _np(hT)
    for (bb, h) in [(0, 0), (cfg.B - 1, cfg.H - 1), (3, 9)]:
        one = {f: inp[f][bb:bb + 1, h:h + 1] for f in inp}
        ro, rhT = oracle.gated_fwd(one["q"], one["k"], one["v"], one["beta"],
                                   gates[bb:bb + 1, h:h + 1])
        compare({"o": o[bb:bb + 1, h:h + 1], "hT": hT[bb:bb + 1, h:h + 1]},
                {"o": ro, "hT": rhT}, TOL["bf16"])


# ------------------------------------------- tcgen05 gated backward (tc_bwd.cu)

@pytest.mark.parametrize("scale", [0.05, 1.0, 4.0])
@pytest.mark.parametrize("L", [64, 1000])
def test_bf16_tcgen05_backward(L, scale):
    """The tcgen05 gated backward (tc_bwd_kernel<false, true>)
    from a nonzero h0 and dhT, slow to very fast decay (4.0: in-chunk decay
    products far below fp32's range as ratios), a ragged tail at L = 1000;
    every gradient incl. dg and dh0 against the fp64 oracle."""
    import paper_2406_06484_b200 as dn
    d = dn.make_desc(2, 2, L, 128, 128, gated=True, save_states=False)
    # path 1 and 2 launches (state recompute + backward): the tcgen05 backward
    assert dn.deltanet_path(d) == 1 and dn.deltanet_launch_count(d, 1) == 2
    inp = _case(2, 2, L, 128, 128, 64, "bf16", index=890 + L, scale=scale)
    rng = np.random.default_rng(L)
    h0 = 0.3 * rng.standard_normal((2, 2, 128, 128))
    dhT = 0.3 * rng.standard_normal((2, 2, 128, 128))
    got, ref = _gpu(inp, "bf16", 64, h0=h0, dhT=dhT), _ref(inp, h0=h0, dhT=dhT)
    compare(got, ref, TOL["bf16"])
    # per-token gradients: per 64-token window, not only against the tensor max
    row_guard(got, ref, "dbeta", TOL["bf16"])
    row_guard(got, ref, "dg", TOL["bf16"])


def test_bf16_tcgen05_backward_no_l2_and_recompute():
    """Flag off (caller-normalised keys) and the backward without a saved
    workspace (states recomputed by the gated forward inside the call)."""
    import paper_2406_06484_b200 as dn
    inp = _case(1, 2, 200, 128, 128, 64, "bf16", index=897)
    for f in ("q", "k"):
        x = inp[f]
        inp[f] = (x / np.maximum(np.linalg.norm(x, axis=-1, keepdims=True), 1e-6))
    got = _gpu(inp, "bf16", 64, l2norm=False)
    compare(got, _ref(inp, l2norm=False), TOL["bf16"])
    td = torch.bfloat16
    q, k, v, b, dO = (to_dev(inp[f], td) for f in ("q", "k", "v", "beta", "dO"))
    g = to_dev(inp["g"], torch.float32)
    dq, dk, dv, db, dg, _ = dn.deltanet_gated_bwd(q, k, v, b, g, dO, l2norm=False)
    torch.cuda.synchronize()
    for key, t in (("dq", dq), ("dk", dk), ("dv", dv), ("dbeta", db), ("dg", dg)):
        assert np.array_equal(got[key], _np(t)), key


def test_bf16_gated_backward_full_size_sampled_units():
    """BASELINE target shape (B=8 H=16 L=4096) gated forward + backward on the
    tcgen05 kernels; two sampled units' gradients against the oracle."""
    import paper_2406_06484_b200 as dn
    cfg = synth.CONFIGS["target"]
    inp = synth.make_inputs(cfg)
    gates = synth.make_gates(cfg)
    td = torch.bfloat16
    q, k, v, b, dO = (to_dev(inp[f], td) for f in ("q", "k", "v", "beta", "dO"))
    g = to_dev(gates, torch.float32)
    o, hT, ws = dn.deltanet_gated_fwd(q, k, v, b, g)
    dq, dk, dv, db, dg, dh0 = dn.deltanet_gated_bwd(q, k, v, b, g, dO, workspace=ws)
    torch.cuda.synchronize()
    got = {"dq": _np(dq), "dk": _np(dk), "dv": _np(dv), "dbeta": _np(db), "dg": _np(dg),
           "dh0": _np(dh0)}
    for (bb, h) in [(0, 0), (cfg.B - 1, cfg.H - 1)]:
        one = {f: inp[f][bb:bb + 1, h:h + 1] for f in inp}
        r = oracle.gated_bwd(one["q"], one["k"], one["v"], one["beta"],
                             gates[bb:bb + 1, h:h + 1], one["dO"])
        ref = dict(zip(("dq", "dk", "dv", "dbeta", "dg", "dh0"), r))
        sub = {kk: vv[bb:bb + 1, h:h + 1] for kk, vv in got.items()}
        compare(sub, ref, TOL["bf16"])
        row_guard(sub, ref, "dbeta", TOL["bf16"])
        row_guard(sub, ref, "dg", TOL["bf16"])


@pytest.mark.parametrize("L", [1, 63, 65, 128])
def test_bf16_tcgen05_backward_edge_lengths(L):
    """tcgen05 gated backward at a single token, one partial chunk, one
    chunk plus one token and exactly two chunks (the chunk-end gate terms
    and the dH rescale at every boundary), from nonzero h0 and dhT."""
    inp = _case(1, 2, L, 128, 128, 64, "bf16", index=910 + L, scale=1.0)
    rng = np.random.default_rng(100 + L)
    h0 = 0.3 * rng.standard_normal((1, 2, 128, 128))
    dhT = 0.3 * rng.standard_normal((1, 2, 128, 128))
    compare(_gpu(inp, "bf16", 64, h0=h0, dhT=dhT), _ref(inp, h0=h0, dhT=dhT), TOL["bf16"])


def test_bf16_tcgen05_backward_zero_gate_matches_ungated():
    """g = 0: the gated tcgen05 backward reduces to the ungated one (every
    gate factor is exactly 1); same inputs, gradients equal to bf16 output
    rounding, and dg is the exact derivative at g = 0 (oracle)."""
    import paper_2406_06484_b200 as dn
    inp = _case(2, 2, 300, 128, 128, 64, "bf16", index=930)
    inp["g"] = np.zeros_like(inp["g"])
    got = _gpu(inp, "bf16", 64)
    td = torch.bfloat16
    q, k, v, b, dO = (to_dev(inp[f], td) for f in ("q", "k", "v", "beta", "dO"))
    o, hT, ws = dn.deltanet_fwd(q, k, v, b)
    dq, dk, dv, db, dh0 = dn.deltanet_bwd(q, k, v, b, dO, workspace=ws)
    torch.cuda.synchronize()
    ung = {"dq": _np(dq), "dk": _np(dk), "dv": _np(dv), "dbeta": _np(db), "dh0": _np(dh0)}
    compare({kk: got[kk] for kk in ung}, ung, 1e-2)
    compare({"dg": got["dg"]}, {"dg": _ref(inp)["dg"]}, TOL["bf16"])


@pytest.mark.parametrize("shift", [0.02, 0.06])
def test_bf16_tcgen05_positive_log_gates(shift):
    """deltanet.h accepts any finite g: with g > 0 on some tokens the in-chunk
    G_i - G_j is positive for j <= i, and Gamma(i, j) = e^{G_i - G_j} > 1 must
    not be clamped (the tcgen05 kernels masked by clamping the
    exponent at 0).  g = shift - 0.05 softplus(N(0,1)) mixes signs."""
    inp = _case(1, 2, 3 * 64 + 21, 128, 128, 64, "bf16", 970)
    inp["g"] = (inp["g"] + np.float32(shift)).astype(np.float32)
    assert (inp["g"] > 0).any() and (inp["g"] < 0).any()
    rng = np.random.default_rng(971)
    h0 = 0.1 * rng.standard_normal((1, 2, 128, 128))
    dhT = 0.1 * rng.standard_normal((1, 2, 128, 128))
    compare(_gpu(inp, "bf16", 64, h0=h0, dhT=dhT), _ref(inp, h0=h0, dhT=dhT), TOL["bf16"])
