"""GPU parity of the recurrent (token-by-token) inference kernel
(deltanet_recurrent_fwd) against the fp64 oracle's
definition of the delta rule (§2.2), normwise
(R16): 1e-4 for fp32 I/O, 2e-2 for bf16 I/O.
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from parity import TOL, compare, to_dev, torch_dtype

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2406_06484_b200 import build
    build.build()


def _inputs(B, H, L, Dk, Dv, dtype, index, keys="silu"):
    cfg = synth.custom_config(B, H, L, Dk, Dv, 64, dtype, index=index)
    return synth.make_inputs(cfg, keys=keys)


def _run(inp, dtype, l2norm=True, h0=None, inplace=False):
    import paper_2406_06484_b200 as dn
    td = torch_dtype(dtype)
    q, k, v, b = (to_dev(inp[f], td) for f in ("q", "k", "v", "beta"))
    h0t = None if h0 is None else to_dev(h0, torch.float32)
    if inplace:
        o, hT = dn.deltanet_recurrent_fwd(q, k, v, b, l2norm=l2norm, h0=h0t, hT=h0t)
    else:
        o, hT = dn.deltanet_recurrent_fwd(q, k, v, b, l2norm=l2norm, h0=h0t)
    torch.cuda.synchronize()
    return {"o": o.float().cpu().numpy(), "hT": hT.cpu().numpy()}


def _oracle(inp, l2norm=True, h0=None):
    o, hT = oracle.recurrent_fwd(inp["q"], inp["k"], inp["v"], inp["beta"], h0=h0, l2norm=l2norm)
    return {"o": o, "hT": hT}


@pytest.mark.parametrize("Dk,Dv", [(16, 16), (32, 64), (64, 32), (128, 128), (256, 64),
                                   (128, 256), (64, 128)])
@pytest.mark.parametrize("l2norm", [True, False])
def test_fp32_shapes(Dk, Dv, l2norm):
    inp = _inputs(2, 2, 45, Dk, Dv, "fp32", index=600 + Dk + Dv)
    rng = np.random.default_rng(Dk * 7 + Dv)
    h0 = (0.3 * rng.standard_normal((2, 2, Dk, Dv))).astype(np.float32)
    got = _run(inp, "fp32", l2norm=l2norm, h0=h0)
    compare(got, _oracle(inp, l2norm=l2norm, h0=h0.astype(np.float64)), TOL["fp32"])


@pytest.mark.parametrize("L", [1, 32, 33, 200])
def test_bf16_lengths(L):
    """Token blocks of 32: exact multiples, a ragged tail, and decode (L=1)."""
    inp = _inputs(2, 3, L, 128, 128, "bf16", index=620 + L)
    got = _run(inp, "bf16")
    compare(got, _oracle(inp), TOL["bf16"])


def test_inplace_state_and_decode_loop():
    """hT aliasing h0 (in-place) equals the out-of-place call, and L single-
    token calls carrying the state equal one call over the L tokens (the same
    per-token arithmetic, so bitwise)."""
    import paper_2406_06484_b200 as dn
    inp = _inputs(1, 2, 40, 128, 128, "bf16", index=640)
    rng = np.random.default_rng(5)
    h0 = (0.2 * rng.standard_normal((1, 2, 128, 128))).astype(np.float32)
    ref = _run(inp, "bf16", h0=h0)
    inpl = _run(inp, "bf16", h0=h0, inplace=True)
    for key in ref:
        assert np.array_equal(ref[key], inpl[key]), key
    td = torch.bfloat16
    q, k, v, b = (to_dev(inp[f], td) for f in ("q", "k", "v", "beta"))
    state = to_dev(h0, torch.float32)
    outs = []
    for t in range(40):
        o, _ = dn.deltanet_recurrent_fwd(q[:, :, t:t + 1].contiguous(), k[:, :, t:t + 1].contiguous(),
                                         v[:, :, t:t + 1].contiguous(), b[:, :, t:t + 1].contiguous(),
                                         h0=state, hT=state)
        outs.append(o)
    torch.cuda.synchronize()
    o_loop = torch.cat(outs, dim=2).float().cpu().numpy()
    assert np.array_equal(o_loop, ref["o"])
    assert np.array_equal(state.cpu().numpy(), ref["hT"])


def test_matches_chunkwise_forward():
    """The recurrent and chunkwise (tcgen05) kernels compute the same forward
    (§3.2: the chunkwise form is exact); both are bf16-rounded, so
    they agree to the bf16 bar against each other."""
    import paper_2406_06484_b200 as dn
    inp = _inputs(2, 2, 256, 128, 128, "bf16", index=650)
    td = torch.bfloat16
    q, k, v, b = (to_dev(inp[f], td) for f in ("q", "k", "v", "beta"))
    o_r, h_r = dn.deltanet_recurrent_fwd(q, k, v, b)
    o_c, h_c, _ = dn.deltanet_fwd(q, k, v, b, chunk=64)
    torch.cuda.synchronize()
    compare({"o": o_r.float().cpu().numpy(), "hT": h_r.cpu().numpy()},
            {"o": o_c.float().cpu().numpy(), "hT": h_c.cpu().numpy()}, TOL["bf16"])


def test_bf16_full_size_sampled_units():
    """BASELINE target config (B=8 H=16 L=4096 d=128) in one launch; the
    oracle checks three sampled units."""
    cfg = synth.CONFIGS["target"]
    inp = synth.make_inputs(cfg)
    got = _run(inp, "bf16")
    for (b, h) in [(0, 0), (cfg.B - 1, cfg.H - 1), (cfg.B // 2, 7)]:
        one = {f: inp[f][b:b + 1, h:h + 1] for f in inp}
        ref = _oracle(one)
        sub = {key: val[b:b + 1, h:h + 1] for key, val in got.items()}
        compare(sub, ref, TOL["bf16"])
