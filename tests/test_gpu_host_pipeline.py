"""deltanet_fwd_bwd_host (include/deltanet.h): forward + backward of
host-resident tensors through the library's three-stream slab pipeline.
Slab results must equal the device-resident calls on the same units
(bitwise where the slab and the whole batch run the same kernels), and the
oracle to the bf16 bar."""
import numpy as np
import pytest
import torch

import synth
from parity import TOL, compare, run_oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2406_06484_b200 import build
    build.build()


def _host(inp, dtype):
    return {f: torch.from_numpy(np.ascontiguousarray(inp[f])).to(dtype).pin_memory()
            for f in ("q", "k", "v", "beta", "dO")}


def _run_host(x, slabs, **kw):
    import paper_2406_06484_b200 as dn
    out = tuple(torch.empty_like(x[f]).pin_memory() for f in ("v", "q", "k", "v", "beta"))
    dn.deltanet_fwd_bwd_host(x["q"], x["k"], x["v"], x["beta"], x["dO"], out=out, slabs=slabs,
                             **kw)
    torch.cuda.synchronize()
    return out


@pytest.mark.parametrize("slabs", [1, 2, 3, 7, 10, 11])
def test_matches_device_calls(slabs):
    """B*H = 10 units in 1..10 slabs (uneven last slab; 11 clamps to 10):
    bitwise equal to deltanet_fwd / deltanet_bwd of the device-resident batch."""
    import paper_2406_06484_b200 as dn
    cfg = synth.custom_config(5, 2, 300, 128, 128, 64, "bf16", index=900)
    inp = synth.make_inputs(cfg)
    x = _host(inp, torch.bfloat16)
    o, dq, dk, dv, db = _run_host(x, slabs)
    xd = {f: t.cuda() for f, t in x.items()}
    ro, _, ws = dn.deltanet_fwd(xd["q"], xd["k"], xd["v"], xd["beta"], want_hT=False)
    g = dn.deltanet_bwd(xd["q"], xd["k"], xd["v"], xd["beta"], xd["dO"], workspace=ws)
    torch.cuda.synchronize()
    for a, b in zip((o, dq, dk, dv, db), (ro, *g[:4])):
        assert torch.equal(a, b.cpu())


def test_long_slabs_against_oracle():
    """Slabs long enough to run the segment-parallel kernels (2 units per
    slab): against the oracle on every unit."""
    cfg = synth.custom_config(2, 2, 2048, 128, 128, 64, "bf16", index=901)
    inp = synth.make_inputs(cfg)
    o, dq, dk, dv, db = _run_host(_host(inp, torch.bfloat16), 2)
    f = lambda t: t.float().numpy().astype(np.float64)
    got = {"o": f(o), "dq": f(dq), "dk": f(dk), "dv": f(dv), "dbeta": f(db)}
    ref = run_oracle(inp)
    compare(got, ref, TOL["bf16"], keys=list(got))


def test_fp32_simt_path():
    cfg = synth.custom_config(3, 2, 70, 32, 64, 16, "fp32", index=902)
    inp = synth.make_inputs(cfg)
    o, dq, dk, dv, db = _run_host(_host(inp, torch.float32), 2, chunk=16)
    f = lambda t: t.numpy().astype(np.float64)
    got = {"o": f(o), "dq": f(dq), "dk": f(dk), "dv": f(dv), "dbeta": f(db)}
    compare(got, run_oracle(inp), TOL["fp32"], keys=list(got))


def test_small_device_buffer_is_an_error():
    import paper_2406_06484_b200 as dn
    cfg = synth.custom_config(2, 2, 64, 128, 128, 64, "bf16", index=903)
    x = _host(synth.make_inputs(cfg), torch.bfloat16)
    out = tuple(torch.empty_like(x[f]) for f in ("v", "q", "k", "v", "beta"))
    small = torch.empty(1024, dtype=torch.uint8, device="cuda")
    lib = dn.load_library()
    d = dn.make_desc(2, 2, 64, 128, 128)
    P = lambda t: t.data_ptr()
    import ctypes
    rc = lib.deltanet_fwd_bwd_host(ctypes.byref(d), *(ctypes.c_void_p(P(x[f])) for f in
                                   ("q", "k", "v", "beta", "dO")),
                                   *(ctypes.c_void_p(P(t)) for t in out), 2,
                                   ctypes.c_void_p(P(small)), 1024, None)
    assert rc == 5


def test_uneven_slabs_with_segments_in_the_last():
    """B*H = 99 units in 2 slabs at L = 2048.  The full slab (50
    units) runs one CTA per unit, the short last slab (49) picks the
    segment-parallel kernels and needs more workspace scratch; the shared
    workspace is sized for both.  Sampled units against the oracle."""
    cfg = synth.custom_config(33, 3, 2048, 128, 128, 64, "bf16", index=904)
    inp = synth.make_inputs(cfg)
    o, dq, dk, dv, db = _run_host(_host(inp, torch.bfloat16), 2)
    f = lambda t: t.float().numpy().astype(np.float64)
    pick = [(0, 0), (16, 1), (16, 2), (32, 2)]  # both slabs, incl. the last unit
    sel = lambda a: np.stack([a[b, h] for b, h in pick])[:, None]
    sub = {k_: sel(v_) for k_, v_ in inp.items()}
    got = {"o": sel(f(o)), "dq": sel(f(dq)), "dk": sel(f(dk)), "dv": sel(f(dv)),
           "dbeta": sel(f(db))}
    compare(got, run_oracle(sub), TOL["bf16"], keys=list(got))


def test_out_buffers_are_checked():
    """Mis-shaped or mis-typed out= buffers are refused before any launch
    (they would be written out of bounds by TMA stores)."""
    import paper_2406_06484_b200 as dn
    cfg = synth.custom_config(1, 2, 130, 128, 128, 64, "bf16", index=905)
    x = {f: t.cuda() for f, t in _host(synth.make_inputs(cfg), torch.bfloat16).items()}
    args = (x["q"], x["k"], x["v"], x["beta"])
    with pytest.raises(dn.DeltaNetError):
        dn.deltanet_fwd(*args, out=torch.empty((1, 2, 129, 128), dtype=torch.bfloat16,
                                               device="cuda"))
    with pytest.raises(dn.DeltaNetError):
        dn.deltanet_fwd(*args, out=torch.empty((1, 2, 130, 128), dtype=torch.float32,
                                               device="cuda"))
    o, _, ws = dn.deltanet_fwd(*args)
    bad = (torch.empty_like(x["q"]), torch.empty_like(x["k"]), torch.empty_like(x["v"]),
           torch.empty((1, 2, 64), dtype=torch.bfloat16, device="cuda"))
    with pytest.raises(dn.DeltaNetError):
        dn.deltanet_bwd(*args, x["dO"], workspace=ws, out=bad)
    with pytest.raises(dn.DeltaNetError):
        dn.deltanet_bwd(*args, x["dO"], workspace=ws.view(torch.int32)[:8])
