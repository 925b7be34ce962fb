"""GPU parity of the layer prologue (deltanet_prologue_fwd / _bwd, SURVEY
§8(f) f1) against oracle/prologue.py (fp64, the definitions of P:96, P:329,
P:340-341) on the same rounded inputs, normwise (R16):
1e-4 for fp32 I/O, 2e-2 for bf16 I/O; the fp32 weight gradients of the bf16
path are reductions of bf16-rounded products and get the bf16 bar."""
import numpy as np
import pytest
import torch

from oracle import prologue as P
from parity import TOL, compare, to_dev, torch_dtype

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2406_06484_b200 import build
    build.build()


def _round(a, dtype):
    t = torch.from_numpy(np.ascontiguousarray(a)).to(torch_dtype(dtype))
    return t.to(torch.float64).numpy()


def _case(B, L, H, Dk, Dv, dtype, seed):
    rng = np.random.default_rng(seed)
    xq, xk = (_round(rng.standard_normal((B, L, H, Dk)), dtype) for _ in range(2))
    xv = _round(rng.standard_normal((B, L, H, Dv)), dtype)
    xb = _round(rng.standard_normal((B, L, H)), dtype)
    wq, wk = (0.5 * rng.standard_normal((H * Dk, 4)).astype(np.float32) for _ in range(2))
    wv = 0.5 * rng.standard_normal((H * Dv, 4)).astype(np.float32)
    g = [_round(rng.standard_normal((B, H, L, Dk)), dtype) for _ in range(2)]
    g.append(_round(rng.standard_normal((B, H, L, Dv)), dtype))
    g.append(_round(rng.standard_normal((B, H, L)), dtype))
    return (xq, xk, xv, xb, wq, wk, wv), g


def _gpu(args, g, dtype, silu_v):
    import paper_2406_06484_b200 as dn
    td = torch_dtype(dtype)
    xs = [to_dev(a, td) for a in args[:4]]
    ws = [to_dev(a, torch.float32) for a in args[4:]]
    gs = [to_dev(a, td) for a in g]
    q, k, v, beta = dn.deltanet_prologue_fwd(*xs, *ws, silu_v=silu_v)
    grads = dn.deltanet_prologue_bwd(*xs, *ws, *gs, silu_v=silu_v)
    torch.cuda.synchronize()
    f = lambda t: t.float().cpu().numpy()
    return [f(t) for t in (q, k, v, beta)], [f(t) for t in grads]


FWD = ("q", "k", "v", "beta")
BWD = ("dxq", "dxk", "dxv", "dxb", "dwq", "dwk", "dwv")


@pytest.mark.parametrize("L", [1, 3, 37, 512, 1100])
@pytest.mark.parametrize("silu_v", [False, True])
def test_fp32(L, silu_v):
    args, g = _case(2, L, 3, 32, 64, "fp32", seed=L)
    fo, bo = _gpu(args, g, "fp32", silu_v)
    rf = P.prologue_fwd(*args, silu_v=silu_v)
    rb = P.prologue_bwd(*args, *g, silu_v=silu_v)
    compare(dict(zip(FWD, fo)), dict(zip(FWD, rf)), TOL["fp32"])
    compare(dict(zip(BWD, bo)), dict(zip(BWD, rb)), TOL["fp32"])


@pytest.mark.parametrize("Dk,Dv", [(128, 128), (16, 256), (256, 16)])
def test_bf16(Dk, Dv):
    args, g = _case(2, 700, 2, Dk, Dv, "bf16", seed=Dk + Dv)
    fo, bo = _gpu(args, g, "bf16", False)
    rf = P.prologue_fwd(*args)
    rb = P.prologue_bwd(*args, *g)
    compare(dict(zip(FWD, fo)), dict(zip(FWD, rf)), TOL["bf16"])
    compare(dict(zip(BWD, bo)), dict(zip(BWD, rb)), TOL["bf16"])


def test_deterministic():
    args, g = _case(2, 1300, 4, 128, 128, "bf16", seed=9)
    a = _gpu(args, g, "bf16", False)
    b = _gpu(args, g, "bf16", False)
    for x, y in zip(a[0] + a[1], b[0] + b[1]):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("silu_v", [False, True])
def test_bf16_tma_tiles(silu_v):
    """bf16 D = 128 (the TMA-staged kernels): several 1024-token tiles, so
    the conv window and the dx look-ahead cross tile and stage boundaries,
    a ragged last tile, and the deterministic dw reduction over tiles."""
    args, g = _case(2, 2 * 1024 + 77, 3, 128, 128, "bf16", seed=31 + silu_v)
    fo, bo = _gpu(args, g, "bf16", silu_v)
    rf = P.prologue_fwd(*args, silu_v=silu_v)
    rb = P.prologue_bwd(*args, *g, silu_v=silu_v)
    compare(dict(zip(FWD, fo)), dict(zip(FWD, rf)), TOL["bf16"])
    compare(dict(zip(BWD, bo)), dict(zip(BWD, rb)), TOL["bf16"])
