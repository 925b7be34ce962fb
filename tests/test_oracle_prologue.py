"""Pins of the layer-prologue oracle (oracle/prologue.py) against the
mathematics, not against itself: central finite differences of every input
and weight, identity / pure-shift filters, causality, and closed forms of
SiLU / sigmoid.  CPU only."""
import numpy as np
import pytest

from oracle import prologue as P


def _rand(rng, B=2, L=11, H=2, D=3):
    xq, xk, xv = (rng.standard_normal((B, L, H, D)) for _ in range(3))
    xb = rng.standard_normal((B, L, H))
    wq, wk, wv = (0.7 * rng.standard_normal((H * D, 4)) for _ in range(3))
    return xq, xk, xv, xb, wq, wk, wv


def test_closed_forms():
    assert P.sigmoid(0.0) == 0.5
    assert P.silu(0.0) == 0.0
    assert P.silu_grad(0.0) == 0.5
    z = np.linspace(-4, 4, 17)
    h = 1e-6
    np.testing.assert_allclose(P.silu_grad(z), (P.silu(z + h) - P.silu(z - h)) / (2 * h),
                               rtol=1e-8, atol=1e-10)


def test_identity_and_shift_filters():
    """w = e_3 (tap on x[t]) is the identity; w = e_0 delays by 3 tokens."""
    rng = np.random.default_rng(0)
    B, L, H, D = 2, 9, 2, 4
    x = rng.standard_normal((B, L, H, D))
    ident = np.zeros((H * D, 4))
    ident[:, 3] = 1.0
    np.testing.assert_array_equal(P.short_conv(x, ident), x)
    delay = np.zeros((H * D, 4))
    delay[:, 0] = 1.0
    y = P.short_conv(x, delay)
    np.testing.assert_array_equal(y[:, 3:], x[:, :-3])
    np.testing.assert_array_equal(y[:, :3], 0.0)
    q, k, v, beta = P.prologue_fwd(x, x, x, x[..., 0], ident, ident, ident)
    np.testing.assert_allclose(q, np.transpose(x * (1 / (1 + np.exp(-x))), (0, 2, 1, 3)),
                               rtol=1e-15)
    np.testing.assert_array_equal(v, np.transpose(x, (0, 2, 1, 3)))


def test_causal_and_depthwise():
    """Perturbing x[t0] changes y only at t in [t0, t0+3] and only in that channel."""
    rng = np.random.default_rng(1)
    B, L, H, D = 1, 12, 2, 3
    x = rng.standard_normal((B, L, H, D))
    w = rng.standard_normal((H * D, 4))
    y0 = P.short_conv(x, w)
    x1 = x.copy()
    x1[0, 5, 1, 2] += 1.0
    d = P.short_conv(x1, w) - y0
    nz = np.argwhere(np.abs(d) > 0)
    assert set(map(tuple, nz[:, 1:])) <= {(t, 1, 2) for t in range(5, 9)}
    np.testing.assert_allclose(d[0, 5:9, 1, 2], w[1 * D + 2][::-1], rtol=1e-12, atol=1e-14)


@pytest.mark.parametrize("silu_v", [False, True])
def test_backward_finite_differences(silu_v):
    rng = np.random.default_rng(2)
    args = _rand(rng)
    B, L, H, D = args[0].shape
    g = [rng.standard_normal((B, H, L, D)) for _ in range(3)] + [rng.standard_normal((B, H, L))]

    def loss(a):
        outs = P.prologue_fwd(*a, silu_v=silu_v)
        return sum(float((o * gg).sum()) for o, gg in zip(outs, g))

    grads = P.prologue_bwd(*args, *g, silu_v=silu_v)
    # grads order: dxq, dxk, dxv, dxb, dwq, dwk, dwv <-> args xq, xk, xv, xb, wq, wk, wv
    h = 1e-6
    for idx in range(7):
        base = [np.array(a, dtype=np.float64) for a in args]
        flat = base[idx].reshape(-1)
        num = np.zeros_like(flat)
        for i in range(flat.size):
            keep = flat[i]
            flat[i] = keep + h
            lp = loss(base)
            flat[i] = keep - h
            lm = loss(base)
            flat[i] = keep
            num[i] = (lp - lm) / (2 * h)
        np.testing.assert_allclose(grads[idx].reshape(-1), num, rtol=1e-6, atol=1e-7,
                                   err_msg=f"input {idx}")
