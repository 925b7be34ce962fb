"""fp64 oracle of the DeltaNet layer prologue -- TEST INFRASTRUCTURE.

Only ``tests/`` (and ``bench.py``'s reference legs) may import this module;
the product path never does.  Plain numpy in float64, loops over the four
taps, no blocking or fusion: the definitions written out.

* Short convolution after the q/k/v projections (§3.4, P:340-341;
  kernel size 4): causal and depthwise (one length-4 filter per
  channel c = h*D + d),  y[t] = sum_{j<4} w[c, j] * x[t - 3 + j],
  x[t < 0] = 0.
* Feature map: SiLU on q and k (SiLU(z) = z * sigmoid(z)); v is left
  linear (the paper names no activation for v; R22) unless
  ``silu_v``.
* beta = sigmoid(W_beta x): the prologue applies the sigmoid to the
  projected pre-activation xb.

Layouts: inputs token-major [B, L, H, D] (xb [B, L, H]) as the projections
produce them; outputs [B, H, L, D] (beta [B, H, L]) as the chunkwise kernel
consumes them.  Weights [H*D, 4].

``prologue_bwd`` is the reverse-mode derivative by the chain rule:
dy = dout * act'(y) with SiLU'(z) = s (1 + z (1 - s)), s = sigmoid(z);
dx[s] = sum_j w[c, j] dy[s + 3 - j] (dy[t >= L] = 0);
dw[c, j] = sum_{b, t} dy[t] x[t - 3 + j];  dxb = dbeta * beta (1 - beta).
Pinned in tests/test_oracle_prologue.py by central finite differences,
identity / shift filters, causality and closed forms.
"""
from __future__ import annotations

import numpy as np

TAPS = 4


def sigmoid(z):
    return 1.0 / (1.0 + np.exp(-z))


def silu(z):
    return z * sigmoid(z)


def silu_grad(z):
    s = sigmoid(z)
    return s * (1.0 + z * (1.0 - s))


def short_conv(x, w):
    """Causal depthwise conv along axis 1 of x [B, L, H, D] with w [H*D, 4]."""
    B, L, H, D = x.shape
    wc = np.asarray(w, dtype=np.float64).reshape(H, D, TAPS)
    x = np.asarray(x, dtype=np.float64)
    y = np.zeros_like(x)
    for j in range(TAPS):
        shift = TAPS - 1 - j  # tap j reads x[t - shift]
        if shift == 0:
            y += wc[None, None, :, :, j] * x
        elif shift < L:
            y[:, shift:] += wc[None, None, :, :, j] * x[:, :L - shift]
    return y


def _to_bhld(y):
    return np.ascontiguousarray(np.transpose(y, (0, 2, 1, 3)))


def _from_bhld(y):
    return np.ascontiguousarray(np.transpose(y, (0, 2, 1, 3)))


def prologue_fwd(xq, xk, xv, xb, wq, wk, wv, silu_v=False):
    """Returns q, k, v [B, H, L, D] and beta [B, H, L] (float64)."""
    yq, yk, yv = short_conv(xq, wq), short_conv(xk, wk), short_conv(xv, wv)
    q, k = silu(yq), silu(yk)
    v = silu(yv) if silu_v else yv
    beta = sigmoid(np.asarray(xb, dtype=np.float64))
    return _to_bhld(q), _to_bhld(k), _to_bhld(v), np.ascontiguousarray(np.transpose(beta, (0, 2, 1)))


def _conv_bwd(x, w, dy):
    """Adjoint of short_conv: dx [B, L, H, D] and dw [H*D, 4]."""
    B, L, H, D = x.shape
    wc = np.asarray(w, dtype=np.float64).reshape(H, D, TAPS)
    x = np.asarray(x, dtype=np.float64)
    dx = np.zeros_like(x)
    dw = np.zeros((H, D, TAPS))
    for j in range(TAPS):
        shift = TAPS - 1 - j
        if shift == 0:
            dx += wc[None, None, :, :, j] * dy
            dw[:, :, j] = (dy * x).sum(axis=(0, 1))
        elif shift < L:
            dx[:, :L - shift] += wc[None, None, :, :, j] * dy[:, shift:]
            dw[:, :, j] = (dy[:, shift:] * x[:, :L - shift]).sum(axis=(0, 1))
    return dx, dw.reshape(H * D, TAPS)


def prologue_bwd(xq, xk, xv, xb, wq, wk, wv, dq, dk, dv, dbeta, silu_v=False):
    """Cotangents dq, dk, dv [B, H, L, D], dbeta [B, H, L] -> dxq, dxk, dxv
    [B, L, H, D], dxb [B, L, H], dwq, dwk, dwv [H*D, 4] (float64)."""
    out = []
    for x, w, g, act in ((xq, wq, dq, True), (xk, wk, dk, True), (xv, wv, dv, silu_v)):
        y = short_conv(x, w)
        dy = _from_bhld(np.asarray(g, dtype=np.float64))
        if act:
            dy = dy * silu_grad(y)
        out.append(_conv_bwd(x, w, dy))
    s = sigmoid(np.asarray(xb, dtype=np.float64))
    dxb = np.transpose(np.asarray(dbeta, dtype=np.float64), (0, 2, 1)) * s * (1.0 - s)
    (dxq, dwq), (dxk, dwk), (dxv, dwv) = out
    return dxq, dxk, dxv, np.ascontiguousarray(dxb), dwq, dwk, dwv
