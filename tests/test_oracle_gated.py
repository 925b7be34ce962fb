"""Pins of the Gated DeltaNet oracle (oracle.gated_fwd / gated_bwd; PAPER.md
Table tab:overview; R23) against the
mathematics, not against itself:
  * g = 0 (alpha = 1) reduces to the pinned ungated oracle, bit for bit;
  * beta = 0 is pure decay: o_t = gamma_t H_0^T q_t, hT = gamma_L H_0, and the
    closed-form dg;
  * a very strong gate forgets the past: o_t = beta_t (k_t . q_t) v_t;
  * central finite differences of every input including g, with and
    without the L2 normalisation;
  * the chunkwise gated form (oracle/forms.py, the derivation the kernels
    follow) equals the recurrence for several chunk sizes and a padded tail,
    forward and backward.
CPU only."""
import numpy as np
import pytest

import oracle
from oracle import forms


def _inp(seed, B=2, H=2, L=23, Dk=6, Dv=5, gmax=0.6):
    rng = np.random.default_rng(seed)
    q = rng.standard_normal((B, H, L, Dk))
    k = rng.standard_normal((B, H, L, Dk))
    v = rng.standard_normal((B, H, L, Dv))
    beta = rng.uniform(0.05, 0.95, (B, H, L))
    g = -rng.uniform(0.0, gmax, (B, H, L))
    dO = rng.standard_normal((B, H, L, Dv))
    h0 = rng.standard_normal((B, H, Dk, Dv))
    dhT = rng.standard_normal((B, H, Dk, Dv))
    return q, k, v, beta, g, dO, h0, dhT


@pytest.mark.parametrize("l2norm", [True, False])
def test_zero_gate_is_ungated_bitwise(l2norm):
    q, k, v, beta, g, dO, h0, dhT = _inp(0)
    z = np.zeros_like(g)
    o, hT = oracle.gated_fwd(q, k, v, beta, z, h0=h0, l2norm=l2norm)
    o1, hT1 = oracle.recurrent_fwd(q, k, v, beta, h0=h0, l2norm=l2norm)
    assert np.array_equal(o, o1) and np.array_equal(hT, hT1)
    gg = oracle.gated_bwd(q, k, v, beta, z, dO, h0=h0, dhT=dhT, l2norm=l2norm)
    gu = oracle.recurrent_bwd(q, k, v, beta, dO, h0=h0, dhT=dhT, l2norm=l2norm)
    for a, b in zip(gg[:4] + gg[5:], gu):
        assert np.array_equal(a, b)


def test_pure_decay_closed_form():
    """beta = 0: H_t = alpha_t H_{t-1}, so o_t = gamma_t H_0^T q_t with
    gamma_t = exp(sum_{j<=t} g_j), hT = gamma_L H_0, and
    dl/dg_j = sum_{t>=j} gamma_t c_t (+ gamma_L <dhT, H_0>), c_t = q_t^T H_0 do_t."""
    q, k, v, beta, g, dO, h0, dhT = _inp(1)
    z = np.zeros_like(beta)
    o, hT = oracle.gated_fwd(q, k, v, z, g, h0=h0, l2norm=False)
    gam = np.exp(np.cumsum(g, axis=-1))
    ref = gam[..., None] * np.einsum("bhtk,bhkv->bhtv", q, h0)
    np.testing.assert_allclose(o, ref, rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(hT, gam[..., -1, None, None] * h0, rtol=1e-13, atol=1e-14)
    dg = oracle.gated_bwd(q, k, v, z, g, dO, h0=h0, dhT=dhT, l2norm=False)[4]
    c = np.einsum("bhtk,bhkv,bhtv->bht", q, h0, dO)
    tail = gam[..., -1] * (dhT * h0).sum((-1, -2))
    ref_dg = np.cumsum((gam * c)[..., ::-1], axis=-1)[..., ::-1] + tail[..., None]
    np.testing.assert_allclose(dg, ref_dg, rtol=1e-11, atol=1e-12)


def test_strong_gate_forgets():
    """alpha = e^-40: S_t = beta_t v_t k_t^T up to 4e-18, o_t = beta_t (k_t.q_t) v_t."""
    q, k, v, beta, g, _, h0, _ = _inp(2)
    g = np.full_like(beta, -40.0)
    o, _ = oracle.gated_fwd(q, k, v, beta, g, h0=h0, l2norm=True)
    qn = q / np.linalg.norm(q, axis=-1, keepdims=True)
    kn = k / np.linalg.norm(k, axis=-1, keepdims=True)
    ref = (beta * (qn * kn).sum(-1))[..., None] * v
    np.testing.assert_allclose(o, ref, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("l2norm", [True, False])
def test_backward_finite_differences(l2norm):
    q, k, v, beta, g, dO, h0, dhT = _inp(3, B=1, H=2, L=9, Dk=4, Dv=3)
    args = [q, k, v, beta, g, h0]

    def loss(a):
        o, hT = oracle.gated_fwd(a[0], a[1], a[2], a[3], a[4], h0=a[5], l2norm=l2norm)
        return float((o * dO).sum() + (hT * dhT).sum())

    dq, dk, dv, db, dg, dh0 = oracle.gated_bwd(q, k, v, beta, g, dO, h0=h0, dhT=dhT,
                                               l2norm=l2norm)
    h = 1e-6
    for idx, grad in enumerate((dq, dk, dv, db, dg, dh0)):
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
        np.testing.assert_allclose(grad.reshape(-1), num, rtol=1e-6, atol=1e-7,
                                   err_msg=f"input {idx}")


@pytest.mark.parametrize("C", [4, 8, 16, 64])
def test_chunkwise_gated_forward_equals_recurrence(C):
    q, k, v, beta, g, _, h0, _ = _inp(4, B=1, H=1, L=37, gmax=2.0)
    kn = k / np.linalg.norm(k, axis=-1, keepdims=True)
    qn = q / np.linalg.norm(q, axis=-1, keepdims=True)
    o, hT = oracle.gated_fwd(q, k, v, beta, g, h0=h0, l2norm=True)
    O, H = forms.gated_chunkwise_forward(qn[0, 0], kn[0, 0], v[0, 0], beta[0, 0], g[0, 0], C,
                                         h0[0, 0])
    np.testing.assert_allclose(O, o[0, 0], rtol=1e-11, atol=1e-12)
    np.testing.assert_allclose(H, hT[0, 0], rtol=1e-11, atol=1e-12)


@pytest.mark.parametrize("C", [4, 8, 16])
def test_chunkwise_gated_backward_equals_bptt(C):
    q, k, v, beta, g, dO, h0, dhT = _inp(5, B=1, H=1, L=48, gmax=1.5)
    kn = k / np.linalg.norm(k, axis=-1, keepdims=True)
    qn = q / np.linalg.norm(q, axis=-1, keepdims=True)
    ref = oracle.gated_bwd(qn, kn, v, beta, g, dO, h0=h0, dhT=dhT, l2norm=False)
    got = forms.gated_chunkwise_backward(qn[0, 0], kn[0, 0], v[0, 0], beta[0, 0], g[0, 0],
                                         dO[0, 0], C, h0[0, 0], dhT[0, 0])
    for name, a, b in zip(("dq", "dk", "dv", "dbeta", "dg", "dh0"), got, ref):
        np.testing.assert_allclose(a, b[0, 0], rtol=1e-10, atol=1e-11, err_msg=name)


@pytest.mark.parametrize("L,C", [(160, 16), (135, 5)])
def test_chunkwise_gated_backward_checkpoint_segments(L, C):
    """L > 128: the gated oracle's BPTT walks three checkpoint segments of 64
    tokens (the last ragged) and still equals the independent chunked adjoint
    (oracle/forms.py::gated_chunkwise_backward)."""
    q, k, v, beta, g, dO, h0, dhT = _inp(6 + L, B=1, H=1, L=L, Dk=8, Dv=6, gmax=0.3)
    kn = k / np.linalg.norm(k, axis=-1, keepdims=True)
    qn = q / np.linalg.norm(q, axis=-1, keepdims=True)
    ref = oracle.gated_bwd(qn, kn, v, beta, g, dO, h0=h0, dhT=dhT, l2norm=False)
    got = forms.gated_chunkwise_backward(qn[0, 0], kn[0, 0], v[0, 0], beta[0, 0], g[0, 0],
                                         dO[0, 0], C, h0[0, 0], dhT[0, 0])
    for name, a, b in zip(("dq", "dk", "dv", "dbeta", "dg", "dh0"), got, ref):
        scale = max(1.0, np.abs(b).max())
        np.testing.assert_allclose(a, b[0, 0], rtol=0, atol=1e-10 * scale, err_msg=name)


def test_backward_finite_differences_checkpoint_segments():
    """Central differences at L = 150 (three checkpoint segments, ragged) of
    every input of the gated oracle, incl. g and h0, with L2 normalisation."""
    q, k, v, beta, g, dO, h0, dhT = _inp(9, B=1, H=1, L=150, Dk=3, Dv=2, gmax=0.2)
    args = [q, k, v, beta, g, h0]

    def loss(a):
        o, hT = oracle.gated_fwd(a[0], a[1], a[2], a[3], a[4], h0=a[5], l2norm=True)
        return float((o * dO).sum() + (hT * dhT).sum())

    grads = oracle.gated_bwd(q, k, v, beta, g, dO, h0=h0, dhT=dhT, l2norm=True)
    h = 1e-5   # see test_oracle.py::test_backward_checkpoint_segments_finite_differences
    for idx, grad in enumerate(grads):
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
        err = np.abs(grad.reshape(-1) - num)
        assert np.all(err <= 1e-6 * np.abs(num) + 1e-9 * np.abs(num).max()), idx
