"""Pins of the context-parallel oracle (oracle/context.py) against the
full-sequence recurrence and the paper's Householder product -- not against
itself.  A sequence is cut into parts at uneven boundaries (an empty part
included); stitching the per-part transitions must reproduce the prefix end
states, the suffix cotangents, and the part-wise outputs / gradients of one
uncut run.  CPU only."""
import numpy as np
import pytest

import oracle
from oracle import context as cp
from oracle import forms


def _seq(seed, B=2, H=2, L=29, Dk=8, Dv=6):
    rng = np.random.default_rng(seed)
    q = rng.standard_normal((B, H, L, Dk))
    k = rng.standard_normal((B, H, L, Dk))
    v = rng.standard_normal((B, H, L, Dv))
    beta = rng.uniform(0.05, 0.95, (B, H, L))
    dO = rng.standard_normal((B, H, L, Dv))
    return q, k, v, beta, dO


CUTS = [0, 7, 7, 20, 29]  # parts of 7, 0, 13, 9 tokens


def _parts(x, cuts=CUTS, axis=2):
    return [np.take(x, range(a, b), axis=axis) for a, b in zip(cuts[:-1], cuts[1:])]


def test_psi_is_householder_product():
    """Psi of one unit = P_1^n of PAPER.md Eq. 4 (forms.householder_product),
    with unit keys; one token gives I - beta k k^T; beta = 0 gives I."""
    q, k, v, beta, _ = _seq(0, B=1, H=1)
    psi, _ = cp.transition(q, k, v, beta, l2norm=True)
    kn = k / np.linalg.norm(k, axis=-1, keepdims=True)
    np.testing.assert_allclose(psi[0, 0], forms.householder_product(kn[0, 0], beta[0, 0]),
                               rtol=1e-12, atol=1e-12)
    psi1, _ = cp.transition(q[:, :, :1], k[:, :, :1], v[:, :, :1], beta[:, :, :1])
    np.testing.assert_allclose(psi1[0, 0], np.eye(8) - beta[0, 0, 0] * np.outer(kn[0, 0, 0],
                                                                                 kn[0, 0, 0]),
                               rtol=1e-13, atol=1e-14)
    psi0, hl0 = cp.transition(q, k, v, np.zeros_like(beta))
    np.testing.assert_array_equal(psi0[0, 0], np.eye(8))
    np.testing.assert_array_equal(hl0, 0.0)


@pytest.mark.parametrize("l2norm", [True, False])
def test_end_state_affine_in_start_state(l2norm):
    """H_end(H_start) from the recurrence = Psi^T H_start + Hloc for random H_start."""
    q, k, v, beta, _ = _seq(1)
    if not l2norm:
        k = 0.3 * k
    psi, hloc = cp.transition(q, k, v, beta, l2norm=l2norm)
    h0 = np.random.default_rng(2).standard_normal((2, 2, 8, 6))
    _, hT = oracle.recurrent_fwd(q, k, v, beta, h0=h0, l2norm=l2norm)
    np.testing.assert_allclose(hT, np.swapaxes(psi, -1, -2) @ h0 + hloc, rtol=1e-10, atol=1e-12)


def test_forward_stitching_reproduces_uncut_run():
    q, k, v, beta, _ = _seq(3)
    h0 = np.random.default_rng(4).standard_normal((2, 2, 8, 6))
    o_full, hT_full = oracle.recurrent_fwd(q, k, v, beta, h0=h0)
    P = len(CUTS) - 1
    tr = [cp.transition(*xs) for xs in zip(*(_parts(x) for x in (q, k, v, beta)))]
    psi_all = np.stack([t[0] for t in tr])
    loc_all = np.stack([t[1] for t in tr])
    outs = []
    for p in range(P):
        hs = cp.state_scan(psi_all, loc_all, p, edge=h0)
        _, hpre = oracle.recurrent_fwd(q[:, :, :CUTS[p]], k[:, :, :CUTS[p]], v[:, :, :CUTS[p]],
                                       beta[:, :, :CUTS[p]], h0=h0)
        np.testing.assert_allclose(hs, hpre, rtol=1e-10, atol=1e-12, err_msg=f"part {p}")
        sl = slice(CUTS[p], CUTS[p + 1])
        o_p, hT_p = oracle.recurrent_fwd(q[:, :, sl], k[:, :, sl], v[:, :, sl], beta[:, :, sl],
                                         h0=hs)
        outs.append(o_p)
    np.testing.assert_allclose(np.concatenate(outs, axis=2), o_full, rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(hT_p, hT_full, rtol=1e-10, atol=1e-12)


def test_backward_stitching_reproduces_uncut_run():
    q, k, v, beta, dO = _seq(5)
    rng = np.random.default_rng(6)
    h0 = rng.standard_normal((2, 2, 8, 6))
    dhT = rng.standard_normal((2, 2, 8, 6))
    full = oracle.recurrent_bwd(q, k, v, beta, dO, h0=h0, dhT=dhT)
    P = len(CUTS) - 1
    xs = list(zip(*(_parts(x) for x in (q, k, v, beta, dO))))
    tr = [cp.transition(*x[:4]) for x in xs]
    psi_all = np.stack([t[0] for t in tr])
    loc_all = np.stack([t[1] for t in tr])
    dloc_all = np.stack([cp.bwd_transition(*x) for x in xs])
    grads = [[] for _ in range(4)]
    for p in range(P):
        hs = cp.state_scan(psi_all, loc_all, p, edge=h0)
        ge = cp.state_scan(psi_all, dloc_all, p, reverse=True, edge=dhT)
        # dl/dH_end(p) = dh0 of the uncut suffix after part p
        suf = slice(CUTS[p + 1], CUTS[-1])
        _, hmid = oracle.recurrent_fwd(q[:, :, :CUTS[p + 1]], k[:, :, :CUTS[p + 1]],
                                       v[:, :, :CUTS[p + 1]], beta[:, :, :CUTS[p + 1]], h0=h0)
        ref = oracle.recurrent_bwd(q[:, :, suf], k[:, :, suf], v[:, :, suf], beta[:, :, suf],
                                   dO[:, :, suf], h0=hmid, dhT=dhT)[4]
        np.testing.assert_allclose(ge, ref, rtol=1e-10, atol=1e-12, err_msg=f"part {p}")
        g = oracle.recurrent_bwd(*xs[p], h0=hs, dhT=ge)
        for i in range(4):
            grads[i].append(g[i])
        if p == 0:
            np.testing.assert_allclose(g[4], full[4], rtol=1e-10, atol=1e-12)
    for i in range(4):
        np.testing.assert_allclose(np.concatenate(grads[i], axis=2), full[i], rtol=1e-9,
                                   atol=1e-11, err_msg=f"grad {i}")


def test_cotangent_chain_is_adjoint():
    """<dl/dH_start, dH> for a perturbation dH of H_start equals the change of
    l = sum <dO, o>, i.e. dHloc + Psi dhT is the adjoint of the affine map
    (central difference; l is linear in H_start, so it is exact)."""
    q, k, v, beta, dO = _seq(7)
    rng = np.random.default_rng(8)
    h0 = rng.standard_normal((2, 2, 8, 6))
    dh = rng.standard_normal((2, 2, 8, 6))
    dhT = rng.standard_normal((2, 2, 8, 6))
    psi, _ = cp.transition(q, k, v, beta)
    g = cp.bwd_transition(q, k, v, beta, dO) + psi @ dhT

    def loss(h):
        o, hT = oracle.recurrent_fwd(q, k, v, beta, h0=h)
        return float((o * dO).sum() + (hT * dhT).sum())

    num = (loss(h0 + dh) - loss(h0 - dh)) / 2
    np.testing.assert_allclose((g * dh).sum(), num, rtol=1e-10)
