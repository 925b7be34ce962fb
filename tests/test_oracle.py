"""Pins for the fp64 oracle (CPU only, -m "not gpu").

The oracle is the plain token-by-token delta rule (§2.2 lines
82-97).  Nothing here re-calls the oracle's own formula: each test checks it
against something the paper or the mathematics fixes independently --
a hand-derived example, closed forms, the paper's invariants, the paper's
other forms of the same computation (WY / UT / chunkwise / parallel, coded
separately in oracle/forms.py), and central finite differences.
"""
import json
import os

import numpy as np
import pytest

import oracle
from oracle import forms

GOLD = os.path.join(os.path.dirname(__file__), "golden", "hand_example_L2_d2.json")


def _b(x):  # add the [B=1, H=1] axes
    return np.asarray(x, dtype=np.float64)[None, None]


def _rand_unit(rng, L, dk, dv, unit_keys=True):
    q = rng.standard_normal((L, dk))
    k = rng.standard_normal((L, dk))
    if unit_keys:
        q /= np.linalg.norm(q, axis=1, keepdims=True)
        k /= np.linalg.norm(k, axis=1, keepdims=True)
    v = rng.standard_normal((L, dv))
    beta = 1.0 / (1.0 + np.exp(-rng.standard_normal(L)))
    return q, k, v, beta


def _fwd(q, k, v, beta, h0=None, l2norm=False):
    o, hT = oracle.recurrent_fwd(_b(q), _b(k), _b(v), _b(beta),
                                 None if h0 is None else _b(h0), l2norm=l2norm)
    return o[0, 0], hT[0, 0]


def _bwd(q, k, v, beta, dO, h0=None, dhT=None, l2norm=False):
    g = oracle.recurrent_bwd(_b(q), _b(k), _b(v), _b(beta), _b(dO),
                             None if h0 is None else _b(h0),
                             None if dhT is None else _b(dhT), l2norm=l2norm)
    return [a[0, 0] for a in g]


# --------------------------------------------------------------------------
# Golden example (hand arithmetic, tests/golden/hand_example_L2_d2.json)
# --------------------------------------------------------------------------

def test_golden_hand_arithmetic():
    """Re-derive the fixture's forward values by scalar hand arithmetic so the
    fixture itself is checked, independent of any matrix code."""
    g = json.load(open(GOLD))
    # step 1: S0 = 0, k1 = (1,0), v1 = (1,2), beta1 = 1/2 -> r = v1
    S1 = [[0.5 * 1 * 1, 0.5 * 1 * 0], [0.5 * 2 * 1, 0.5 * 2 * 0]]
    assert np.allclose(S1, g["S1"], atol=0)
    # step 2: S1 k2 = (0.3, 0.6), r = v2 - S1 k2 = (2.7, -1.6), beta2 = 1
    r = [3 - 0.3, -1 - 0.6]
    S2 = [[S1[0][0] + r[0] * 0.6, S1[0][1] + r[0] * 0.8],
          [S1[1][0] + r[1] * 0.6, S1[1][1] + r[1] * 0.8]]
    assert np.allclose(S2, g["S2"], atol=1e-15)
    assert np.allclose([S1[0][0], S1[1][0]], g["o"][0], atol=0)      # S1 q1
    assert np.allclose([S2[0][1], S2[1][1]], g["o"][1], atol=1e-15)  # S2 q2


def test_golden_forward():
    g = json.load(open(GOLD))
    o, hT = _fwd(np.array(g["q"]), np.array(g["k"]), np.array(g["v"]),
                 np.array(g["beta"]))
    assert np.abs(o - np.array(g["o"])).max() <= 1e-14
    assert np.abs(hT.T - np.array(g["S2"])).max() <= 1e-14


@pytest.mark.parametrize("l2", [False, True])
def test_golden_backward(l2):
    g = json.load(open(GOLD))
    dq, dk, dv, db, dh0 = _bwd(np.array(g["q"]), np.array(g["k"]), np.array(g["v"]),
                               np.array(g["beta"]), np.array(g["dO"]), l2norm=l2)
    ref = g["l2_off"]
    want_dq = g["l2_on"]["dq"] if l2 else ref["dq"]
    want_dk = g["l2_on"]["dk"] if l2 else ref["dk"]
    assert np.abs(dq - want_dq).max() <= 1e-14
    assert np.abs(dk - want_dk).max() <= 1e-14
    assert np.abs(dv - ref["dv"]).max() <= 1e-14
    assert np.abs(db - ref["dbeta"]).max() <= 1e-14
    assert np.abs(dh0.T - np.array(ref["dS0"])).max() <= 1e-14


def test_golden_ut_wy():
    """UT transform (Eq. 10-11) and WY P (Eq. 6) on the fixture's chunk C=2."""
    g = json.load(open(GOLD))
    K, V, b = np.array(g["k"]), np.array(g["v"]), np.array(g["beta"])
    Tinv = forms.ut_inverse(K, b)
    _, W, U = forms.ut_transform(K, V, b)
    assert np.abs(Tinv - g["Tinv_C2"]).max() <= 1e-15
    assert np.abs(W - g["W_C2"]).max() <= 1e-15
    assert np.abs(U - g["U_C2"]).max() <= 1e-15
    P = np.eye(2) - W.T @ K
    assert np.abs(P - g["P_C2"]).max() <= 1e-15
    assert np.abs(forms.householder_product(K, b) - P).max() <= 1e-15


# --------------------------------------------------------------------------
# Invariants and closed forms stated by the paper
# --------------------------------------------------------------------------

def test_beta_zero_leaves_memory_unmodified():
    """P:96 'when beta_t = 0, the memory remains unmodified'."""
    rng = np.random.default_rng(1)
    q, k, v, _ = _rand_unit(rng, 37, 8, 5)
    h0 = rng.standard_normal((8, 5))
    o, hT = _fwd(q, k, v, np.zeros(37), h0=h0)
    assert np.array_equal(hT, h0)
    assert np.abs(o - q @ h0).max() <= 1e-14       # o_t = S_0 q_t
    o0, hT0 = _fwd(q, k, v, np.zeros(37))
    assert not o0.any() and not hT0.any()


def test_orthonormal_keys_retrieve_exactly():
    """P:96 / P:331: beta = 1 with unit keys writes v exactly; orthonormal keys
    do not interfere, so querying k_j returns v_j."""
    rng = np.random.default_rng(2)
    d = 16
    Qm, _ = np.linalg.qr(rng.standard_normal((d, d)))
    K = Qm.T[:10]
    V = rng.standard_normal((10, 6))
    q = np.vstack([K, K])                    # after all writes, read each key
    k = np.vstack([K, np.zeros((10, d))])
    v = np.vstack([V, np.zeros((10, 6))])
    beta = np.concatenate([np.ones(10), np.zeros(10)])
    o, _ = _fwd(q, k, v, beta)
    assert np.abs(o[10:] - V).max() <= 1e-12


def test_rebinding_overwrites():
    """with beta = 1 the old value is completely removed."""
    rng = np.random.default_rng(3)
    kk = rng.standard_normal(12); kk /= np.linalg.norm(kk)
    va, vb = rng.standard_normal(4), rng.standard_normal(4)
    q = np.vstack([kk, kk]); k = q.copy(); v = np.vstack([va, vb])
    o, _ = _fwd(q, k, v, np.ones(2))
    assert np.abs(o[1] - vb).max() <= 1e-12
    assert np.abs(o[0] - va).max() <= 1e-12


def test_single_step_closed_form():
    """P:117 base case u_1 = beta_1 v_1, so o_1 = beta_1 (k_1 . q_1) v_1; its
    gradients are the closed forms of SURVEY §8c (L=1)."""
    rng = np.random.default_rng(4)
    q, k, v, b = rng.standard_normal((1, 7)), rng.standard_normal((1, 7)), \
        rng.standard_normal((1, 3)), np.array([0.3])
    do = rng.standard_normal((1, 3))
    o, _ = _fwd(q, k, v, b)
    kq = float(k[0] @ q[0]); vd = float(v[0] @ do[0])
    assert np.abs(o[0] - b[0] * kq * v[0]).max() <= 1e-14
    dq, dk, dv, db, _ = _bwd(q, k, v, b, do)
    assert np.abs(dv[0] - b[0] * kq * do[0]).max() <= 1e-14
    assert abs(db[0] - kq * vd) <= 1e-14
    assert np.abs(dq[0] - b[0] * vd * k[0]).max() <= 1e-14
    assert np.abs(dk[0] - b[0] * vd * q[0]).max() <= 1e-14


def test_l2_normalisation_and_eps_guard():
    """P:329-331 L2 norm; reading R9 (x / max(||x||, eps)): scaling the raw
    q, k leaves the output unchanged, zero rows stay zero (no NaN)."""
    rng = np.random.default_rng(5)
    q, k, v, b = _rand_unit(rng, 20, 8, 4, unit_keys=False)
    o1, h1 = _fwd(q, k, v, b, l2norm=True)
    o2, h2 = _fwd(3.7 * q, 0.2 * k, v, b, l2norm=True)
    assert np.abs(o1 - o2).max() <= 1e-13 and np.abs(h1 - h2).max() <= 1e-13
    qn = q / np.linalg.norm(q, axis=1, keepdims=True)
    kn = k / np.linalg.norm(k, axis=1, keepdims=True)
    o3, _ = _fwd(qn, kn, v, b, l2norm=False)
    assert np.abs(o1 - o3).max() <= 1e-13
    q[3] = 0; k[5] = 0
    o4, _ = _fwd(q, k, v, b, l2norm=True)
    assert np.isfinite(o4).all() and not o4[3].any()


def test_transition_eigenstructure():
    """P:330-331 (reading R7): for unit k, I - beta k k^T fixes k-perp and
    scales k by 1 - beta; at beta = 1 it is a projection.  Checked through the
    oracle: one step from S_0 = h0 with v = 0 is S_0 (I - beta k k^T)."""
    rng = np.random.default_rng(6)
    d = 9
    kk = rng.standard_normal(d); kk /= np.linalg.norm(kk)
    for beta in (0.0, 0.37, 1.0):
        h0 = np.eye(d)                         # S_0 = I -> S_1 = I - beta k k^T
        _, hT = _fwd(np.zeros((1, d)), kk[None], np.zeros((1, d)), np.array([beta]), h0=h0)
        M = hT.T
        assert np.abs(M @ kk - (1 - beta) * kk).max() <= 1e-14
        perp = rng.standard_normal(d); perp -= (perp @ kk) * kk
        assert np.abs(M @ perp - perp).max() <= 1e-14
        if beta == 1.0:
            assert np.abs(M @ M - M).max() <= 1e-14


# --------------------------------------------------------------------------
# The paper's other forms of the same computation
# --------------------------------------------------------------------------

@pytest.mark.parametrize("C", [1, 4, 8, 16, 32, 96])
def test_chunkwise_equals_recurrence(C):
    """Eq. 8-9 + Eq. 10-11 (chunkwise, forms.py) == §2.2 recurrence (oracle) for
    every chunk size; C = 1 is the recurrent form, C = L the parallel one.
    L = 96 is not a multiple of 32 (ragged tail, reading R14)."""
    rng = np.random.default_rng(10 + C)
    q, k, v, b = _rand_unit(rng, 96, 12, 7)
    h0 = 0.3 * rng.standard_normal((12, 7))
    o, hT = _fwd(q, k, v, b, h0=h0)
    oc, hc = forms.chunkwise_forward(q, k, v, b, C, S0=h0.T)
    assert np.abs(o - oc).max() <= 1e-12
    assert np.abs(hT - hc.T).max() <= 1e-12


def test_parallel_form_equals_recurrence():
    """P:258-262 fully parallel form A = (QK^T . M) T (reading R8)."""
    rng = np.random.default_rng(20)
    q, k, v, b = _rand_unit(rng, 40, 10, 6)
    A, Op = forms.parallel_form(q, k, v, b)
    o, _ = _fwd(q, k, v, b)
    assert np.abs(o - Op).max() <= 1e-12
    assert not np.triu(A, 1).any()


def test_wy_ut_householder_agree():
    """Eq. 7 (recursive w, u) == Eq. 10-11 (UT); P = I - sum w k^T (Eq. 6) ==
    ordered Householder product (Eq. 4); S from zero = sum u k^T (Eq. 6)."""
    rng = np.random.default_rng(21)
    q, k, v, b = _rand_unit(rng, 24, 16, 5)
    Wr, Ur = forms.wy_recursive(k, v, b)
    T, W, U = forms.ut_transform(k, v, b)
    assert np.abs(Wr - W).max() <= 1e-12 and np.abs(Ur - U).max() <= 1e-12
    assert np.allclose(np.diag(T), b, atol=0, rtol=1e-15)   # diag(T) = beta (R1)
    P = np.eye(16) - W.T @ k
    assert np.abs(P - forms.householder_product(k, b)).max() <= 1e-12
    _, hT = _fwd(q, k, v, b)
    assert np.abs(hT.T - U.T @ k).max() <= 1e-12
    # substitution == explicit inverse
    Ti = forms.ut_inverse(k, b)
    Lm = np.tril((k * b[:, None]) @ k.T, -1)
    assert np.abs(Ti - np.linalg.inv(np.eye(24) + Lm)).max() <= 1e-12


def test_streaming_split_equals_whole():
    """h0 / hT streaming (reading R13): two halves == the whole sequence."""
    rng = np.random.default_rng(22)
    q, k, v, b = _rand_unit(rng, 50, 8, 8)
    o, hT = _fwd(q, k, v, b)
    o1, h1 = _fwd(q[:23], k[:23], v[:23], b[:23])
    o2, h2 = _fwd(q[23:], k[23:], v[23:], b[23:], h0=h1)
    assert np.abs(np.vstack([o1, o2]) - o).max() <= 1e-13
    assert np.abs(h2 - hT).max() <= 1e-13


def test_padding_is_noop():
    """Reading R14: appending beta = 0, zero rows changes nothing."""
    rng = np.random.default_rng(23)
    q, k, v, b = _rand_unit(rng, 30, 8, 8)
    o, hT = _fwd(q, k, v, b)
    z = np.zeros((5, 8))
    op, hp = _fwd(np.vstack([q, z]), np.vstack([k, z]), np.vstack([v, z]),
                  np.concatenate([b, np.zeros(5)]))
    assert np.array_equal(op[:30], o) and np.array_equal(hp, hT)
    assert not op[30:].any()


# --------------------------------------------------------------------------
# Backward: finite differences, chunkwise adjoint, linearity
# --------------------------------------------------------------------------

def _loss(q, k, v, b, dO, h0, dhT, l2):
    o, hT = _fwd(q, k, v, b, h0=h0, l2norm=l2)
    return float((o * dO).sum() + (hT * dhT).sum())


@pytest.mark.parametrize("l2", [False, True])
def test_backward_matches_finite_differences(l2):
    """Central differences (h = 1e-6) of <O, dO> + <hT, dhT> w.r.t. every raw
    input (q, k, v, beta, h0); rel <= 1e-6 above 1e-8, abs <= 1e-8 below."""
    rng = np.random.default_rng(30 + l2)
    L, dk, dv = 9, 5, 4
    q, k, v, b = _rand_unit(rng, L, dk, dv, unit_keys=not l2)
    if l2:
        q *= 1.7; k *= 0.8
    h0 = 0.5 * rng.standard_normal((dk, dv))
    dO = rng.standard_normal((L, dv))
    dhT = rng.standard_normal((dk, dv))
    dq, dk_, dv_, db, dh0 = _bwd(q, k, v, b, dO, h0=h0, dhT=dhT, l2norm=l2)
    args = [q, k, v, b, h0]
    grads = [dq, dk_, dv_, db, dh0]
    eps = 1e-6
    for ai, (a, g) in enumerate(zip(args, grads)):
        num = np.zeros_like(a)
        for idx in np.ndindex(a.shape):
            ap = [x.copy() for x in args]; am = [x.copy() for x in args]
            ap[ai][idx] += eps; am[ai][idx] -= eps
            num[idx] = (_loss(*ap[:4], dO, ap[4], dhT, l2) -
                        _loss(*am[:4], dO, am[4], dhT, l2)) / (2 * eps)
        big = np.abs(num) > 1e-8
        assert np.all(np.abs(g - num)[~big] <= 1e-8)
        rel = np.abs(g - num)[big] / np.abs(num)[big]
        assert rel.max(initial=0) <= 1e-6, (ai, rel.max())


@pytest.mark.parametrize("C", [1, 4, 8, 32])
def test_chunkwise_backward_equals_bptt(C):
    """SURVEY App. A.2 (the chunked reverse sweep the GPU kernels implement)
    == the oracle's token-level BPTT, including dh0 with a nonzero h0/dhT."""
    rng = np.random.default_rng(40 + C)
    L, dk, dv = 32, 8, 6
    q, k, v, b = _rand_unit(rng, L, dk, dv)
    h0 = 0.4 * rng.standard_normal((dk, dv))
    dO = rng.standard_normal((L, dv)); dhT = rng.standard_normal((dk, dv))
    ref = _bwd(q, k, v, b, dO, h0=h0, dhT=dhT)
    got = forms.chunkwise_backward(q, k, v, b, dO, C, S0=h0, dST=dhT)
    for r, g in zip(ref, got):
        assert np.abs(r - g).max() <= 1e-12


@pytest.mark.parametrize("l2", [False, True])
def test_backward_checkpoint_segments_finite_differences(l2):
    """The oracle's backward re-derives S_{t-1} from checkpoints every 64
    tokens (deltanet_oracle.c CKPT).  L = 150 = 64 + 64 + 22 walks three
    checkpoint segments with a ragged last one; central differences of
    <O, dO> + <hT, dhT> w.r.t. every input pin that path (rel <= 1e-6 above
    1e-8, abs <= 1e-8 below), with h0 and dhT nonzero."""
    rng = np.random.default_rng(130 + l2)
    L, dk, dv = 150, 3, 2
    q, k, v, b = _rand_unit(rng, L, dk, dv, unit_keys=not l2)
    if l2:
        q *= 1.3; k *= 0.7
    h0 = 0.5 * rng.standard_normal((dk, dv))
    dO = rng.standard_normal((L, dv))
    dhT = rng.standard_normal((dk, dv))
    grads = _bwd(q, k, v, b, dO, h0=h0, dhT=dhT, l2norm=l2)
    args = [q, k, v, b, h0]
    # h = 1e-5: at L = 150 the loss is O(10^2), so the rounding floor of a
    # central difference, ~1e-16 |loss| / h, must stay below the bar; the
    # truncation error is O(h^2).  Bar: |g - num| <= 1e-6 |num| + 1e-9 max|num|
    eps = 1e-5
    for ai, (a, g) in enumerate(zip(args, grads)):
        num = np.zeros_like(a)
        for idx in np.ndindex(a.shape):
            ap = [x.copy() for x in args]; am = [x.copy() for x in args]
            ap[ai][idx] += eps; am[ai][idx] -= eps
            num[idx] = (_loss(*ap[:4], dO, ap[4], dhT, l2) -
                        _loss(*am[:4], dO, am[4], dhT, l2)) / (2 * eps)
        err = np.abs(g - num)
        bar = 1e-6 * np.abs(num) + 1e-9 * np.abs(num).max()
        assert np.all(err <= bar), (ai, (err / np.maximum(np.abs(num), 1e-300)).max())


@pytest.mark.parametrize("L,C", [(160, 16), (192, 64), (135, 5), (131, 1)])
def test_backward_checkpoint_segments_equal_chunkwise_adjoint(L, C):
    """Three or more checkpoint segments (L > 128; 160, 135, 131 ragged) at d = 16: the
    oracle's BPTT == the independent chunked adjoint of SURVEY App. A.2
    (oracle/forms.py::chunkwise_backward), every output incl. dh0."""
    rng = np.random.default_rng(200 + L + C)
    dk, dv = 16, 12
    q, k, v, b = _rand_unit(rng, L, dk, dv)
    h0 = 0.4 * rng.standard_normal((dk, dv))
    dO = rng.standard_normal((L, dv)); dhT = rng.standard_normal((dk, dv))
    ref = _bwd(q, k, v, b, dO, h0=h0, dhT=dhT)
    got = forms.chunkwise_backward(q, k, v, b, dO, C, S0=h0, dST=dhT)
    for r, g in zip(ref, got):
        assert np.abs(r - g).max() <= 1e-11 * max(1.0, np.abs(r).max())


def test_l2_adjoint_eps_branch_finite_differences():
    """Reading R9: below ||x|| = eps the normalisation divides by the constant
    eps, so the adjoint is dx = dy / eps.  Rows of q and k scaled to ~1e-8
    (and one exactly zero) stay inside that branch under the FD step; the
    oracle's gradients of those rows match central differences."""
    rng = np.random.default_rng(77)
    L, dk, dv = 12, 4, 3
    q, k, v, b = _rand_unit(rng, L, dk, dv, unit_keys=False)
    q[3] *= 1e-8 / np.linalg.norm(q[3])
    k[5] *= 2e-8 / np.linalg.norm(k[5])
    q[7] = 0.0
    k[9] = 0.0
    h0 = 0.5 * rng.standard_normal((dk, dv))
    dO = rng.standard_normal((L, dv)); dhT = rng.standard_normal((dk, dv))
    dq, dk_, _, _, _ = _bwd(q, k, v, b, dO, h0=h0, dhT=dhT, l2norm=True)
    h = 1e-10   # keeps ||x|| < 1e-6 (the eps of R9)
    for which, rows in ((0, (3, 7)), (1, (5, 9))):
        g = (dq, dk_)[which]
        for r in rows:
            for j in range(dk):
                ap = [q.copy(), k.copy()]; am = [q.copy(), k.copy()]
                ap[which][r, j] += h; am[which][r, j] -= h
                num = (_loss(ap[0], ap[1], v, b, dO, h0, dhT, True) -
                       _loss(am[0], am[1], v, b, dO, h0, dhT, True)) / (2 * h)
                assert abs(g[r, j] - num) <= 1e-5 * max(1.0, abs(num)), (which, r, j)
    # and the branch really is the constant-divisor one: a 2x larger tiny row
    # has the same gradient (dx = dy / eps does not depend on ||x||)
    q2 = q.copy(); q2[3] *= 2.0
    dq2 = _bwd(q2, k, v, b, dO, h0=h0, dhT=dhT, l2norm=True)[0]
    ratio = np.abs(dq2[3]).max() / np.abs(dq[3]).max()
    assert 0.5 < ratio < 2.0   # dy changes only through o, not through 1/||x||


def test_backward_linear_in_cotangent_and_zero():
    rng = np.random.default_rng(50)
    q, k, v, b = _rand_unit(rng, 17, 6, 6, unit_keys=False)
    dO = rng.standard_normal((17, 6))
    g1 = _bwd(q, k, v, b, dO, l2norm=True)
    g2 = _bwd(q, k, v, b, 2.5 * dO, l2norm=True)
    for a, c in zip(g1, g2):
        assert np.abs(2.5 * a - c).max() <= 1e-12 * max(1.0, np.abs(c).max())
    for a in _bwd(q, k, v, b, 0 * dO, l2norm=True):
        assert not a.any()


def test_multi_unit_threads_match_single():
    """Units are independent; the threaded oracle returns the same bits."""
    rng = np.random.default_rng(60)
    B, H, L, d = 2, 3, 70, 6
    q = rng.standard_normal((B, H, L, d)); k = rng.standard_normal((B, H, L, d))
    v = rng.standard_normal((B, H, L, d)); b = rng.random((B, H, L))
    dO = rng.standard_normal((B, H, L, d))
    o1, h1 = oracle.recurrent_fwd(q, k, v, b, nthreads=1)
    o4, h4 = oracle.recurrent_fwd(q, k, v, b, nthreads=4)
    assert np.array_equal(o1, o4) and np.array_equal(h1, h4)
    g1 = oracle.recurrent_bwd(q, k, v, b, dO, nthreads=1)
    g4 = oracle.recurrent_bwd(q, k, v, b, dO, nthreads=5)
    for a, c in zip(g1, g4):
        assert np.array_equal(a, c)
    # unit (1,2) alone
    ou, _ = oracle.recurrent_fwd(q[1:2, 2:3], k[1:2, 2:3], v[1:2, 2:3], b[1:2, 2:3])
    assert np.array_equal(ou[0, 0], o1[1, 2])
