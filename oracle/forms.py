"""The paper's other forms of the delta rule, fp64 numpy -- TEST INFRASTRUCTURE.

Each function restates one passage of PAPER.md for ONE (batch, head) unit,
in the paper's orientation (S is d_v x d_k, o_t = S_t q_t) unless noted.
They exist only to pin the recurrent oracle (tests/test_oracle.py): two
independent codings of the same mathematics must agree to rounding.

Inputs are already normalised (callers pass unit-norm keys when the test
needs them); chunk sizes must divide L here except where noted.
"""
from __future__ import annotations

import numpy as np


def householder_product(K, beta):
    """P = prod_{t=1..n} (I - beta_t k_t k_t^T), left to right.
    PAPER.md §3.2 Eq. 4 (lines 138-141) and the P_i^j definition (line 143)."""
    n, d = K.shape
    P = np.eye(d)
    for t in range(n):
        P = P @ (np.eye(d) - beta[t] * np.outer(K[t], K[t]))
    return P


def wy_recursive(K, V, beta):
    """Eq. 7: the sequential WY recursions
    w_r = beta_r (k_r - sum_{i<r} w_i (k_i^T k_r)),
    u_r = beta_r (v_r - sum_{i<r} u_i (k_i^T k_r))."""
    C = K.shape[0]
    W = np.zeros_like(K)
    U = np.zeros_like(V)
    for r in range(C):
        w = K[r].copy()
        u = V[r].copy()
        for i in range(r):
            kk = K[i] @ K[r]
            w -= W[i] * kk
            u -= U[i] * kk
        W[r] = beta[r] * w
        U[r] = beta[r] * u
    return W, U


def ut_inverse(K, beta):
    """(I + tril(diag(beta) K K^T, -1))^{-1} by forward substitution, the loop
    of Listing 1 applied to ONE chunk (reading R3):
        T = -(K_beta K^T).tril(-1)
        for i in 1..C-1:  T[i,:i] += sum_m T[i,m] T[m,:i]
        T += I
    """
    C = K.shape[0]
    Kb = K * beta[:, None]
    T = -np.tril(Kb @ K.T, -1)
    for i in range(1, C):
        T[i, :i] = T[i, :i] + (T[i, :, None] * T[:, :i]).sum(-2)
    return T + np.eye(C)


def ut_transform(K, V, beta):
    """Eq. 10-11: T = (I + tril(diag(b)KK^T,-1))^{-1} diag(b),
    W = T K, U = T V.  Returns (T, W, U) with the paper's T (diag(beta) inside;
    reading R1)."""
    T = ut_inverse(K, beta) * beta[None, :]
    return T, T @ K, T @ V


def chunkwise_forward(Q, K, V, beta, C, S0=None):
    """Eq. 8-9 with W, U from Eq. 10-11, written as in
    Listing 1 (lines 1108-1117) but per chunk and with an optional initial
    state.  The listing's S is d_k x d_v (= S^T of §2.2); we keep that
    orientation internally and return O and S_final^T.
    Mask: inclusive tril for QK^T (reading R4).  L need not divide C: the tail
    is zero-padded with beta = 0 (reading R14)."""
    L, dk = K.shape
    dv = V.shape[1]
    pad = (-L) % C
    if pad:
        Q = np.vstack([Q, np.zeros((pad, dk))])
        K = np.vstack([K, np.zeros((pad, dk))])
        V = np.vstack([V, np.zeros((pad, dv))])
        beta = np.concatenate([beta, np.zeros(pad)])
    S = np.zeros((dk, dv)) if S0 is None else S0.T.copy()  # listing orientation
    O = np.zeros((L + pad, dv))
    for c in range((L + pad) // C):
        sl = slice(c * C, (c + 1) * C)
        q, k, v, b = Q[sl], K[sl], V[sl], beta[sl]
        _, w, u = ut_transform(k, v, b)
        u = u - w @ S
        o_inter = q @ S
        A = np.tril(q @ k.T)
        O[sl] = A @ u + o_inter
        S = S + k.T @ u
    return O[:L], S.T


def parallel_form(Q, K, V, beta):
    """Fully parallel form, §3.2: A = (QK^T . M) T,
    O = A V, with T the whole-sequence UT matrix (Eq. 10; reading R8)."""
    T, _, _ = ut_transform(K, V, beta)
    A = np.tril(Q @ K.T) @ T
    return A, A @ V


def chunkwise_backward(Q, K, V, beta, dO, C, S0=None, dST=None):
    """Chunkwise reverse sweep (the paper gives no backward,
    reading R12).  Kernel orientation H = S^T (d_k x d_v).  Inputs are the
    (already normalised) q, k.  Returns dQ, dK, dV, dbeta, dH0 (H orientation).
    Used to pin the chunked backward design the GPU kernels follow against
    the recurrent BPTT oracle."""
    L, dk = K.shape
    dv = V.shape[1]
    assert L % C == 0
    n = L // C
    H = np.zeros((dk, dv)) if S0 is None else S0.copy()  # S0 given as H0 here
    Hs, Ws, Us, Ups, Ts, As = [], [], [], [], [], []
    for c in range(n):
        sl = slice(c * C, (c + 1) * C)
        q, k, v, b = Q[sl], K[sl], V[sl], beta[sl]
        Tinv = ut_inverse(k, b)
        W = Tinv @ (k * b[:, None])
        U = Tinv @ (v * b[:, None])
        Up = U - W @ H
        Hs.append(H.copy()); Ws.append(W); Ups.append(Up); Ts.append(Tinv)
        As.append(np.tril(q @ k.T))
        H = H + k.T @ Up
    dQ = np.zeros_like(Q); dK = np.zeros_like(K); dV = np.zeros_like(V)
    db = np.zeros_like(beta)
    dH = np.zeros((dk, dv)) if dST is None else dST.copy()
    for c in reversed(range(n)):
        sl = slice(c * C, (c + 1) * C)
        q, k, v, b, do = Q[sl], K[sl], V[sl], beta[sl], dO[sl]
        Ht, W, Up, Tinv, A = Hs[c], Ws[c], Ups[c], Ts[c], As[c]
        Kb, Vb = k * b[:, None], v * b[:, None]
        dUp = k @ dH + A.T @ do
        dA = np.tril(do @ Up.T)
        dq = do @ Ht.T + dA @ k
        dkk = Up @ dH.T + dA.T @ q
        dW = -dUp @ Ht.T
        dH = dH + q.T @ do - W.T @ dUp
        dTinv = dW @ Kb.T + dUp @ Vb.T
        dKb = Tinv.T @ dW
        dVb = Tinv.T @ dUp
        dkk = dkk + b[:, None] * dKb
        dV[sl] = b[:, None] * dVb
        dbc = (dKb * k).sum(1) + (dVb * v).sum(1)
        G = np.tril(-Tinv.T @ dTinv @ Tinv.T, -1)
        KK = k @ k.T
        dbc = dbc + (G * KK).sum(1)
        bG = b[:, None] * G
        dkk = dkk + bG @ k + bG.T @ k
        dQ[sl] = dq; dK[sl] = dkk; db[sl] = dbc
    return dQ, dK, dV, db, dH


# ---------------------------------------------------------------- Gated DeltaNet
def _gate_tables(g):
    """Within one chunk: G_r = sum_{j<=r} g_j, gamma_r = exp(G_r) and
    Gamma[r, i] = exp(G_r - G_i) for i <= r (0 above the diagonal), formed as
    exponentials of differences so no ratio over- or underflows."""
    G = np.cumsum(g)
    diff = G[:, None] - G[None, :]
    Gam = np.where(np.tril(np.ones_like(diff)) > 0, np.exp(np.minimum(diff, 0.0)), 0.0)
    return G, np.exp(G), Gam


def gated_chunkwise_forward(Q, K, V, beta, g, C, H0=None):
    """Chunkwise form of Gated DeltaNet (PAPER.md Table tab:overview, P:757:
    S_t = S_{t-1}(alpha_t(I - beta_t k_t k_t^T)) + beta_t v_t k_t^T, alpha = e^g)
    derived like Eq. 8-11 (R23), kernel orientation H = S^T.
    Per chunk, with G, gamma, Gamma of _gate_tables:
        X  = (I + tril(diag(beta) (Gamma . K K^T), -1))^{-1}
        W  = X diag(beta gamma) K,   U = X diag(beta) V,   U' = U - W H
        O  = diag(gamma) Q H + (Gamma . tril(Q K^T)) U'
        H <- gamma_C H + (diag(gamma_C / gamma) K)^T U'
    The tail is padded with beta = 0, g = 0 (an exact no-op).  Returns O, H."""
    L, dk = K.shape
    dv = V.shape[1]
    pad = (-L) % C
    if pad:
        Q = np.vstack([Q, np.zeros((pad, dk))])
        K = np.vstack([K, np.zeros((pad, dk))])
        V = np.vstack([V, np.zeros((pad, dv))])
        beta = np.concatenate([beta, np.zeros(pad)])
        g = np.concatenate([g, np.zeros(pad)])
    H = np.zeros((dk, dv)) if H0 is None else H0.copy()
    O = np.zeros((L + pad, dv))
    for c in range((L + pad) // C):
        sl = slice(c * C, (c + 1) * C)
        q, k, v, b = Q[sl], K[sl], V[sl], beta[sl]
        G, gam, Gam = _gate_tables(g[sl])
        X = np.linalg.inv(np.eye(C) + np.tril(b[:, None] * Gam * (k @ k.T), -1))
        W = X @ ((b * gam)[:, None] * k)
        U = X @ (b[:, None] * v)
        Up = U - W @ H
        O[sl] = gam[:, None] * (q @ H) + (Gam * np.tril(q @ k.T)) @ Up
        H = gam[-1] * H + ((gam[-1] / gam)[:, None] * k).T @ Up
    return O[:L], H


def gated_chunkwise_backward(Q, K, V, beta, g, dO, C, H0=None, dHT=None):
    """Chunked reverse sweep of gated_chunkwise_forward (R23), H
    orientation, already-normalised q, k; L a multiple of C.  Returns dQ, dK,
    dV, dbeta, dg, dH0.  Per chunk, with D = gamma_C / gamma, dH = dl/dH_next:
      dU' = diag(D) K dH + A^T dO,  A = Gamma . tril(QK^T),  dA = tril(dO U'^T)
      dQ  = diag(gamma) dO H^T + (Gamma . dA) K
      dK  = diag(D) U' dH^T + (Gamma . dA)^T Q + UT / inverse adjoints
      dH <- gamma_C dH + (diag(gamma) Q)^T dO - W^T dU'
    and dG_r (w.r.t. the cumulative log-gate) collects the gamma, Gamma and D
    factors; dg = reverse cumulative sum of dG within the chunk."""
    L, dk = K.shape
    dv = V.shape[1]
    assert L % C == 0
    n = L // C
    H = np.zeros((dk, dv)) if H0 is None else H0.copy()
    saved = []
    for c in range(n):
        sl = slice(c * C, (c + 1) * C)
        q, k, v, b = Q[sl], K[sl], V[sl], beta[sl]
        G, gam, Gam = _gate_tables(g[sl])
        X = np.linalg.inv(np.eye(C) + np.tril(b[:, None] * Gam * (k @ k.T), -1))
        W = X @ ((b * gam)[:, None] * k)
        U = X @ (b[:, None] * v)
        Up = U - W @ H
        saved.append((H.copy(), X, W, Up, G, gam, Gam))
        H = gam[-1] * H + ((gam[-1] / gam)[:, None] * k).T @ Up
    dQ = np.zeros_like(Q); dK = np.zeros_like(K); dV = np.zeros_like(V)
    db = np.zeros_like(beta); dg = np.zeros_like(g)
    dH = np.zeros((dk, dv)) if dHT is None else dHT.copy()
    for c in reversed(range(n)):
        sl = slice(c * C, (c + 1) * C)
        q, k, v, b, do = Q[sl], K[sl], V[sl], beta[sl], dO[sl]
        Ht, X, W, Up, G, gam, Gam = saved[c]
        D = gam[-1] / gam
        QK = np.tril(q @ k.T)
        A = Gam * QK
        dG = np.zeros(C)
        # H_next = gamma_C H + (D K)^T U'
        dUp = (D[:, None] * k) @ dH + A.T @ do
        dKbar = Up @ dH.T                       # w.r.t. D K
        dkk = D[:, None] * dKbar
        dD = (dKbar * k).sum(1)
        dG[-1] += (dD * D).sum() + gam[-1] * (dH * Ht).sum()
        dG -= dD * D
        # O = diag(gamma) Q H + A U'
        dA = np.tril(do @ Up.T)
        dS = Gam * dA
        dq = gam[:, None] * (do @ Ht.T) + dS @ k
        dkk = dkk + dS.T @ q
        dG += gam * (q * (do @ Ht.T)).sum(1)
        dGam = dA * QK
        # U' = U - W H
        dW = -dUp @ Ht.T
        dHn = gam[-1] * dH + (gam[:, None] * q).T @ do - W.T @ dUp
        # W = X diag(beta gamma) K, U = X diag(beta) V
        Kbg = (b * gam)[:, None] * k
        Vb = b[:, None] * v
        dX = dUp @ Vb.T + dW @ Kbg.T
        dKbg = X.T @ dW
        dVb = X.T @ dUp
        dV[sl] = b[:, None] * dVb
        dkk = dkk + (b * gam)[:, None] * dKbg
        rk = (dKbg * k).sum(1)
        dbc = (dVb * v).sum(1) + gam * rk
        dG += b * gam * rk
        # X = (I + Kg)^{-1},  Kg = tril(diag(beta) (Gamma . K K^T), -1)
        Gb = np.tril(-X.T @ dX @ X.T, -1)
        KK = k @ k.T
        dbc = dbc + (Gb * Gam * KK).sum(1)
        E = b[:, None] * Gb * Gam
        dkk = dkk + E @ k + E.T @ k
        dGam = dGam + b[:, None] * Gb * KK
        # Gamma[r, i] = exp(G_r - G_i)
        T = dGam * Gam
        dG += T.sum(1) - T.sum(0)
        dg[sl] = np.cumsum(dG[::-1])[::-1]
        dQ[sl] = dq; dK[sl] = dkk; db[sl] = dbc
        dH = dHn
    return dQ, dK, dV, db, dg, dH
