"""fp64 oracle of context parallelism -- TEST INFRASTRUCTURE.

Only ``tests/`` (and ``bench.py``'s reference legs) may import this module;
the product path never does.

A sequence split into consecutive parts is processed part by part, the parts
stitched by the affine composition of the delta-rule state update.  Per token
(§2.2), in the orientation H = S^T (R2),
    H_t = (I - beta_t k_t k_t^T) H_{t-1} + beta_t k_t v_t^T,
so over a part of tokens 1..n
    H_end = Psi^T H_start + Hloc,
    Psi   = (I - beta_1 k_1 k_1^T) (I - beta_2 k_2 k_2^T) ... (I - beta_n k_n k_n^T)
(the product P_1^n of the Householder factors, §3.2 Eq. 4 and the
P_i^j definition; it is symmetric factor by factor, so Psi^T is
the same product in reverse order) and Hloc the part's end state from
H_start = 0.  The reverse-mode chain of one part is the adjoint of that map,
    dl/dH_start = Psi dl/dH_end + dHloc,
dHloc = dl/dH_start with dl/dH_end = 0 (l is linear in H_start, so dHloc does
not depend on H_start).  k is L2-normalised first when ``l2norm``.

``transition`` and ``bwd_transition`` compute these for every (b, h) unit;
``state_scan`` folds gathered transitions exactly as include/deltanet.h's
deltanet_state_scan defines.  Pinned in tests/test_oracle_context.py against
the full-sequence recurrence (prefix end states, suffix cotangents, part-wise
outputs and gradients), the Householder product of oracle/forms.py, and the
linearity of H_end in H_start.
"""
from __future__ import annotations

import numpy as np

from . import recurrent_bwd, recurrent_fwd


def _normalised(k, l2norm, eps):
    k = np.asarray(k, dtype=np.float64)
    if not l2norm:
        return k
    n = np.sqrt((k * k).sum(-1, keepdims=True))
    return k / np.maximum(n, eps)


def transition(q, k, v, beta, l2norm=True, eps=1e-6):
    """(Psi [B,H,Dk,Dk], Hloc [B,H,Dk,Dv]) of the sequence q..beta [B,H,L,.]."""
    B, H, L, Dk = np.shape(k)
    kn = _normalised(k, l2norm, eps)
    b = np.asarray(beta, dtype=np.float64)
    psi = np.zeros((B, H, Dk, Dk))
    for bb in range(B):
        for hh in range(H):
            P = np.eye(Dk)
            for t in range(L):
                kt = kn[bb, hh, t]
                # P <- P (I - beta k k^T)
                P = P - b[bb, hh, t] * np.outer(P @ kt, kt)
            psi[bb, hh] = P
    _, hloc = recurrent_fwd(q, k, v, beta, l2norm=l2norm, eps=eps)
    return psi, hloc


def bwd_transition(q, k, v, beta, dO, l2norm=True, eps=1e-6):
    """dHloc [B,H,Dk,Dv]: dl/dH_start of the sequence with dl/dH_end = 0."""
    return recurrent_bwd(q, k, v, beta, dO, l2norm=l2norm, eps=eps)[4]


def state_scan(psi_all, loc_all, part, reverse=False, edge=None):
    """deltanet_state_scan of include/deltanet.h on [P,B,H,.,.] arrays:
    forward  H <- Psi_p^T H + loc_p for p = 0 .. part-1, from edge (h0);
    reverse  G <- Psi_p G + loc_p for p = P-1 down to part+1, from edge (dhT)."""
    psi_all = np.asarray(psi_all, dtype=np.float64)
    loc_all = np.asarray(loc_all, dtype=np.float64)
    P = loc_all.shape[0]
    out = np.zeros(loc_all.shape[1:]) if edge is None else np.array(edge, dtype=np.float64)
    order = range(P - 1, part, -1) if reverse else range(part)
    for p in order:
        m = psi_all[p] if reverse else np.swapaxes(psi_all[p], -1, -2)
        out = m @ out + loc_all[p]
    return out


__all__ = ["transition", "bwd_transition", "state_scan"]
