"""fp64 CPU oracle for the DeltaNet delta-rule layer -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product path (``paper_2406_06484_b200``) never imports it and shares no code
with it; the only thing both sides use is the seeded input generator in
``synth/``, which holds none of the method's arithmetic.

``recurrent_fwd`` / ``recurrent_bwd`` wrap the plain C oracle
(``deltanet_oracle.c``): the token-by-token delta rule of PAPER.md §2.2
(lines 82-97) with optional L2-normalised q, k (§3.3), and its
reverse-mode derivative (reading R12).  ``forms.py`` holds the
paper's other forms of the same computation (WY, UT, chunkwise, parallel),
used only to pin the oracle.

Parity pinned by tests/test_oracle.py (see DESIGN.md §Oracle pins).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "deltanet_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


class _Desc(ctypes.Structure):
    _fields_ = [
        ("B", ctypes.c_int), ("H", ctypes.c_int), ("L", ctypes.c_int),
        ("Dk", ctypes.c_int), ("Dv", ctypes.c_int), ("l2norm", ctypes.c_int),
        ("eps", ctypes.c_double), ("nthreads", ctypes.c_int),
    ]


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain -O2, not tuned)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c99", "-fPIC", "-shared", "-pthread",
               "-o", _LIB, _SRC, "-lm"]
        subprocess.run(cmd, check=True, cwd=_HERE)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB)
            P = ctypes.POINTER(ctypes.c_double)
            for name in ("dn_oracle_fwd",):
                fn = getattr(lib, name)
                fn.argtypes = [ctypes.POINTER(_Desc)] + [P] * 7
                fn.restype = ctypes.c_int
            lib.dn_oracle_bwd.argtypes = [ctypes.POINTER(_Desc)] + [P] * 12
            lib.dn_oracle_bwd.restype = ctypes.c_int
            lib.dn_oracle_gated_fwd.argtypes = [ctypes.POINTER(_Desc)] + [P] * 8
            lib.dn_oracle_gated_fwd.restype = ctypes.c_int
            lib.dn_oracle_gated_bwd.argtypes = [ctypes.POINTER(_Desc)] + [P] * 14
            lib.dn_oracle_gated_bwd.restype = ctypes.c_int
            _lib = lib
    return _lib


def _ptr(a):
    if a is None:
        return ctypes.POINTER(ctypes.c_double)()
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _f64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


def default_threads() -> int:
    return max(1, len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count() or 1)


def recurrent_fwd(q, k, v, beta, h0=None, l2norm=True, eps=1e-6, nthreads=None):
    """O, hT of the delta rule.  q,k [B,H,L,Dk], v [B,H,L,Dv], beta [B,H,L],
    h0 [B,H,Dk,Dv] (H = S^T, reading R2).  All upcast to fp64 exactly."""
    q, k, v, beta, h0 = map(_f64, (q, k, v, beta, h0))
    B, H, L, Dk = q.shape
    Dv = v.shape[-1]
    o = np.zeros((B, H, L, Dv))
    hT = np.zeros((B, H, Dk, Dv))
    d = _Desc(B, H, L, Dk, Dv, int(bool(l2norm)), float(eps),
              int(nthreads or default_threads()))
    rc = _load().dn_oracle_fwd(ctypes.byref(d), _ptr(q), _ptr(k), _ptr(v),
                               _ptr(beta), _ptr(h0), _ptr(o), _ptr(hT))
    if rc:
        raise RuntimeError(f"dn_oracle_fwd failed ({rc})")
    return o, hT


def recurrent_bwd(q, k, v, beta, dO, h0=None, dhT=None, l2norm=True, eps=1e-6,
                  nthreads=None):
    """dq, dk, dv, dbeta, dh0 by reverse mode through the recurrence.
    Gradients are w.r.t. the RAW q, k when l2norm (reading R10)."""
    q, k, v, beta, dO, h0, dhT = map(_f64, (q, k, v, beta, dO, h0, dhT))
    B, H, L, Dk = q.shape
    Dv = v.shape[-1]
    dq = np.zeros_like(q)
    dk = np.zeros_like(k)
    dv = np.zeros_like(v)
    db = np.zeros_like(beta)
    dh0 = np.zeros((B, H, Dk, Dv))
    d = _Desc(B, H, L, Dk, Dv, int(bool(l2norm)), float(eps),
              int(nthreads or default_threads()))
    rc = _load().dn_oracle_bwd(ctypes.byref(d), _ptr(q), _ptr(k), _ptr(v),
                               _ptr(beta), _ptr(h0), _ptr(dO), _ptr(dhT),
                               _ptr(dq), _ptr(dk), _ptr(dv), _ptr(db), _ptr(dh0))
    if rc:
        raise RuntimeError(f"dn_oracle_bwd failed ({rc})")
    return dq, dk, dv, db, dh0


def gated_fwd(q, k, v, beta, g, h0=None, l2norm=True, eps=1e-6, nthreads=None):
    """O, hT of Gated DeltaNet (PAPER.md Table tab:overview):
    S_t = S_{t-1} (alpha_t (I - beta_t k_t k_t^T)) + beta_t v_t k_t^T,
    alpha_t = exp(g_t), g [B,H,L] the log-decay (R23)."""
    q, k, v, beta, g, h0 = map(_f64, (q, k, v, beta, g, h0))
    B, H, L, Dk = q.shape
    Dv = v.shape[-1]
    o = np.zeros((B, H, L, Dv))
    hT = np.zeros((B, H, Dk, Dv))
    d = _Desc(B, H, L, Dk, Dv, int(bool(l2norm)), float(eps),
              int(nthreads or default_threads()))
    rc = _load().dn_oracle_gated_fwd(ctypes.byref(d), _ptr(q), _ptr(k), _ptr(v), _ptr(beta),
                                     _ptr(g), _ptr(h0), _ptr(o), _ptr(hT))
    if rc:
        raise RuntimeError(f"dn_oracle_gated_fwd failed ({rc})")
    return o, hT


def gated_bwd(q, k, v, beta, g, dO, h0=None, dhT=None, l2norm=True, eps=1e-6, nthreads=None):
    """dq, dk, dv, dbeta, dg, dh0 of Gated DeltaNet by reverse mode."""
    q, k, v, beta, g, dO, h0, dhT = map(_f64, (q, k, v, beta, g, dO, h0, dhT))
    B, H, L, Dk = q.shape
    Dv = v.shape[-1]
    dq, dk, dv = np.zeros_like(q), np.zeros_like(k), np.zeros_like(v)
    db, dg = np.zeros_like(beta), np.zeros_like(beta)
    dh0 = np.zeros((B, H, Dk, Dv))
    d = _Desc(B, H, L, Dk, Dv, int(bool(l2norm)), float(eps),
              int(nthreads or default_threads()))
    rc = _load().dn_oracle_gated_bwd(ctypes.byref(d), _ptr(q), _ptr(k), _ptr(v), _ptr(beta),
                                     _ptr(g), _ptr(h0), _ptr(dO), _ptr(dhT), _ptr(dq),
                                     _ptr(dk), _ptr(dv), _ptr(db), _ptr(dg), _ptr(dh0))
    if rc:
        raise RuntimeError(f"dn_oracle_gated_bwd failed ({rc})")
    return dq, dk, dv, db, dg, dh0


__all__ = ["build", "recurrent_fwd", "recurrent_bwd", "gated_fwd", "gated_bwd",
           "default_threads"]
