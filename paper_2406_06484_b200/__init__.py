"""B200 (sm_100a) DeltaNet chunkwise delta-rule layer -- Python binding.

Thin ctypes marshalling over ``libdeltanet.so`` (C ABI: include/deltanet.h).
Every step of the forward and backward runs in the library's CUDA kernels;
PyTorch only provides device memory and the current stream.  There is no CPU
fallback: without the built library, or without a CUDA device, every call
raises.

    o, hT, ws = deltanet_fwd(q, k, v, beta, chunk=64)
    dq, dk, dv, dbeta, dh0 = deltanet_bwd(q, k, v, beta, dO, chunk=64, workspace=ws)

Shapes: q, k [B,H,L,Dk]; v, dO [B,H,L,Dv]; beta [B,H,L]; states [B,H,Dk,Dv]
(fp32, orientation H = S^T).  dtype bf16 or fp32 (same for all I/O).
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdeltanet.so")

DELTANET_BF16 = 0
DELTANET_FP32 = 1
DELTANET_L2NORM_QK = 1 << 0
DELTANET_SAVE_STATES = 1 << 1
DELTANET_PROLOGUE_SILU_V = 1 << 3
DELTANET_FORCE_SIMT = 1 << 2
DELTANET_NO_SEGMENTS = 1 << 4
DELTANET_FORCE_SPLIT = 1 << 6
DELTANET_COMPENSATED = 1 << 7
DELTANET_GATED = 1 << 5


class deltanet_desc(ctypes.Structure):
    _fields_ = [("B", ctypes.c_int), ("H", ctypes.c_int), ("L", ctypes.c_int),
                ("Dk", ctypes.c_int), ("Dv", ctypes.c_int), ("chunk", ctypes.c_int),
                ("dtype", ctypes.c_int), ("flags", ctypes.c_uint),
                ("l2_eps", ctypes.c_float)]


EXPORTED = ("deltanet_workspace_bytes", "deltanet_fwd", "deltanet_bwd", "deltanet_path",
            "deltanet_launch_count", "deltanet_strerror", "deltanet_abi_version",
            "deltanet_recurrent_fwd", "deltanet_prologue_fwd", "deltanet_prologue_bwd",
            "deltanet_prologue_workspace_bytes", "deltanet_fwd_transition",
            "deltanet_bwd_transition", "deltanet_state_scan", "deltanet_gated_fwd",
            "deltanet_gated_bwd", "deltanet_gated_recurrent_fwd", "deltanet_fwd_bwd_host",
            "deltanet_fwd_bwd_host_device_bytes")

_lib = None


def load_library(path: str = LIB_PATH):
    """Load libdeltanet.so (raises if missing -- no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"libdeltanet.so not built ({path}); run "
                           "`python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(path)
    P = ctypes.c_void_p
    D = ctypes.POINTER(deltanet_desc)
    lib.deltanet_workspace_bytes.argtypes = [D]
    lib.deltanet_workspace_bytes.restype = ctypes.c_size_t
    lib.deltanet_fwd.argtypes = [D, P, P, P, P, P, P, P, P, ctypes.c_size_t, P]
    lib.deltanet_fwd.restype = ctypes.c_int
    lib.deltanet_bwd.argtypes = [D, P, P, P, P, P, P, P, P, P, P, P, P, P, ctypes.c_size_t, P]
    lib.deltanet_bwd.restype = ctypes.c_int
    lib.deltanet_recurrent_fwd.argtypes = [D, P, P, P, P, P, P, P, P]
    lib.deltanet_recurrent_fwd.restype = ctypes.c_int
    lib.deltanet_prologue_fwd.argtypes = [D] + [P] * 12
    lib.deltanet_prologue_fwd.restype = ctypes.c_int
    lib.deltanet_prologue_bwd.argtypes = [D] + [P] * 19 + [ctypes.c_size_t, P]
    lib.deltanet_prologue_bwd.restype = ctypes.c_int
    lib.deltanet_prologue_workspace_bytes.argtypes = [D]
    lib.deltanet_prologue_workspace_bytes.restype = ctypes.c_size_t
    lib.deltanet_fwd_transition.argtypes = [D] + [P] * 7 + [ctypes.c_size_t, P]
    lib.deltanet_fwd_transition.restype = ctypes.c_int
    lib.deltanet_bwd_transition.argtypes = [D] + [P] * 7 + [ctypes.c_size_t, P]
    lib.deltanet_bwd_transition.restype = ctypes.c_int
    lib.deltanet_state_scan.argtypes = [D, ctypes.c_int, ctypes.c_int, ctypes.c_int] + [P] * 5
    lib.deltanet_state_scan.restype = ctypes.c_int
    lib.deltanet_gated_fwd.argtypes = [D] + [P] * 9 + [ctypes.c_size_t, P]
    lib.deltanet_gated_fwd.restype = ctypes.c_int
    lib.deltanet_gated_bwd.argtypes = [D] + [P] * 15 + [ctypes.c_size_t, P]
    lib.deltanet_gated_bwd.restype = ctypes.c_int
    lib.deltanet_gated_recurrent_fwd.argtypes = [D] + [P] * 9
    lib.deltanet_gated_recurrent_fwd.restype = ctypes.c_int
    lib.deltanet_fwd_bwd_host.argtypes = [D] + [P] * 10 + [ctypes.c_int, P, ctypes.c_size_t, P]
    lib.deltanet_fwd_bwd_host.restype = ctypes.c_int
    lib.deltanet_fwd_bwd_host_device_bytes.argtypes = [D, ctypes.c_int]
    lib.deltanet_fwd_bwd_host_device_bytes.restype = ctypes.c_size_t
    lib.deltanet_path.argtypes = [D]
    lib.deltanet_path.restype = ctypes.c_int
    lib.deltanet_launch_count.argtypes = [D, ctypes.c_int]
    lib.deltanet_launch_count.restype = ctypes.c_int
    lib.deltanet_strerror.argtypes = [ctypes.c_int]
    lib.deltanet_strerror.restype = ctypes.c_char_p
    lib.deltanet_abi_version.argtypes = []
    lib.deltanet_abi_version.restype = ctypes.c_int
    _lib = lib
    return lib


class DeltaNetError(RuntimeError):
    pass


def deltanet_strerror(code: int) -> str:
    return load_library().deltanet_strerror(int(code)).decode()


def _check(rc: int, what: str):
    if rc != 0:
        raise DeltaNetError(f"{what}: {deltanet_strerror(rc)} (code {rc})")


def make_desc(B, H, L, Dk, Dv, chunk=64, dtype=torch.bfloat16, l2norm=True,
              save_states=True, force_simt=False, eps=1e-6, segments=True,
              gated=False, force_split=False, extra_flags=0) -> deltanet_desc:
    dt = {torch.bfloat16: DELTANET_BF16, torch.float32: DELTANET_FP32}[dtype]
    flags = ((DELTANET_L2NORM_QK if l2norm else 0) |
             (DELTANET_SAVE_STATES if save_states else 0) |
             (DELTANET_FORCE_SIMT if force_simt else 0) |
             (0 if segments else DELTANET_NO_SEGMENTS) |
             (DELTANET_GATED if gated else 0) |
             (DELTANET_FORCE_SPLIT if force_split else 0) | int(extra_flags))
    return deltanet_desc(B, H, L, Dk, Dv, chunk, dt, flags, eps)


def _desc_for(q, v, chunk, l2norm, save_states, force_simt, eps, segments=True, gated=False,
              force_split=False, extra_flags=0):
    B, H, L, Dk = q.shape
    return make_desc(B, H, L, Dk, v.shape[-1], chunk, q.dtype, l2norm, save_states,
                     force_simt, eps, segments, gated, force_split, extra_flags)


def deltanet_workspace_bytes(desc: deltanet_desc) -> int:
    return int(load_library().deltanet_workspace_bytes(ctypes.byref(desc)))


def deltanet_path(desc: deltanet_desc) -> int:
    return int(load_library().deltanet_path(ctypes.byref(desc)))


def deltanet_launch_count(desc: deltanet_desc, which: int) -> int:
    return int(load_library().deltanet_launch_count(ctypes.byref(desc), int(which)))


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _need(t, name, dtype, device):
    if t is None:
        return
    if not t.is_cuda:
        raise DeltaNetError(f"{name} must be a CUDA tensor (no CPU path)")
    if t.dtype != dtype:
        raise DeltaNetError(f"{name} has dtype {t.dtype}, expected {dtype}")
    if t.device != device:
        raise DeltaNetError(f"{name} on {t.device}, expected {device}")
    if not t.is_contiguous():
        raise DeltaNetError(f"{name} must be contiguous")


def _need_out(t, name, shape, dtype, device):
    """An output buffer (out=...) is written by TMA / plain stores of the
    library: check dtype, device, contiguity and the exact shape first."""
    _need(t, name, dtype, device)
    if t is not None and tuple(t.shape) != tuple(shape):
        raise DeltaNetError(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")


def _need_inputs(q, k, v, beta, dO=None):
    B, H, L, Dk = q.shape
    if tuple(k.shape) != (B, H, L, Dk) or v.dim() != 4 or tuple(v.shape[:3]) != (B, H, L) \
            or tuple(beta.shape) != (B, H, L) or (dO is not None and dO.shape != v.shape):
        raise DeltaNetError("shape mismatch: q, k [B,H,L,Dk], v, dO [B,H,L,Dv], beta [B,H,L]")


def alloc_workspace(desc: deltanet_desc, device) -> torch.Tensor:
    n = deltanet_workspace_bytes(desc)
    return torch.empty(max(n, 16), dtype=torch.uint8, device=device)


def _stream(device):
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def deltanet_fwd(q, k, v, beta, *, chunk=64, l2norm=True, h0=None, save_states=True,
                 workspace=None, want_hT=True, force_simt=False, eps=1e-6, out=None,
                 segments=True, force_split=False, extra_flags=0):
    """Forward of the chunkwise delta rule (§3.2 Eq. 8-11).
    ``segments=False`` forbids the segment-parallel forward;
    ``force_split`` selects the split tcgen05 kernels at d = 128 (§4.10).
    Returns (o, hT or None, workspace)."""
    lib = load_library()
    dev = q.device
    for t, n in ((q, "q"), (k, "k"), (v, "v"), (beta, "beta")):
        _need(t, n, q.dtype, dev)
    _need(h0, "h0", torch.float32, dev)
    _need_inputs(q, k, v, beta)
    d = _desc_for(q, v, chunk, l2norm, save_states, force_simt, eps, segments,
                  force_split=force_split, extra_flags=extra_flags)
    B, H, L, Dk = q.shape
    Dv = v.shape[-1]
    _need_out(h0, "h0", (B, H, Dk, Dv), torch.float32, dev)
    _need_out(out, "out", (B, H, L, Dv), q.dtype, dev)
    o = out if out is not None else torch.empty((B, H, L, Dv), dtype=q.dtype, device=dev)
    hT = torch.empty((B, H, Dk, Dv), dtype=torch.float32, device=dev) if want_hT else None
    if workspace is None:
        workspace = alloc_workspace(d, dev)
    _need(workspace, "workspace", torch.uint8, dev)
    rc = lib.deltanet_fwd(ctypes.byref(d), _ptr(q), _ptr(k), _ptr(v), _ptr(beta), _ptr(h0),
                          _ptr(o), _ptr(hT), _ptr(workspace), workspace.numel(), _stream(dev))
    _check(rc, "deltanet_fwd")
    return o, hT, workspace


def deltanet_recurrent_fwd(q, k, v, beta, *, l2norm=True, h0=None, want_hT=True, eps=1e-6,
                           out=None, hT=None):
    """Recurrent (token-by-token) forward for inference / decode (PAPER.md
    §2.2; include/deltanet.h deltanet_recurrent_fwd).  Passing
    hT=h0 updates the state in place.  Returns (o, hT or None)."""
    lib = load_library()
    dev = q.device
    for t, n in ((q, "q"), (k, "k"), (v, "v"), (beta, "beta")):
        _need(t, n, q.dtype, dev)
    _need(h0, "h0", torch.float32, dev)
    _need(hT, "hT", torch.float32, dev)
    _need_inputs(q, k, v, beta)
    B, H, L, Dk = q.shape
    Dv = v.shape[-1]
    for t, n in ((h0, "h0"), (hT, "hT")):
        _need_out(t, n, (B, H, Dk, Dv), torch.float32, dev)
    _need_out(out, "out", (B, H, L, Dv), q.dtype, dev)
    d = make_desc(B, H, L, Dk, Dv, 64, q.dtype, l2norm=l2norm, eps=eps)
    o = out if out is not None else torch.empty((B, H, L, Dv), dtype=q.dtype, device=dev)
    if hT is None and want_hT:
        hT = torch.empty((B, H, Dk, Dv), dtype=torch.float32, device=dev)
    rc = lib.deltanet_recurrent_fwd(ctypes.byref(d), _ptr(q), _ptr(k), _ptr(v), _ptr(beta),
                                    _ptr(h0), _ptr(o), _ptr(hT), _stream(dev))
    _check(rc, "deltanet_recurrent_fwd")
    return o, hT


def _prologue_desc(xq, xv, silu_v):
    B, L, H, Dk = xq.shape
    Dv = xv.shape[-1]
    d = make_desc(B, H, L, Dk, Dv, 64, xq.dtype, l2norm=False, save_states=False)
    if silu_v:
        d.flags |= DELTANET_PROLOGUE_SILU_V
    return d


def deltanet_prologue_fwd(xq, xk, xv, xb, wq, wk, wv, *, silu_v=False, out=None):
    """Layer prologue (include/deltanet.h deltanet_prologue_fwd; PAPER.md
    P:96): short causal conv (width 4) + SiLU on
    q, k, sigmoid on beta, [B, L, H, D] -> [B, H, L, D].  Returns (q, k, v, beta)."""
    lib = load_library()
    dev = xq.device
    for t, n in ((xq, "xq"), (xk, "xk"), (xv, "xv"), (xb, "xb")):
        _need(t, n, xq.dtype, dev)
    for t, n in ((wq, "wq"), (wk, "wk"), (wv, "wv")):
        _need(t, n, torch.float32, dev)
    B, L, H, Dk = xq.shape
    Dv = xv.shape[-1]
    d = _prologue_desc(xq, xv, silu_v)
    if out is not None:
        for t, n, shp in zip(out, ("q", "k", "v", "beta"),
                             ((B, H, L, Dk), (B, H, L, Dk), (B, H, L, Dv), (B, H, L))):
            _need_out(t, n, shp, xq.dtype, dev)
    if out is None:
        out = (torch.empty((B, H, L, Dk), dtype=xq.dtype, device=dev),
               torch.empty((B, H, L, Dk), dtype=xq.dtype, device=dev),
               torch.empty((B, H, L, Dv), dtype=xq.dtype, device=dev),
               torch.empty((B, H, L), dtype=xq.dtype, device=dev))
    rc = lib.deltanet_prologue_fwd(ctypes.byref(d), _ptr(xq), _ptr(xk), _ptr(xv), _ptr(xb),
                                   _ptr(wq), _ptr(wk), _ptr(wv), *[_ptr(t) for t in out],
                                   _stream(dev))
    _check(rc, "deltanet_prologue_fwd")
    return out


def deltanet_prologue_bwd(xq, xk, xv, xb, wq, wk, wv, dq, dk, dv, dbeta, *, silu_v=False,
                          workspace=None, out=None):
    """Backward of the prologue: returns (dxq, dxk, dxv, dxb, dwq, dwk, dwv)."""
    lib = load_library()
    dev = xq.device
    for t, n in ((dq, "dq"), (dk, "dk"), (dv, "dv"), (dbeta, "dbeta")):
        _need(t, n, xq.dtype, dev)
    d = _prologue_desc(xq, xv, silu_v)
    if workspace is None:
        n = int(lib.deltanet_prologue_workspace_bytes(ctypes.byref(d)))
        workspace = torch.empty(max(n, 16), dtype=torch.uint8, device=dev)
    if out is None:
        out = (torch.empty_like(xq), torch.empty_like(xk), torch.empty_like(xv),
               torch.empty_like(xb), torch.empty_like(wq), torch.empty_like(wk),
               torch.empty_like(wv))
    else:
        for t, ref, n in zip(out, (xq, xk, xv, xb, wq, wk, wv),
                             ("dxq", "dxk", "dxv", "dxb", "dwq", "dwk", "dwv")):
            _need_out(t, n, ref.shape, ref.dtype, dev)
    rc = lib.deltanet_prologue_bwd(ctypes.byref(d), _ptr(xq), _ptr(xk), _ptr(xv), _ptr(xb),
                                   _ptr(wq), _ptr(wk), _ptr(wv), _ptr(dq), _ptr(dk), _ptr(dv),
                                   _ptr(dbeta), *[_ptr(t) for t in out], _ptr(workspace),
                                   workspace.numel(), _stream(dev))
    _check(rc, "deltanet_prologue_bwd")
    return out


def deltanet_bwd(q, k, v, beta, dO, *, chunk=64, l2norm=True, h0=None, dhT=None,
                 workspace=None, states_saved=True, want_dh0=True, force_simt=False,
                 eps=1e-6, out=None, segments=True, force_split=False, extra_flags=0):
    """Backward: gradients w.r.t. raw q, k, v, beta (and h0).  With
    states_saved=True the workspace must come from deltanet_fwd(save_states=True)
    on the same inputs.  Returns (dq, dk, dv, dbeta, dh0 or None)."""
    lib = load_library()
    dev = q.device
    for t, n in ((q, "q"), (k, "k"), (v, "v"), (beta, "beta"), (dO, "dO")):
        _need(t, n, q.dtype, dev)
    _need(h0, "h0", torch.float32, dev)
    _need(dhT, "dhT", torch.float32, dev)
    if workspace is None:
        states_saved = False
    d = _desc_for(q, v, chunk, l2norm, states_saved, force_simt, eps, segments,
                  force_split=force_split, extra_flags=extra_flags)
    B, H, L, Dk = q.shape
    Dv = v.shape[-1]
    _need_inputs(q, k, v, beta, dO)
    if out is not None:
        dq, dk, dv, db = out
        for t, ref, n in ((dq, q, "dq"), (dk, k, "dk"), (dv, v, "dv"), (db, beta, "dbeta")):
            _need_out(t, n, ref.shape, ref.dtype, dev)
    else:
        dq = torch.empty_like(q)
        dk = torch.empty_like(k)
        dv = torch.empty_like(v)
        db = torch.empty_like(beta)
    for t, n in ((h0, "h0"), (dhT, "dhT")):
        _need_out(t, n, (B, H, Dk, Dv), torch.float32, dev)
    dh0 = torch.empty((B, H, Dk, Dv), dtype=torch.float32, device=dev) if want_dh0 else None
    if workspace is None:
        workspace = alloc_workspace(d, dev)
    _need(workspace, "workspace", torch.uint8, dev)
    rc = lib.deltanet_bwd(ctypes.byref(d), _ptr(q), _ptr(k), _ptr(v), _ptr(beta), _ptr(h0),
                          _ptr(dO), _ptr(dhT), _ptr(dq), _ptr(dk), _ptr(dv), _ptr(db),
                          _ptr(dh0), _ptr(workspace), workspace.numel(), _stream(dev))
    _check(rc, "deltanet_bwd")
    return dq, dk, dv, db, dh0


def deltanet_fwd_transition(q, k, v, beta, *, l2norm=True, eps=1e-6, psi=None, hloc=None,
                            workspace=None):
    """Transition of this sequence (include/deltanet.h, context parallelism):
    H_end = psi^T H_start + hloc.  Returns (psi [B,H,Dk,Dk], hloc [B,H,Dk,Dv])."""
    lib = load_library()
    dev = q.device
    for t, n in ((q, "q"), (k, "k"), (v, "v"), (beta, "beta")):
        _need(t, n, q.dtype, dev)
    B, H, L, Dk = q.shape
    Dv = v.shape[-1]
    d = make_desc(B, H, L, Dk, Dv, 64, q.dtype, l2norm=l2norm, eps=eps)
    if psi is None:
        psi = torch.empty((B, H, Dk, Dk), dtype=torch.float32, device=dev)
    if hloc is None:
        hloc = torch.empty((B, H, Dk, Dv), dtype=torch.float32, device=dev)
    _need_out(psi, "psi", (B, H, Dk, Dk), torch.float32, dev)
    _need_out(hloc, "hloc", (B, H, Dk, Dv), torch.float32, dev)
    if workspace is None:
        workspace = alloc_workspace(d, dev)
    _need(workspace, "workspace", torch.uint8, dev)
    rc = lib.deltanet_fwd_transition(ctypes.byref(d), _ptr(q), _ptr(k), _ptr(v), _ptr(beta),
                                     _ptr(psi), _ptr(hloc), _ptr(workspace), workspace.numel(),
                                     _stream(dev))
    _check(rc, "deltanet_fwd_transition")
    return psi, hloc


def deltanet_bwd_transition(q, k, v, beta, dO, *, l2norm=True, eps=1e-6, workspace=None,
                            states_saved=True, dhloc=None):
    """Local cotangent chain dl/dH_start of this sequence with dl/dH_end = 0.
    With states_saved the workspace comes from deltanet_fwd(save_states=True)
    over the same q, k, v, beta.  Returns dhloc [B,H,Dk,Dv]."""
    lib = load_library()
    dev = q.device
    for t, n in ((q, "q"), (k, "k"), (v, "v"), (beta, "beta"), (dO, "dO")):
        _need(t, n, q.dtype, dev)
    B, H, L, Dk = q.shape
    Dv = v.shape[-1]
    if workspace is None:
        states_saved = False
    d = make_desc(B, H, L, Dk, Dv, 64, q.dtype, l2norm=l2norm, save_states=states_saved, eps=eps)
    if workspace is None:
        workspace = alloc_workspace(d, dev)
    _need(workspace, "workspace", torch.uint8, dev)
    if dhloc is None:
        dhloc = torch.empty((B, H, Dk, Dv), dtype=torch.float32, device=dev)
    _need_out(dhloc, "dhloc", (B, H, Dk, Dv), torch.float32, dev)
    rc = lib.deltanet_bwd_transition(ctypes.byref(d), _ptr(q), _ptr(k), _ptr(v), _ptr(beta),
                                     _ptr(dO), _ptr(dhloc), _ptr(workspace), workspace.numel(),
                                     _stream(dev))
    _check(rc, "deltanet_bwd_transition")
    return dhloc


def deltanet_state_scan(psi_all, loc_all, part, *, reverse=False, edge=None, out=None):
    """Boundary state of part ``part`` from the gathered transitions
    psi_all [P,B,H,Dk,Dk], loc_all [P,B,H,Dk,Dv] (include/deltanet.h):
    forward H_start(part) from edge = h0, or (reverse) dH_end(part) from
    edge = dhT.  Returns out [B,H,Dk,Dv] fp32."""
    lib = load_library()
    dev = loc_all.device
    P, B, H, Dk, Dv = loc_all.shape
    for t, n in ((psi_all, "psi_all"), (loc_all, "loc_all"), (edge, "edge")):
        _need(t, n, torch.float32, dev)
    if out is None:
        out = torch.empty((B, H, Dk, Dv), dtype=torch.float32, device=dev)
    _need_out(out, "out", (B, H, Dk, Dv), torch.float32, dev)
    if tuple(psi_all.shape) != (P, B, H, Dk, Dk):
        raise DeltaNetError("psi_all must be [P,B,H,Dk,Dk]")
    d = make_desc(B, H, 0, Dk, Dv, 64, torch.bfloat16)
    rc = lib.deltanet_state_scan(ctypes.byref(d), int(P), int(part), int(bool(reverse)),
                                 _ptr(psi_all), _ptr(loc_all), _ptr(edge), _ptr(out),
                                 _stream(dev))
    _check(rc, "deltanet_state_scan")
    return out


def deltanet_gated_fwd(q, k, v, beta, g, *, chunk=64, l2norm=True, h0=None, save_states=True,
                       workspace=None, want_hT=True, force_simt=False, eps=1e-6, out=None):
    """Forward of Gated DeltaNet (PAPER.md Table tab:overview; DESIGN.md
    R23): g [B,H,L] fp32 log-decay, alpha = exp(g).  Returns (o, hT, workspace)."""
    lib = load_library()
    dev = q.device
    for t, n in ((q, "q"), (k, "k"), (v, "v"), (beta, "beta")):
        _need(t, n, q.dtype, dev)
    _need(g, "g", torch.float32, dev)
    _need(h0, "h0", torch.float32, dev)
    _need_inputs(q, k, v, beta)
    d = _desc_for(q, v, chunk, l2norm, save_states, force_simt, eps, gated=True)
    B, H, L, Dk = q.shape
    Dv = v.shape[-1]
    _need_out(g, "g", (B, H, L), torch.float32, dev)
    _need_out(h0, "h0", (B, H, Dk, Dv), torch.float32, dev)
    _need_out(out, "out", (B, H, L, Dv), q.dtype, dev)
    o = out if out is not None else torch.empty((B, H, L, Dv), dtype=q.dtype, device=dev)
    hT = torch.empty((B, H, Dk, Dv), dtype=torch.float32, device=dev) if want_hT else None
    if workspace is None:
        workspace = alloc_workspace(d, dev)
    _need(workspace, "workspace", torch.uint8, dev)
    rc = lib.deltanet_gated_fwd(ctypes.byref(d), _ptr(q), _ptr(k), _ptr(v), _ptr(beta), _ptr(g),
                                _ptr(h0), _ptr(o), _ptr(hT), _ptr(workspace), workspace.numel(),
                                _stream(dev))
    _check(rc, "deltanet_gated_fwd")
    return o, hT, workspace


def deltanet_gated_bwd(q, k, v, beta, g, dO, *, chunk=64, l2norm=True, h0=None, dhT=None,
                       workspace=None, states_saved=True, want_dh0=True, force_simt=False,
                       eps=1e-6):
    """Backward of Gated DeltaNet.  Returns (dq, dk, dv, dbeta, dg, dh0 or None)."""
    lib = load_library()
    dev = q.device
    for t, n in ((q, "q"), (k, "k"), (v, "v"), (beta, "beta"), (dO, "dO")):
        _need(t, n, q.dtype, dev)
    for t, n in ((g, "g"), (h0, "h0"), (dhT, "dhT")):
        _need(t, n, torch.float32, dev)
    if workspace is None:
        states_saved = False
    _need_inputs(q, k, v, beta, dO)
    d = _desc_for(q, v, chunk, l2norm, states_saved, force_simt, eps, gated=True)
    B, H, L, Dk = q.shape
    Dv = v.shape[-1]
    _need_out(g, "g", (B, H, L), torch.float32, dev)
    for t, n in ((h0, "h0"), (dhT, "dhT")):
        _need_out(t, n, (B, H, Dk, Dv), torch.float32, dev)
    dq, dk, dv, db = (torch.empty_like(t) for t in (q, k, v, beta))
    dg = torch.empty_like(g)
    dh0 = torch.empty((B, H, Dk, Dv), dtype=torch.float32, device=dev) if want_dh0 else None
    if workspace is None:
        workspace = alloc_workspace(d, dev)
    _need(workspace, "workspace", torch.uint8, dev)
    rc = lib.deltanet_gated_bwd(ctypes.byref(d), _ptr(q), _ptr(k), _ptr(v), _ptr(beta), _ptr(g),
                                _ptr(h0), _ptr(dO), _ptr(dhT), _ptr(dq), _ptr(dk), _ptr(dv),
                                _ptr(db), _ptr(dg), _ptr(dh0), _ptr(workspace),
                                workspace.numel(), _stream(dev))
    _check(rc, "deltanet_gated_bwd")
    return dq, dk, dv, db, dg, dh0


def deltanet_gated_recurrent_fwd(q, k, v, beta, g, *, l2norm=True, h0=None, want_hT=True,
                                 eps=1e-6, out=None, hT=None):
    """Recurrent (token-by-token) gated forward for inference / decode.
    Passing hT=h0 updates the state in place.  Returns (o, hT or None)."""
    lib = load_library()
    dev = q.device
    for t, n in ((q, "q"), (k, "k"), (v, "v"), (beta, "beta")):
        _need(t, n, q.dtype, dev)
    for t, n in ((g, "g"), (h0, "h0"), (hT, "hT")):
        _need(t, n, torch.float32, dev)
    _need_inputs(q, k, v, beta)
    B, H, L, Dk = q.shape
    Dv = v.shape[-1]
    _need_out(g, "g", (B, H, L), torch.float32, dev)
    for t, n in ((h0, "h0"), (hT, "hT")):
        _need_out(t, n, (B, H, Dk, Dv), torch.float32, dev)
    _need_out(out, "out", (B, H, L, Dv), q.dtype, dev)
    d = make_desc(B, H, L, Dk, Dv, 64, q.dtype, l2norm=l2norm, eps=eps)
    o = out if out is not None else torch.empty((B, H, L, Dv), dtype=q.dtype, device=dev)
    if hT is None and want_hT:
        hT = torch.empty((B, H, Dk, Dv), dtype=torch.float32, device=dev)
    rc = lib.deltanet_gated_recurrent_fwd(ctypes.byref(d), _ptr(q), _ptr(k), _ptr(v),
                                          _ptr(beta), _ptr(g), _ptr(h0), _ptr(o), _ptr(hT),
                                          _stream(dev))
    _check(rc, "deltanet_gated_recurrent_fwd")
    return o, hT


def deltanet_fwd_bwd_host(q, k, v, beta, dO, *, out, slabs=8, chunk=64, l2norm=True,
                          dev_buffer=None, device=None, eps=1e-6):
    """Forward + backward of host (CPU, ideally pinned) tensors through the
    library's copy/compute pipeline (include/deltanet.h deltanet_fwd_bwd_host).
    ``out`` = (o, dq, dk, dv, dbeta) host tensors.  Asynchronous on the
    current stream of ``device``.  Returns (dev_buffer, out)."""
    lib = load_library()
    dev = torch.device(device if device is not None else "cuda")
    for t, n in ((q, "q"), (k, "k"), (v, "v"), (beta, "beta"), (dO, "dO"), *zip(out, "o dq dk dv dbeta".split())):
        if t.is_cuda:
            raise DeltaNetError(f"{n} must be a host tensor for deltanet_fwd_bwd_host")
        if not t.is_contiguous() or t.dtype != q.dtype:
            raise DeltaNetError(f"{n} must be contiguous with dtype {q.dtype}")
    _need_inputs(q, k, v, beta, dO)
    for t, ref, n in zip(out, (v, q, k, v, beta), "o dq dk dv dbeta".split()):
        if t.shape != ref.shape:
            raise DeltaNetError(f"{n} has shape {tuple(t.shape)}, expected {tuple(ref.shape)}")
    B, H, L, Dk = q.shape
    d = make_desc(B, H, L, Dk, v.shape[-1], chunk, q.dtype, l2norm=l2norm, eps=eps)
    need = int(lib.deltanet_fwd_bwd_host_device_bytes(ctypes.byref(d), int(slabs)))
    if dev_buffer is None or dev_buffer.numel() < need:
        dev_buffer = torch.empty(max(need, 16), dtype=torch.uint8, device=dev)
    o, dq, dk, dv, db = out
    rc = lib.deltanet_fwd_bwd_host(ctypes.byref(d), _ptr(q), _ptr(k), _ptr(v), _ptr(beta),
                                   _ptr(dO), _ptr(o), _ptr(dq), _ptr(dk), _ptr(dv), _ptr(db),
                                   int(slabs), _ptr(dev_buffer), dev_buffer.numel(),
                                   _stream(dev))
    _check(rc, "deltanet_fwd_bwd_host")
    return dev_buffer, out


class DeltaNetChunkFunction(torch.autograd.Function):
    """autograd wrapper: o = DeltaNet(q, k, v, beta) with L2-normalised q, k."""

    @staticmethod
    def forward(ctx, q, k, v, beta, chunk=64, l2norm=True):
        o, _, ws = deltanet_fwd(q, k, v, beta, chunk=chunk, l2norm=l2norm, want_hT=False)
        ctx.save_for_backward(q, k, v, beta, ws)
        ctx.chunk, ctx.l2norm = chunk, l2norm
        return o

    @staticmethod
    def backward(ctx, dO):
        q, k, v, beta, ws = ctx.saved_tensors
        dq, dk, dv, db, _ = deltanet_bwd(q, k, v, beta, dO.contiguous(), chunk=ctx.chunk,
                                         l2norm=ctx.l2norm, workspace=ws, want_dh0=False)
        return dq, dk, dv, db, None, None


def deltanet(q, k, v, beta, chunk=64, l2norm=True):
    return DeltaNetChunkFunction.apply(q, k, v, beta, chunk, l2norm)


__all__ = ["deltanet_fwd", "deltanet_bwd", "deltanet_workspace_bytes", "deltanet_path",
           "deltanet_launch_count", "deltanet_strerror", "deltanet_desc", "make_desc",
           "load_library", "alloc_workspace", "DeltaNetError", "deltanet", "EXPORTED",
           "LIB_PATH", "deltanet_fwd_transition", "deltanet_bwd_transition",
           "deltanet_state_scan", "deltanet_gated_fwd", "deltanet_gated_bwd",
           "deltanet_gated_recurrent_fwd", "DELTANET_GATED"]
