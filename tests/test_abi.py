"""CPU-side checks of the C-ABI library: it builds/loads, exports every symbol
include/deltanet.h declares, and rejects bad arguments before any launch."""
import ctypes
import os
import re

import pytest

import paper_2406_06484_b200 as dn
from paper_2406_06484_b200 import build as dnbuild

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "deltanet.h")


@pytest.fixture(scope="module")
def lib():
    dnbuild.build()
    return dn.load_library()


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(deltanet_[a-z_]+)\s*\(", src)))


def test_header_declares_expected_api():
    names = declared_functions()
    for n in ("deltanet_fwd", "deltanet_bwd", "deltanet_workspace_bytes", "deltanet_strerror"):
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert set(dn.EXPORTED) == set(declared_functions())


def test_no_torch_types_in_abi():
    src = open(HEADER).read()
    assert "torch" not in src.lower().replace("pytorch", "") or "at::" not in src
    assert "at::Tensor" not in src and "c10" not in src


def test_abi_version_and_strerror(lib):
    assert lib.deltanet_abi_version() == 8
    for code in range(6):
        assert dn.deltanet_strerror(code)
    assert "unknown" in dn.deltanet_strerror(99)


def _desc(**kw):
    base = dict(B=2, H=3, L=100, Dk=128, Dv=128, chunk=64, dtype=0, flags=1, l2_eps=1e-6)
    base.update(kw)
    return dn.deltanet_desc(**base)


def test_workspace_and_validation(lib):
    d = _desc()
    n = dn.deltanet_workspace_bytes(d)
    # states: B*H*ceil(L/C)*Dk*Dv*2 bytes at least
    assert n >= 2 * 3 * 2 * 64 * 64 * 2
    assert dn.deltanet_workspace_bytes(_desc(Dk=48)) == 0          # unsupported
    assert dn.deltanet_workspace_bytes(_desc(chunk=8)) == 0
    assert dn.deltanet_workspace_bytes(_desc(dtype=7)) == 0
    assert dn.deltanet_workspace_bytes(_desc(L=-1)) == 0
    assert dn.deltanet_path(_desc(Dk=48)) == -1
    assert dn.deltanet_path(_desc(dtype=1)) == 0                   # fp32 -> SIMT
    assert dn.deltanet_path(_desc(flags=1 | 4)) == 0               # FORCE_SIMT
    assert dn.deltanet_path(_desc()) == 1                          # tcgen05
    assert dn.deltanet_path(_desc(L=0)) != -1                     # L = 0: nothing to run


@pytest.mark.parametrize("D", [64, 256])
def test_split_path_shapes(lib, D):
    """Dk = Dv in {64, 256} (BASELINE configs[3] is d = 256) run the split
    tcgen05 kernels (path 2); d = 128 only with
    DELTANET_FORCE_SPLIT; gated, other chunks and unequal dims are refused."""
    d = _desc(Dk=D, Dv=D)
    assert dn.deltanet_path(d) == 2
    assert dn.deltanet_workspace_bytes(d) > 0
    assert dn.deltanet_launch_count(d, 0) == 2 and dn.deltanet_launch_count(d, 1) == 4
    saved = _desc(Dk=D, Dv=D, flags=1 | dn.DELTANET_SAVE_STATES)
    assert dn.deltanet_launch_count(saved, 1) == 2  # records from the forward
    assert dn.deltanet_path(_desc(flags=1 | dn.DELTANET_FORCE_SPLIT)) == 2
    assert dn.deltanet_path(_desc()) == 1
    assert dn.deltanet_path(_desc(Dk=D, Dv=D, flags=1 | dn.DELTANET_GATED)) == -1
    assert dn.deltanet_path(_desc(Dk=D, Dv=D, chunk=32)) == -1
    assert dn.deltanet_path(_desc(Dk=D, Dv=D, dtype=1)) == 0     # fp32 -> SIMT


@pytest.mark.parametrize("shape", [dict(Dk=64, Dv=128), dict(chunk=128), dict(chunk=32),
                                   dict(Dk=128, Dv=64), dict(Dk=16, Dv=16, chunk=16)])
def test_bf16_outside_tcgen05_shapes_is_unsupported(lib, shape):
    """bf16 descriptors outside the tcgen05 shapes are refused (UNSUPPORTED,
    before any launch) unless DELTANET_FORCE_SIMT asks for the CUDA-core
    kernels explicitly: no silent fallback 10^3-10^4x below the roofline.
    fp32 I/O (the parity mode) always runs on the CUDA-core kernels."""
    D = ctypes.byref
    nul = None
    a = ctypes.c_void_p(16 * 1024)
    d = _desc(**shape)
    assert dn.deltanet_path(d) == -1
    assert dn.deltanet_workspace_bytes(d) == 0
    assert dn.deltanet_launch_count(d, 0) == -1
    assert lib.deltanet_fwd(D(d), a, a, a, a, nul, a, nul, a, 1 << 34, nul) == 2
    assert lib.deltanet_bwd(D(d), a, a, a, a, nul, a, nul, a, a, a, a, nul, a, 1 << 34, nul) == 2
    forced = _desc(flags=1 | dn.DELTANET_FORCE_SIMT, **shape)
    assert dn.deltanet_path(forced) == 0 and dn.deltanet_workspace_bytes(forced) > 0
    assert dn.deltanet_path(_desc(dtype=1, **shape)) == 0


def test_errors_before_launch(lib):
    """Argument errors return before any CUDA call (works without a GPU)."""
    D = ctypes.byref
    d = _desc()
    nul = None
    rc = lib.deltanet_fwd(D(d), nul, nul, nul, nul, nul, nul, nul, nul, 0, nul)
    assert rc == 1
    rc = lib.deltanet_fwd(D(_desc(Dk=48)), nul, nul, nul, nul, nul, nul, nul, nul, 0, nul)
    assert rc == 2
    p = ctypes.c_void_p(16 * 1024 + 4)  # misaligned fake pointer, never dereferenced
    a = ctypes.c_void_p(16 * 1024)
    rc = lib.deltanet_fwd(D(d), p, a, a, a, nul, a, nul, a, 1 << 30, nul)
    assert rc == 3
    rc = lib.deltanet_fwd(D(d), a, a, a, a, nul, a, nul, a, 16, nul)  # workspace too small
    assert rc == 5
    rc = lib.deltanet_bwd(D(d), a, a, a, a, nul, nul, nul, a, a, a, a, nul, a, 1 << 30, nul)
    assert rc == 1  # dO missing
    # empty problem: nothing to do, no launch
    e = _desc(B=0)
    assert lib.deltanet_fwd(D(e), nul, nul, nul, nul, nul, nul, nul, nul, 0, nul) == 0
    assert dn.deltanet_launch_count(e, 0) == 0


def test_binding_refuses_cpu_tensors(lib):
    import torch
    q = torch.zeros(1, 1, 16, 16)
    with pytest.raises(dn.DeltaNetError):
        dn.deltanet_fwd(q, q, q, torch.zeros(1, 1, 16), chunk=16)


def test_recurrent_errors_before_launch(lib):
    """deltanet_recurrent_fwd validates shapes/dtype (not chunk) before any launch."""
    D = ctypes.byref
    nul = None
    a = ctypes.c_void_p(16 * 1024)
    p = ctypes.c_void_p(16 * 1024 + 4)
    assert lib.deltanet_recurrent_fwd(D(_desc()), nul, nul, nul, nul, nul, nul, nul, nul) == 1
    assert lib.deltanet_recurrent_fwd(D(_desc(Dk=48)), a, a, a, a, nul, a, nul, nul) == 2
    assert lib.deltanet_recurrent_fwd(D(_desc(dtype=7)), a, a, a, a, nul, a, nul, nul) == 2
    assert lib.deltanet_recurrent_fwd(D(_desc()), p, a, a, a, nul, a, nul, nul) == 3
    # chunk is not part of the recurrent form: an invalid chunk is not an error
    assert dn.deltanet_launch_count(_desc(chunk=8), 2) == 1
    assert dn.deltanet_launch_count(_desc(B=0), 2) == 0
    e = _desc(B=0)
    assert lib.deltanet_recurrent_fwd(D(e), nul, nul, nul, nul, nul, nul, nul, nul) == 0


def test_context_parallel_errors_before_launch(lib):
    """The transition / scan entry points validate before any launch: the
    tcgen05 shapes only (bf16, Dk = Dv = 128, chunk 64), null outputs, part
    range, misalignment; L = 0 and B*H = 0 are legal."""
    D = ctypes.byref
    nul = None
    a = ctypes.c_void_p(16 * 1024)
    p = ctypes.c_void_p(16 * 1024 + 4)
    ok = dict(Dk=128, Dv=128, chunk=64)
    # UNSUPPORTED outside the tcgen05 shapes
    assert lib.deltanet_fwd_transition(D(_desc(Dk=64, Dv=64)), a, a, a, a, a, a, a, 1 << 34, nul) == 2
    assert lib.deltanet_fwd_transition(D(_desc(**ok, dtype=1)), a, a, a, a, a, a, a, 1 << 34, nul) == 2
    assert lib.deltanet_fwd_transition(D(_desc(**ok, flags=4)), a, a, a, a, a, a, a, 1 << 34, nul) == 2
    assert lib.deltanet_state_scan(D(_desc(Dk=64, Dv=64)), 2, 0, 0, a, a, nul, a, nul) == 2
    # null required pointers, bad part index, misalignment
    assert lib.deltanet_fwd_transition(D(_desc(**ok)), a, a, a, a, nul, a, a, 1 << 34, nul) == 1
    assert lib.deltanet_fwd_transition(D(_desc(**ok)), nul, a, a, a, a, a, a, 1 << 34, nul) == 1
    assert lib.deltanet_fwd_transition(D(_desc(**ok)), a, a, a, a, p, a, a, 1 << 34, nul) == 3
    assert lib.deltanet_bwd_transition(D(_desc(**ok)), a, a, a, a, nul, a, a, 1 << 30, nul) == 1
    assert lib.deltanet_bwd_transition(D(_desc(**ok)), a, a, a, a, a, a, nul, 0, nul) == 5
    for nparts, part, rev in ((0, 0, 0), (2, 2, 0), (2, -1, 1), (2, 0, 2)):
        assert lib.deltanet_state_scan(D(_desc(**ok)), nparts, part, rev, a, a, nul, a, nul) == 1
    assert lib.deltanet_state_scan(D(_desc(**ok)), 2, 1, 0, nul, a, nul, a, nul) == 1
    assert lib.deltanet_state_scan(D(_desc(**ok)), 2, 1, 0, a, a, nul, p, nul) == 3
    # nothing to do: B*H = 0
    e = _desc(B=0, **ok)
    assert lib.deltanet_fwd_transition(D(e), nul, nul, nul, nul, nul, nul, nul, 0, nul) == 0
    assert lib.deltanet_state_scan(D(e), 2, 0, 0, nul, nul, nul, nul, nul) == 0
    for which in (5, 6, 7):
        assert dn.deltanet_launch_count(_desc(**ok), which) >= 1
        assert dn.deltanet_launch_count(e, which) == 0
        assert dn.deltanet_launch_count(_desc(Dk=64, Dv=64), which) == -1


def test_gated_errors_before_launch(lib):
    """Gated entry points: g without dg is INVALID_ARG; the plain entry points
    refuse a descriptor carrying DELTANET_GATED; the workspace query with the
    flag covers the gated path; the CP transitions refuse it."""
    D = ctypes.byref
    nul = None
    a = ctypes.c_void_p(16 * 1024)
    big = 1 << 34
    d = _desc()
    assert lib.deltanet_gated_bwd(D(d), a, a, a, a, a, nul, a, nul, a, a, a, a, nul, nul, a, big,
                                  nul) == 1
    dg = _desc(flags=dn.DELTANET_GATED)
    assert lib.deltanet_fwd(D(dg), a, a, a, a, nul, a, nul, a, big, nul) == 1
    assert dn.deltanet_workspace_bytes(dg) > 0
    ok = _desc(Dk=128, Dv=128, chunk=64, flags=dn.DELTANET_GATED)
    assert lib.deltanet_fwd_transition(D(ok), a, a, a, a, a, a, a, 1 << 34, nul) == 2
    assert dn.deltanet_launch_count(dg, 0) == 1


def test_workspace_holds_segment_prep_records(lib):
    """A segmented forward (few units, many chunks) reserves
    pass 1's per-chunk prep records [T' | T'' | s | 1/s] (16.5 KB per chunk
    per unit) beyond the same shape without segments."""
    B, H, L = 1, 2, 64 * 40
    seg = _desc(B=B, H=H, L=L, flags=1 | 2)
    noseg = _desc(B=B, H=H, L=L, flags=1 | 2 | dn.DELTANET_NO_SEGMENTS)
    assert dn.deltanet_launch_count(seg, 0) == 3 and dn.deltanet_launch_count(noseg, 0) == 1
    prec = B * H * (L // 64) * (2 * 64 * 64 * 2 + 2 * 64 * 4)
    assert dn.deltanet_workspace_bytes(seg) - dn.deltanet_workspace_bytes(noseg) >= prec
