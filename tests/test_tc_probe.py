"""GPU probe of the tcgen05 operand conventions (tests/cuda/mma_probe.cu):
every (A major, B major, M, negate, accumulate) combination the product
kernels use, against a plain fp32 matmul of the same bf16 values."""
import ctypes
import os
import subprocess

import pytest
import torch

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def probe():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    src = os.path.join(HERE, "cuda", "mma_probe.cu")
    lib = os.path.join(HERE, "cuda", "libprobe.so")
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-std=c++17",
                    "-Xcompiler", "-fPIC", "-shared", "-o", lib, src], check=True)
    L = ctypes.CDLL(lib)
    L.probe_mma.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_int] * 7
    L.probe_mma.restype = ctypes.c_int
    L.probe_mma_ts.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] * 3
    L.probe_mma_ts.restype = ctypes.c_int
    L.probe_tmem_bw.argtypes = [ctypes.c_int] * 3
    L.probe_tmem_bw.restype = ctypes.c_longlong
    L.probe_mma_tput.argtypes = [ctypes.c_int] * 5 + [ctypes.POINTER(ctypes.c_longlong)]
    L.probe_mma_tput.restype = ctypes.c_longlong
    L.probe_mma_issue.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_longlong)]
    L.probe_mma_issue.restype = ctypes.c_longlong
    L.probe_mma_batch.argtypes = [ctypes.c_int] * 3
    L.probe_mma_batch.restype = ctypes.c_longlong
    L.probe_mma_sw.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] * 6
    L.probe_mma_sw.restype = ctypes.c_int
    return L


@pytest.mark.parametrize("M,N,K", [(128, 64, 64), (128, 128, 64), (128, 64, 128),
                                   (64, 64, 128), (64, 128, 128), (64, 128, 64)])
@pytest.mark.parametrize("a_mn", [0, 1])
@pytest.mark.parametrize("b_mn", [0, 1])
def test_mma_layouts(probe, M, N, K, a_mn, b_mn):
    g = torch.Generator().manual_seed(M * 1000 + N * 10 + K + a_mn * 7 + b_mn * 3)
    A = torch.randn(M, K, generator=g).bfloat16()
    B = torch.randn(N, K, generator=g).bfloat16()
    ref = A.float() @ B.float().T
    Ad, Bd = A.cuda(), B.cuda()
    D = torch.zeros(M, N, device="cuda")
    rc = probe.probe_mma(Ad.data_ptr(), Bd.data_ptr(), None, D.data_ptr(), M, N, K, a_mn, b_mn, 0, 0)
    assert rc == 0
    err = (D.cpu() - ref).abs().max().item()
    assert err <= 1e-3 * ref.abs().max().item(), err


@pytest.mark.parametrize("M", [64, 128])
@pytest.mark.parametrize("init", [0, 1])
@pytest.mark.parametrize("neg", [0, 1])
def test_mma_negate_accumulate(probe, M, init, neg):
    N, K = 64, 128
    g = torch.Generator().manual_seed(M)
    A = torch.randn(M, K, generator=g).bfloat16()
    B = torch.randn(N, K, generator=g).bfloat16()
    D0 = torch.randn(M, N, generator=g) if init else torch.zeros(M, N)
    ref = D0 + (-1 if neg else 1) * (A.float() @ B.float().T)
    D = torch.zeros(M, N, device="cuda")
    D0d, Ad, Bd = D0.cuda(), A.cuda(), B.cuda()  # keep device copies alive
    rc = probe.probe_mma(Ad.data_ptr(), Bd.data_ptr(),
                         D0d.data_ptr() if init else None, D.data_ptr(), M, N, K, 0, 1, neg, 0)
    assert rc == 0
    assert (D.cpu() - ref).abs().max().item() <= 1e-3 * ref.abs().max().item()


@pytest.mark.parametrize("N", [64, 128])
@pytest.mark.parametrize("init", [0, 1])
def test_mma_m64_lane_offset_16(probe, N, init):
    """M=64 accumulator at TMEM lane offset 16 (rows in lanes 16-31 of each
    32-lane quadrant), the pairing the backward kernel relies on."""
    M, K = 64, 128
    g = torch.Generator().manual_seed(N + init)
    A = torch.randn(M, K, generator=g).bfloat16()
    B = torch.randn(N, K, generator=g).bfloat16()
    D0 = torch.randn(M, N, generator=g) if init else torch.zeros(M, N)
    ref = D0 + A.float() @ B.float().T
    Ad, Bd, D0d = A.cuda(), B.cuda(), D0.cuda()
    D = torch.zeros(M, N, device="cuda")
    rc = probe.probe_mma(Ad.data_ptr(), Bd.data_ptr(), D0d.data_ptr() if init else None,
                         D.data_ptr(), M, N, K, 0, 1, 0, 16)
    assert rc == 0
    assert (D.cpu() - ref).abs().max().item() <= 1e-3 * ref.abs().max().item()


@pytest.mark.parametrize("N,K", [(64, 64), (128, 64), (64, 128), (128, 128)])
@pytest.mark.parametrize("b_mn", [0, 1])
def test_mma_a_from_tmem(probe, N, K, b_mn):
    """tcgen05.mma with the A operand in TMEM (M=128, bf16 pairs per column)."""
    g = torch.Generator().manual_seed(N * 3 + K + b_mn)
    A = torch.randn(128, K, generator=g).bfloat16()
    B = torch.randn(N, K, generator=g).bfloat16()
    ref = A.float() @ B.float().T
    Ad, Bd = A.cuda(), B.cuda()
    D = torch.zeros(128, N, device="cuda")
    assert probe.probe_mma_ts(Ad.data_ptr(), Bd.data_ptr(), D.data_ptr(), N, K, b_mn) == 0
    assert (D.cpu() - ref).abs().max().item() <= 1e-3 * ref.abs().max().item()


def test_tmem_read_throughput(probe):
    """Measure TMEM -> register bandwidth (bytes per SM cycle); informational."""
    res = {}
    for nt in (128, 256, 512):
        iters, ncols = 200, 128
        cyc = probe.probe_tmem_bw(nt, iters, ncols)
        byts = nt * iters * ncols * 4
        res[nt] = byts / cyc
    print("\nTMEM read bytes/cycle by thread count:", {k: round(v, 1) for k, v in res.items()})
    assert all(v > 0 for v in res.values())


def test_mma_throughput(probe):
    """Cycles per tcgen05.mma (K=16) from SWIZZLE_NONE tiles; informational
    (ideal: max(M,128) * N / 256)."""
    rows = []
    for (M, N) in ((128, 64), (128, 128), (64, 64), (64, 128)):
        for a_mn, b_mn in ((0, 0), (0, 1), (1, 0), (1, 1)):
            iss = ctypes.c_longlong(0)
            n = 256
            cyc = probe.probe_mma_tput(M, N, n, a_mn, b_mn, ctypes.byref(iss))
            rows.append(f"M={M} N={N} a_mn={a_mn} b_mn={b_mn}: {cyc / n:6.1f} cyc/mma "
                        f"(issue {iss.value / n:5.1f}), ideal {max(M, 128) * N / 256:5.1f}")
    print("\n" + "\n".join(rows))


def test_mma_issue_patterns(probe):
    """M=128 N=64 K=16 MMAs: cycles per instruction for three issue patterns
    (0: descriptors rebuilt per MMA, lane 0; 1: precomputed, lane 0;
    2: whole warp + elect.sync); informational, ideal 32."""
    rows = []
    for v in (0, 1, 2, 3, 4, 5):
        iss = ctypes.c_longlong(0)
        reps = 32
        nw = v - 1 if v >= 3 else 1
        cyc = probe.probe_mma_issue(v, reps, ctypes.byref(iss))
        rows.append(f"variant {v} ({nw} issuing warps): {cyc / (8 * reps * nw):6.1f} cyc/mma "
                    f"aggregate (per-warp issue {iss.value / (8 * reps):5.1f})")
    print("\n" + "\n".join(rows))


def test_mma_m64_batches(probe):
    """M=64 MMA batches (B MN-major), accumulators at lane offset 0 only or
    alternating 0/16; informational cycles per MMA."""
    rows = []
    for N in (64, 128):
        for l16 in (0, 1):
            n = 256
            cyc = probe.probe_mma_batch(N, l16, n)
            rows.append(f"M=64 N={N} lane16_alternate={l16}: {cyc / n:6.1f} cyc/mma")
    print("\n" + "\n".join(rows))


@pytest.mark.parametrize("M,N,K", [(128, 64, 64), (128, 128, 64), (128, 64, 128),
                                   (64, 64, 128), (64, 128, 128), (64, 128, 64)])
@pytest.mark.parametrize("a_mn", [0, 1])
@pytest.mark.parametrize("b_mn", [0, 1])
@pytest.mark.parametrize("sw", [1, 2, 3])
def test_mma_sw128_layouts(probe, M, N, K, a_mn, b_mn, sw):
    """SWIZZLE_128B tiles (tc_common.cuh sw_off, desc_k_sw, desc_mn_sw) as
    K-major and MN-major operands, alone or mixed with IL tiles."""
    g = torch.Generator().manual_seed(M * 1000 + N * 10 + K + a_mn * 7 + b_mn * 3 + sw)
    A = torch.randn(M, K, generator=g).bfloat16()
    B = torch.randn(N, K, generator=g).bfloat16()
    ref = A.float() @ B.float().T
    Ad, Bd = A.cuda(), B.cuda()
    D = torch.zeros(M, N, device="cuda")
    assert probe.probe_mma_sw(Ad.data_ptr(), Bd.data_ptr(), D.data_ptr(), M, N, K, a_mn, b_mn, sw) == 0
    err = (D.cpu() - ref).abs().max().item()
    assert err <= 1e-3 * ref.abs().max().item(), err
