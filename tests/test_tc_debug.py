"""Intermediate-level check of the tcgen05 forward kernel (test-only build
with -DDN_DEBUG): the per-chunk quantities L, X=(I+L)^{-1}, W, U, U', O, H of
unit 0 are dumped and compared with an fp64 restatement of PAPER.md §3.2
(Eq. 8-11) on the same bf16 inputs.  Localises a failure of the end-to-end
parity tests to one stage of the kernel."""
import ctypes
import glob
import os
import subprocess

import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)

OFF = dict(L=0, X=4096, GQK=8192, W=12288, U=20480, UP=28672, O=36864, H=45056, S=61440,
           R=61504, B=61568)


@pytest.fixture(scope="module")
def dbg_lib():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    out = os.path.join(HERE, "cuda", "libdeltanet_dbg.so")
    srcs = sorted(glob.glob(os.path.join(ROOT, "paper_2406_06484_b200", "csrc", "*.cu")))
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-std=c++17",
                    "-DDN_DEBUG", "-Xcompiler", "-fPIC", "-shared", "-I",
                    os.path.join(ROOT, "include"), "-o", out, *srcs], check=True)
    lib = ctypes.CDLL(out)
    lib.dn_debug_set.argtypes = [ctypes.c_void_p, ctypes.c_int]
    return lib


def _ref_chunk(q, k, v, beta, c, C=64):
    """fp64 restatement (per chunk) of Eq. 10-11 then Eq. 8-9 for one unit,
    with L2-normalised q, k; H_c from the exact recurrence of chunks < c,
    rounded to bf16 as the kernel's MMA operand."""
    f = lambda a: np.asarray(a, dtype=np.float64)
    q, k, v, beta = f(q), f(k), f(v), f(beta)
    nq = np.linalg.norm(q, axis=1); nk = np.linalg.norm(k, axis=1)
    qh = q / np.maximum(nq, 1e-6)[:, None]; kh = k / np.maximum(nk, 1e-6)[:, None]
    H = np.zeros((k.shape[1], v.shape[1]))
    out = {}
    for cc in range(c + 1):
        sl = slice(cc * C, (cc + 1) * C)
        Q, K, V, b = qh[sl], kh[sl], v[sl], beta[sl]
        Hb = synth.round_to_bf16(H.astype(np.float32)).astype(np.float64)
        Lm = np.tril((b[:, None] * K) @ K.T, -1)
        X = np.linalg.inv(np.eye(C) + Lm)
        W = X @ (b[:, None] * K)
        U = X @ (b[:, None] * V)
        Up = U - W @ Hb
        O = Q @ Hb + np.tril(Q @ K.T) @ Up
        Hn = Hb + K.T @ Up if cc == c else H + K.T @ (U - W @ H)
        if cc == c:
            s = 1 / np.maximum(nk[sl], 1e-6); r = 1 / np.maximum(nq[sl], 1e-6)
            out = dict(L=Lm, X=X, GQK=q[sl] @ k[sl].T, W=W.T, U=U.T, UP=Up.T,
                       O=O / r[:, None], H=Hn.T, S=s, R=r, B=b)
        H = Hn
    return out


@pytest.mark.parametrize("chunk_idx", [0, 2])
def test_fwd_intermediates(dbg_lib, chunk_idx):
    import paper_2406_06484_b200 as dn
    cfg = synth.custom_config(1, 1, 4 * 64, 128, 128, 64, "bf16", index=777)
    inp = synth.make_inputs(cfg)
    td = torch.bfloat16
    q, k, v, b = (torch.from_numpy(inp[f]).to(td).cuda() for f in ("q", "k", "v", "beta"))
    buf = torch.zeros(62000, device="cuda")
    assert dbg_lib.dn_debug_set(buf.data_ptr(), chunk_idx) == 0
    d = dn.make_desc(1, 1, cfg.L, 128, 128, 64, td)
    ws = torch.empty(dn.deltanet_workspace_bytes(d), dtype=torch.uint8, device="cuda")
    o = torch.empty_like(v)
    hT = torch.empty(1, 1, 128, 128, device="cuda")
    P = ctypes.c_void_p
    dbg_lib.deltanet_fwd.argtypes = [P] * 9 + [ctypes.c_size_t, P]
    rc = dbg_lib.deltanet_fwd(ctypes.addressof(d), q.data_ptr(), k.data_ptr(), v.data_ptr(),
                              b.data_ptr(), None, o.data_ptr(), hT.data_ptr(), ws.data_ptr(),
                              ws.numel(), None)
    assert rc == 0
    torch.cuda.synchronize()
    got = buf.cpu().numpy().astype(np.float64)
    ref = _ref_chunk(inp["q"][0, 0], inp["k"][0, 0], inp["v"][0, 0], inp["beta"][0, 0],
                     chunk_idx)
    shapes = dict(L=(64, 64), X=(64, 64), GQK=(64, 64), W=(128, 64), U=(128, 64),
                  UP=(128, 64), O=(64, 128), H=(128, 128), S=(64,), R=(64,), B=(64,))
    errs = {}
    for key, shp in shapes.items():
        n = int(np.prod(shp))
        g = got[OFF[key]:OFF[key] + n].reshape(shp)
        rr = ref[key]
        if key == "GQK":
            g = np.tril(g)  # only the causal part is consumed
            rr = np.tril(rr)
        errs[key] = float(np.abs(g - rr).max() / max(np.abs(rr).max(), 1e-30))
    print(errs)
    bad = {k_: e for k_, e in errs.items() if e > 2e-2}
    assert not bad, errs
