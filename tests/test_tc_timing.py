"""Test-only phase timeline of the tcgen05 forward (build with -DDN_TIMING):
clock64 stamps of CTA 0 per chunk, printed as per-phase cycle means.  Not a
correctness test; it is skipped unless DN_TIMING=1 is set in the environment."""
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


@pytest.mark.skipif(os.environ.get("DN_TIMING") != "1", reason="profiling aid; set DN_TIMING=1")
def test_fwd_timeline():
    import paper_2406_06484_b200 as dn
    out = os.path.join(HERE, "cuda", "libdeltanet_tim.so")
    srcs = sorted(glob.glob(os.path.join(ROOT, "paper_2406_06484_b200", "csrc", "*.cu")))
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                    "-DDN_TIMING", "-Xcompiler", "-fPIC", "-shared", "-I",
                    os.path.join(ROOT, "include"), "-o", out, *srcs], check=True)
    lib = ctypes.CDLL(out)
    cfg = synth.CONFIGS["target"]
    x = synth.make_inputs(cfg, b_range=range(1))
    td = torch.bfloat16
    q, k, v, b = (torch.from_numpy(x[f]).to(td).cuda() for f in ("q", "k", "v", "beta"))
    NC = cfg.L // 64
    buf = torch.zeros(NC * 32, dtype=torch.int64, device="cuda")
    lib.dn_timing_set.argtypes = [ctypes.c_void_p]
    assert lib.dn_timing_set(buf.data_ptr()) == 0
    d = dn.make_desc(1, cfg.H, cfg.L, 128, 128, 64, td)
    ws = torch.empty(dn.deltanet_workspace_bytes(d), dtype=torch.uint8, device="cuda")
    o = torch.empty_like(v)
    P = ctypes.c_void_p
    lib.deltanet_fwd.argtypes = [P] * 9 + [ctypes.c_size_t, P]
    for _ in range(2):
        rc = lib.deltanet_fwd(ctypes.addressof(d), q.data_ptr(), k.data_ptr(), v.data_ptr(),
                              b.data_ptr(), None, o.data_ptr(), None, ws.data_ptr(), ws.numel(),
                              None)
        assert rc == 0
    torch.cuda.synchronize()
    t = buf.cpu().numpy().reshape(NC, 32).astype(np.int64)
    names = {0: "P start", 1: "P tma", 2: "P empty", 3: "P gram issued+norms", 4: "P gram wait",
             5: "P S2 (A, L)", 6: "P substitution", 7: "P T + WU issue", 8: "P WU wait",
             9: "P W conv + full", 10: " sub L1", 11: " sub L2a", 12: " sub L2b",
             13: " sub L3a", 14: " sub L3b", 16: "S start", 17: "S full wait",
             22: "S MMA issue + bulk wait", 18: "S U' wait",
             19: "S Z + HO issue", 20: "S HO wait", 21: "S H/O conv + store"}
    rows = []
    for grp in ([0, 1, 2, 3, 4, 5, 10, 11, 12, 13, 14, 6, 7, 8, 9], [16, 17, 22, 18, 19, 20, 21]):
        for a_, b_ in zip(grp[:-1], grp[1:]):
            dt = (t[2:-2, b_] - t[2:-2, a_])
            rows.append(f"{names[b_]:28s} {dt.mean():9.0f} cycles")
        per = np.diff(t[2:-2, grp[0]]).mean()
        rows.append(f"{'-- per chunk (' + ('P' if grp[0] == 0 else 'S') + ')':28s} {per:9.0f} cycles")
    print("\n" + "\n".join(rows))
