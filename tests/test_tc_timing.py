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


@pytest.fixture(scope="module")
def timlib():
    out = os.path.join(HERE, "cuda", "libdeltanet_tim.so")
    srcs = sorted(glob.glob(os.path.join(ROOT, "paper_2406_06484_b200", "csrc", "*.cu")))
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                    "-DDN_TIMING", "-Xcompiler", "-fPIC", "-shared", "-I",
                    os.path.join(ROOT, "include"), "-o", out, *srcs], check=True)
    return ctypes.CDLL(out)


@pytest.mark.skipif(os.environ.get("DN_TIMING") != "1", reason="profiling aid; set DN_TIMING=1")
def test_fwd_timeline(timlib):
    import paper_2406_06484_b200 as dn
    lib = timlib
    # DN_TIMING_CFG=long: the segmented forward (CTA 0 = pass 3's first segment)
    cfg = synth.CONFIGS[os.environ.get("DN_TIMING_CFG", "target")]
    B = int(os.environ.get("DN_TIMING_B", cfg.B))  # full bench batch: HBM contended
    x = synth.make_inputs(cfg, b_range=range(B))
    td = torch.bfloat16
    q, k, v, b = (torch.from_numpy(x[f]).to(td).cuda() for f in ("q", "k", "v", "beta"))
    NC = cfg.L // 64
    buf = torch.zeros(NC * 32, dtype=torch.int64, device="cuda")
    lib.dn_timing_set.argtypes = [ctypes.c_void_p]
    assert lib.dn_timing_set(buf.data_ptr()) == 0
    gated = os.environ.get("DN_TIMING_GATED") == "1"  # the gated forward
    d = dn.make_desc(B, cfg.H, cfg.L, 128, 128, 64, td, gated=gated)
    ws = torch.empty(dn.deltanet_workspace_bytes(d), dtype=torch.uint8, device="cuda")
    o = torch.empty_like(v)
    gate = -0.05 * torch.nn.functional.softplus(torch.randn(b.shape, device="cuda"))
    P = ctypes.c_void_p
    lib.deltanet_fwd.argtypes = [P] * 9 + [ctypes.c_size_t, P]
    lib.deltanet_gated_fwd.argtypes = [P] * 10 + [ctypes.c_size_t, P]
    for _ in range(2):
        if gated:
            rc = lib.deltanet_gated_fwd(ctypes.addressof(d), q.data_ptr(), k.data_ptr(),
                                        v.data_ptr(), b.data_ptr(), gate.data_ptr(), None,
                                        o.data_ptr(), None, ws.data_ptr(), ws.numel(), None)
        else:
            rc = lib.deltanet_fwd(ctypes.addressof(d), q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                  b.data_ptr(), None, o.data_ptr(), None, ws.data_ptr(),
                                  ws.numel(), None)
        assert rc == 0
    torch.cuda.synchronize()
    t = buf.cpu().numpy().reshape(NC, 32).astype(np.int64)
    t = t[:int((t[:, 0] != 0).sum())]  # segmented: CTA 0 walks its segment only
    names = {0: "P start", 1: "P tma+empty wait", 2: "P norms", 3: "P gram wait",
             21: " S2 tmem ld + s", 22: " S2 sync", 23: " S2 A/L writes",
             4: "P S2 sync + gk_free", 10: " sub L1", 15: " T: wu_done(c-1) wait",
             31: " T: writes + fence + sync", 11: " sub L2a", 12: " sub L2b", 13: " sub L3a",
             14: " sub L3b", 5: "P substitution", 6: " T: X record stores", 7: "P WU wait",
             8: "P W conv + full", 16: "S start", 17: "S full/up'/zfree wait", 18: "S Z conv",
             19: "S ho/st wait", 20: "S H/O conv"}
    rows = []
    for grp in ([0, 1, 2, 3, 21, 22, 23, 4, 10, 11, 12, 13, 14, 5, 15, 31, 6, 7, 8],
                [16, 17, 18, 19, 20]):
        for a_, b_ in zip(grp[:-1], grp[1:]):
            dt = (t[2:-2, b_] - t[2:-2, a_])
            rows.append(f"{names[b_]:28s} {dt.mean():9.0f} cycles")
        per = np.diff(t[2:-2, grp[0]]).mean()
        rows.append(f"{'-- per chunk (' + ('P' if grp[0] == 0 else 'S') + ')':28s} {per:9.0f} cycles")
    for s_, nm in ((24, "M t_ready rcv"), (25, "M w_free rcv"), (26, "M bar_empty rcv"),
                   (27, "M v_full rcv"), (28, "M Gram issued (this chunk)"),
                   (29, "W13 Q load issued (this chunk)"), (30, "W13 K load issued (this chunk)")):
        dt = t[2:-2, s_] - t[2:-2, 0]
        rows.append(f"{nm:28s} {dt.mean():9.0f} cycles after prep chunk start")
    print("\n" + "\n".join(rows))


@pytest.mark.skipif(os.environ.get("DN_TIMING") != "1", reason="profiling aid; set DN_TIMING=1")
def test_bwd_timeline(timlib):
    import paper_2406_06484_b200 as dn
    lib = timlib
    cfg = synth.CONFIGS["target"]
    B = int(os.environ.get("DN_TIMING_B", cfg.B))  # full bench batch: HBM contended
    x = synth.make_inputs(cfg, b_range=range(B))
    td = torch.bfloat16
    q, k, v, b, dO = (torch.from_numpy(x[f]).to(td).cuda() for f in ("q", "k", "v", "beta", "dO"))
    NC = cfg.L // 64
    buf = torch.zeros(NC * 32 + B * cfg.H * 4, dtype=torch.int64, device="cuda")
    lib.dn_timing_set_bwd.argtypes = [ctypes.c_void_p]
    assert lib.dn_timing_set_bwd(buf.data_ptr()) == 0
    gated = os.environ.get("DN_TIMING_GATED") == "1"  # the gated backward
    d = dn.make_desc(B, cfg.H, cfg.L, 128, 128, 64, td, gated=gated)
    ws = torch.empty(dn.deltanet_workspace_bytes(d), dtype=torch.uint8, device="cuda")
    o = torch.empty_like(v)
    g = [torch.empty_like(t) for t in (q, k, v, b)]
    gate = -0.05 * torch.nn.functional.softplus(torch.randn(b.shape, device="cuda"))
    dgate = torch.empty_like(gate)
    P = ctypes.c_void_p
    lib.deltanet_fwd.argtypes = [P] * 9 + [ctypes.c_size_t, P]
    lib.deltanet_bwd.argtypes = [P] * 14 + [ctypes.c_size_t, P]
    lib.deltanet_gated_fwd.argtypes = [P] * 10 + [ctypes.c_size_t, P]
    lib.deltanet_gated_bwd.argtypes = [P] * 16 + [ctypes.c_size_t, P]
    for _ in range(2):
        if gated:
            assert lib.deltanet_gated_fwd(ctypes.addressof(d), q.data_ptr(), k.data_ptr(),
                                          v.data_ptr(), b.data_ptr(), gate.data_ptr(), None,
                                          o.data_ptr(), None, ws.data_ptr(), ws.numel(),
                                          None) == 0
            assert lib.deltanet_gated_bwd(ctypes.addressof(d), q.data_ptr(), k.data_ptr(),
                                          v.data_ptr(), b.data_ptr(), gate.data_ptr(), None,
                                          dO.data_ptr(), None, g[0].data_ptr(), g[1].data_ptr(),
                                          g[2].data_ptr(), g[3].data_ptr(), dgate.data_ptr(),
                                          None, ws.data_ptr(), ws.numel(), None) == 0
            continue
        assert lib.deltanet_fwd(ctypes.addressof(d), q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                b.data_ptr(), None, o.data_ptr(), None, ws.data_ptr(),
                                ws.numel(), None) == 0
        assert lib.deltanet_bwd(ctypes.addressof(d), q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                b.data_ptr(), None, dO.data_ptr(), None, g[0].data_ptr(),
                                g[1].data_ptr(), g[2].data_ptr(), g[3].data_ptr(), None,
                                ws.data_ptr(), ws.numel(), None) == 0
    torch.cuda.synchronize()
    allt = buf.cpu().numpy().astype(np.int64)
    t = allt[:NC * 32].reshape(NC, 32)
    cta = allt[NC * 32:].reshape(B * cfg.H, 4)
    dur = (cta[:, 1] - cta[:, 0]) / 1e3
    span = (cta[:, 1].max() - cta[:, 0].min()) / 1e3
    print(f"\nper-CTA bwd duration us: min {dur.min():.1f} median {np.median(dur):.1f} "
          f"max {dur.max():.1f}; kernel span {span:.1f} us; CTA 0 {dur[0]:.1f} us "
          f"(SM {cta[0, 2]}); start skew {(cta[:, 0].max() - cta[:, 0].min()) / 1e3:.1f} us")
    names = {0: "start", 1: "main wait + k norms", 2: "U' conv + R wait", 3: "R conv + Q wait",
             4: "q norms + G wait", 5: "P2 A_m, q/k_hat, dU wait", 6: "P3 dU' conv",
             7: "P wait", 8: "P5 P, dV, dX", 9: "P5b dH image", 10: "A wait",
             11: "P6 dA, Y", 12: "G wait", 13: "P7 G1, dbeta", 14: "K wait",
             15: "P8 dq/dk epilogue"}
    rows = []
    seq = list(range(16))
    for a_, b_ in zip(seq[:-1], seq[1:]):
        dt = (t[2:-2, b_] - t[2:-2, a_])
        rows.append(f"{names[b_]:28s} {dt.mean():9.0f} cycles")
    rows.append(f"{'-- per chunk':28s} {np.diff(t[2:-2, 0]).mean():9.0f} cycles")
    # issuer stamps (slots 16-29), relative to the SIMT chunk start (slot 0)
    inames = {16: "I main+dHimg rcv", 17: "I K H issued (MB_R)", 18: "I (stamp only)",
              19: "I dH^T K^T issued", 20: "I A rcv", 21: "I P3 rcv", 22: "I M3/M4 issued",
              23: "I P5 rcv", 24: "I M5a+dQ issued", 25: "I P6 rcv", 26: "I M6 issued",
              27: "I P7 rcv"}
    for s_ in range(16, 28):
        dt = t[2:-2, s_] - t[2:-2, 0]
        rows.append(f"{inames[s_]:28s} {dt.mean():9.0f} cycles after chunk start")
    if gated:  # sub-phase stamps of the gated path
        for s_, a_, nm in ((31, 7, "P5 gated DD + D rescale"), (28, 10, "P6 T1 sums + dS"),
                           (11, 28, "P6 dO scale + signal")):
            rows.append(f"{nm:28s} {(t[2:-2, s_] - t[2:-2, a_]).mean():9.0f} cycles")
    print("\n" + "\n".join(rows))
