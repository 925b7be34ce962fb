"""Phase timeline of the split tcgen05 kernels: builds the
library with -DDN_TIMING, runs the d = 256 workload (BASELINE configs[3]) and
prints, per kernel, the mean clock64 offset of each stamp from the start of
the chunk iteration (chain kernels: CTA (0, 0); local kernel: CTA (NC/2, 0)).
Profiling aid, not a test.  Usage: python tools/sp_timeline.py [D]"""
import ctypes
import glob
import os
import subprocess
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2406_06484_b200 as dn  # noqa: E402

FWD = {0: "ctl h_img rcv", 1: "ctl loads ok, U/U'/O issue", 2: "ctl z_ready rcv",
       3: "ctl k/a ok, H issue", 4: "ctl q_done+stores read", 5: "ctl ho_done",
       8: "simt up_done rcv", 9: "simt z_free ok", 10: "simt Z conv + hand-off",
       11: "simt ho_done rcv", 12: "simt st_free ok", 13: "simt H/O conv + hand-off"}
BWD = {0: "ctl dh_img rcv", 1: "ctl k/dO/A ok, dU' issue", 2: "ctl du_ready rcv",
       3: "ctl dv_ready rcv", 4: "ctl q ok, dH issue", 5: "ctl rr_ready rcv",
       6: "ctl dh_done", 8: "simt du_done rcv", 9: "simt st_free(prev) ok",
       10: "simt dU' conv + hand-off", 11: "simt p_done rcv", 12: "simt dV + hand-off",
       13: "simt r_done/v rcv", 14: "simt R/db + hand-off", 15: "simt dh_done rcv",
       16: "simt st_free ok", 17: "simt dH image + hand-off"}


def build():
    out = os.path.join(ROOT, "tests", "cuda", "libdeltanet_sptim.so")
    srcs = sorted(glob.glob(os.path.join(ROOT, "paper_2406_06484_b200", "csrc", "*.cu")))
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                    "--expt-relaxed-constexpr", "-DDN_TIMING", "-Xcompiler", "-fPIC", "-shared",
                    "-I", os.path.join(ROOT, "include"), "-o", out, *srcs], check=True)
    return ctypes.CDLL(out)


def main(D):
    lib = build()
    B, H, L = (4, 8, 4096) if D == 256 else (8, 16, 4096)
    g = torch.Generator(device="cuda").manual_seed(0)
    mk = lambda: torch.randn((B, H, L, D), device="cuda", generator=g).to(torch.bfloat16)
    q, k, v, dO = mk(), mk(), mk(), mk()
    beta = torch.sigmoid(torch.randn((B, H, L), device="cuda", generator=g)).to(torch.bfloat16)
    d = dn.make_desc(B, H, L, D, D, 64, torch.bfloat16)
    ws = torch.empty(dn.deltanet_workspace_bytes(d), dtype=torch.uint8, device="cuda")
    o, dq, dk, dv = (torch.empty_like(q) for _ in range(4))
    db = torch.empty_like(beta)
    P = ctypes.c_void_p
    lib.deltanet_fwd.argtypes = [P] * 9 + [ctypes.c_size_t, P]
    lib.deltanet_bwd.argtypes = [P] * 14 + [ctypes.c_size_t, P]
    lib.sp_timing_set.argtypes = [P, ctypes.c_int]
    NC = L // 64
    buf = torch.zeros(NC * 32, dtype=torch.int64, device="cuda")

    def run():
        assert lib.deltanet_fwd(ctypes.addressof(d), q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                beta.data_ptr(), None, o.data_ptr(), None, ws.data_ptr(),
                                ws.numel(), None) == 0
        assert lib.deltanet_bwd(ctypes.addressof(d), q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                beta.data_ptr(), None, dO.data_ptr(), None, dq.data_ptr(),
                                dk.data_ptr(), dv.data_ptr(), db.data_ptr(), None,
                                ws.data_ptr(), ws.numel(), None) == 0
        torch.cuda.synchronize()

    run()
    for kern, names in ((1, FWD), (2, BWD)):
        buf.zero_()
        assert lib.sp_timing_set(buf.data_ptr(), kern) == 0
        run()
        t = buf.view(NC, 32).cpu().numpy().astype(np.float64)
        base = t[:, 0]
        per = np.diff(base)
        print(f"== {'fwd' if kern == 1 else 'bwd'} chain, d={D}: {per[2:-2].mean():.0f} cycles "
              f"per chunk iteration (CTA 0)")
        for s, name in sorted(names.items()):
            col = t[2:-2, s] - base[2:-2]
            if np.all(t[2:-2, s] == 0):
                continue
            print(f"  {name:32s} {col.mean():8.0f}")
    buf.zero_()
    assert lib.sp_timing_set(buf.data_ptr(), 3) == 0
    run()
    t = buf.view(NC, 32).cpu().numpy().astype(np.float64)
    t0 = t[8, 2]
    print(f"== bwd local, d={D} (CTA NC/2): stamps relative to the CTA start")
    for ss in range(8):
        if t[ss, 0] == 0:
            continue
        print(f"  sub-step {ss}: start {t[ss, 0] - t0:7.0f}  operands in {t[ss, 1] - t0:7.0f}  "
              f"issued {t[ss, 2] - t0:7.0f}")
    lab = ["v_all wait start", "v_all rcv", "dA/dX conv", "Y conv", "G/KK rcv", "G1 conv",
           "k_done rcv", "epilogue"]
    for i, n in enumerate(lab):
        print(f"  simt {n:20s} {t[9, i] - t0:8.0f}")
    print(f"  ctl v_all {t[8, 0] - t0:8.0f}   epi_done {t[8, 1] - t0:8.0f}")
    lib.sp_timing_set(None, 0)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 256)
