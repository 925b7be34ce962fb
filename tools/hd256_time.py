"""Time the d = 256 (BASELINE configs[3]: B=4 H=8 L=4096) and d = 64 forward
and backward, per kernel, with CUDA events on the launching stream (warm-up
first).  Usage: python tools/hd256_time.py [D ...]"""
import sys

import torch

sys.path.insert(0, '.')
import paper_2406_06484_b200 as dn  # noqa: E402


def clocks():
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
        return (pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h))
    except Exception as e:  # noqa: BLE001
        return (None, str(e))


def run(B, H, L, D, reps=30):
    g = torch.Generator(device='cuda').manual_seed(0)
    mk = lambda: torch.randn((B, H, L, D), device='cuda', generator=g).to(torch.bfloat16)
    q, k, v, dO = mk(), mk(), mk(), mk()
    b = torch.sigmoid(torch.randn((B, H, L), device='cuda', generator=g)).to(torch.bfloat16)
    o, hT, ws = dn.deltanet_fwd(q, k, v, b)
    r = dn.deltanet_bwd(q, k, v, b, dO, workspace=ws)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    tf, tb = [], []
    for _ in range(reps):
        ev[0].record()
        o, hT, ws = dn.deltanet_fwd(q, k, v, b, workspace=ws)
        ev[1].record()
        r = dn.deltanet_bwd(q, k, v, b, dO, workspace=ws)
        ev[2].record()
        torch.cuda.synchronize()
        tf.append(ev[0].elapsed_time(ev[1]))
        tb.append(ev[1].elapsed_time(ev[2]))
    d = dn.make_desc(B, H, L, D, D, 64, torch.bfloat16)
    med = lambda x: sorted(x)[len(x) // 2]
    print(f"B={B} H={H} L={L} d={D} path {dn.deltanet_path(d)}: fwd {med(tf):.4f} ms "
          f"(min {min(tf):.4f}), bwd {med(tb):.4f} ms (min {min(tb):.4f}), "
          f"step {med(tf) + med(tb):.4f} ms; sm clock, throttle {clocks()}", flush=True)


if __name__ == "__main__":
    Ds = [int(x) for x in sys.argv[1:]] or [256, 64]
    for D in Ds:
        if D == 256:
            run(4, 8, 4096, 256)
        elif D == 64:
            run(8, 16, 4096, 64)
        else:
            run(8, 16, 4096, D)
