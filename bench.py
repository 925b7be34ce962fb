#!/usr/bin/env python
"""Benchmark: tokens/s of forward+backward of one DeltaNet layer
(H=16, d=128, L=4096, C=64, bf16 I/O, fp32 accumulate) on 1..8 B200.

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]

One "step" = deltanet_fwd (save states) + deltanet_bwd over one batch of
synthetic inputs resident in HBM, i.e. every row of SURVEY §8(a).  Each rank
owns B=8 batch rows (weak scaling: per-GPU work fixed; at N=8 this is the
BASELINE "sharded" B=64 config).  The (b, h) units are independent, so there
is no collective in the timed region; the NCCL all-gather of outputs and
gradients (north_star) is timed separately and reported as "gather".  The
sharding, the step and the gather are paper_2406_06484_b200.data_parallel
(the code the gloo tests drive).  A second record, "strong_scaling", runs
BASELINE configs[4] as stated -- B=64 in total, 64/N rows per rank -- so at
N=1 it is the single-GPU B=64 (1024-unit) measurement.

`python bench.py --gpus N` without a torchrun environment re-launches itself
under torch.distributed.run with N processes (127.0.0.1 rendezvous).

Prints ONE JSON line on rank 0 (contract in the task statement / DESIGN.md).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "tokens/s fwd+bwd DeltaNet layer (H=16,d=128,L=4K) at 1/2/4/8 B200; % bf16 TC peak"
B_PER_RANK, H, L, D, C = 8, 16, 4096, 128, 64


# unit slabs of the host-buffer pipeline in the e2e leg
E2E_SLABS = int(os.environ.get("DELTANET_E2E_SLABS", "8"))  # 8 measured best (8..64)


def per_token_head(dk, dv, c, s):
    """Algorithmic work per token x head."""
    f_fwd = 6 * dk * dv + 2 * c * (3 * dk + 2 * dv) + c * c / 3
    f_bwd = 12 * dk * dv + 2 * c * (6 * dk + 4 * dv) + 4 * c * c
    b_fwd = s * (2 * dk + 2 * dv + 1)          # read q,k,v,beta; write o
    b_bwd = s * (4 * dk + 3 * dv + 2)          # read q,k,v,beta,dO; write dq,dk,dv,dbeta
    return f_fwd, f_bwd, b_fwd, b_bwd


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        j = json.load(open(p))
        return {"hbm_gbs": j["hbm_gbs"], "tf_burst": j["bf16_tflops"],
                "tf_sustained": j.get("bf16_tflops_sustained", j["bf16_tflops"]),
                "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "tf_burst": 1590.0, "tf_sustained": 1400.0,
            "source": "fallback (B200_PROFILING.md)"}


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region
    (B200_PROFILING.md clocks line).  NVML (the library nvidia-smi reads)
    polled every 5 ms from a thread, so even a ~20 ms timed region gets
    several samples; samples outside [begin(), end()] are dropped."""
    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
               "hw_thermal_slowdown": 0x40, "sw_power_cap": 0x4}

    def __init__(self, device):
        self.device = device
        self.rows = []
        self.window = [None, None]
        self.ok = False
        self.err = None

    def start(self):
        import threading
        try:
            import pynvml as nv
            import torch
            nv.nvmlInit()
            props = torch.cuda.get_device_properties(self.device)
            h = None
            bus = getattr(props, "pci_bus_id", None)
            if bus is not None:
                dom = getattr(props, "pci_domain_id", 0)
                dev_ = getattr(props, "pci_device_id", 0)
                try:
                    h = nv.nvmlDeviceGetHandleByPciBusId(f"{dom:08x}:{bus:02x}:{dev_:02x}.0")
                except Exception:
                    h = None
            if h is None:
                h = nv.nvmlDeviceGetHandleByIndex(self.device.index or 0)
            self.nv, self.h = nv, h
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # no NVML: report it, never guess a clock
            self.err = f"nvml unavailable: {type(e).__name__}"
            return
        self.stop_flag = False

        def loop():
            nv, h = self.nv, self.h
            get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                nv.nvmlDeviceGetCurrentClocksThrottleReasons
            while not self.stop_flag:
                try:
                    self.rows.append((time.perf_counter(), nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM),
                                      nv.nvmlDeviceGetPowerUsage(h) / 1000.0, int(get_reasons(h))))
                except Exception:
                    pass
                time.sleep(0.005)
        self.thread = threading.Thread(target=loop, daemon=True)
        self.thread.start()

    def sample_now(self):
        """One synchronous sample from the calling thread."""
        if not self.ok:
            return
        nv, h = self.nv, self.h
        get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        try:
            self.rows.append((time.perf_counter(), nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM),
                              nv.nvmlDeviceGetPowerUsage(h) / 1000.0, int(get_reasons(h))))
        except Exception:
            pass

    def poll_until(self, event):
        """Sample from the launching thread while the GPU runs the queued
        timed region (the sampler thread may be starved of the GIL)."""
        while not event.query():
            self.sample_now()
            time.sleep(0.002)

    def begin(self):
        self.window[0] = time.perf_counter()

    def end(self):
        self.window[1] = time.perf_counter()

    def stop(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [self.err], "samples": 0}
        self.stop_flag = True
        self.thread.join(timeout=2)
        t0, t1 = self.window
        rows = [r for r in self.rows if t0 is not None and t0 <= r[0] <= (t1 or r[0])]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        sm = sorted(r[1] for r in rows)
        reasons = sorted(n for n, bit in self.REASONS.items() if any(r[3] & bit for r in rows))
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(rows), "power_w_max": max(r[2] for r in rows), "source": "nvml"}


# fp32 CUDA-core roofline of the recurrent kernel: 148 SMs x 4
# SMSPs x 32 lanes / FFMA reciprocal throughput 2 cycles (3-register form,
# B300_MICROARCH.md "Pipe rates") x 2 flop x 1965 MHz
FP32_FFMA_TFLOPS = 148 * 4 * 32 / 2 * 2 * 1.965e9 / 1e12


def measure_recurrent(dn, dev, q, k, v, beta, t_fwd_chunk, peaks):
    """Side measurement (outside the timed step) of deltanet_recurrent_fwd:
    (1) the same prefill workload as the step's forward -- the paper's
    recurrent-vs-chunkwise kernel comparison (fig:kernel_speed);
    (2) decode: one token for B=64 x H=16 sequences, state updated in place."""
    import torch
    stream = torch.cuda.current_stream(dev)

    def timed(fn, reps):
        fn()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        return e0.elapsed_time(e1) * 1e-3 / reps

    B, Hh, Ll, Dk = q.shape
    Dv = v.shape[-1]
    o = torch.empty_like(v)
    t_pre = timed(lambda: dn.deltanet_recurrent_fwd(q, k, v, beta, out=o, want_hT=False), 3)
    flops = 3 * 2 * Dk * Dv * B * Hh * Ll
    prefill = {"workload": f"B={B} H={Hh} L={Ll} d={Dk} (the step's forward)",
               "ms": t_pre * 1e3, "tokens_per_s": B * Ll / t_pre,
               "chunkwise_fwd_ms": t_fwd_chunk * 1e3,
               "chunkwise_speedup": t_pre / t_fwd_chunk,
               "roofline": {"bound": "alu", "achieved": flops / t_pre / 1e12,
                            "peak": FP32_FFMA_TFLOPS, "unit": "TFLOP/s",
                            "frac": flops / t_pre / 1e12 / FP32_FFMA_TFLOPS,
                            "peak_source": "derived: 148 SM x 128 FFMA lanes / 2-cycle rt x 2 x 1.965 GHz"}}
    Bd = 64
    g = torch.Generator(device=dev).manual_seed(7)
    qd = torch.randn((Bd, Hh, 1, Dk), device=dev, generator=g).to(q.dtype)
    kd = torch.randn((Bd, Hh, 1, Dk), device=dev, generator=g).to(q.dtype)
    vd = torch.randn((Bd, Hh, 1, Dv), device=dev, generator=g).to(q.dtype)
    bd = torch.rand((Bd, Hh, 1), device=dev, generator=g).to(q.dtype)
    state = torch.zeros((Bd, Hh, Dk, Dv), dtype=torch.float32, device=dev)
    od = torch.empty_like(vd)
    t_dec = timed(lambda: dn.deltanet_recurrent_fwd(qd, kd, vd, bd, h0=state, hT=state, out=od),
                  50)
    nbytes = 2 * state.numel() * 4 + sum(t.numel() * t.element_size() for t in (qd, kd, vd, bd, od))
    decode = {"workload": f"B={Bd} H={Hh} one token, fp32 state in place",
              "us_per_token_step": t_dec * 1e6, "tokens_per_s": Bd / t_dec,
              "roofline": {"bound": "hbm", "achieved": nbytes / t_dec / 1e9,
                           "peak": peaks["hbm_gbs"], "unit": "GB/s",
                           "frac": nbytes / t_dec / 1e9 / peaks["hbm_gbs"],
                           "bytes_per_step": nbytes}}
    return {"kernel": "deltanet_recurrent_fwd (CUDA cores, fp32 state)", "prefill": prefill,
            "decode": decode}


def measure_prologue(dn, dev, B, H, L, D, peaks):
    """Side measurement (outside the timed step) of the layer prologue
    (SURVEY §8(f) f1): short conv + SiLU + sigmoid + layout change, forward
    and backward, on the step's shapes; HBM-bound (bytes = tensors read and
    written once)."""
    import torch
    stream = torch.cuda.current_stream(dev)
    g = torch.Generator(device=dev).manual_seed(11)
    xs = [torch.randn((B, L, H, D), device=dev, generator=g).to(torch.bfloat16) for _ in range(3)]
    xb = torch.randn((B, L, H), device=dev, generator=g).to(torch.bfloat16)
    ws = [0.5 * torch.randn((H * D, 4), device=dev, generator=g) for _ in range(3)]
    outs = dn.deltanet_prologue_fwd(*xs, xb, *ws)
    gr = [torch.randn_like(t) for t in outs]
    gouts = dn.deltanet_prologue_bwd(*xs, xb, *ws, *gr)

    def timed(fn, reps=10):
        fn()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        return e0.elapsed_time(e1) * 1e-3 / reps

    nb = lambda ts: sum(t.numel() * t.element_size() for t in ts)
    t_f = timed(lambda: dn.deltanet_prologue_fwd(*xs, xb, *ws, out=outs))
    t_b = timed(lambda: dn.deltanet_prologue_bwd(*xs, xb, *ws, *gr, out=gouts))
    bf = nb(xs) + nb([xb]) + nb(outs)
    bb = nb(xs) + nb([xb]) + nb(gr) + nb(gouts[:4])
    roof = lambda by, t: {"bound": "hbm", "achieved": by / t / 1e9, "peak": peaks["hbm_gbs"],
                          "unit": "GB/s", "frac": by / t / 1e9 / peaks["hbm_gbs"],
                          "bytes": by}
    return {"kernel": "deltanet_prologue_fwd / _bwd (short conv 4 + SiLU + sigmoid + layout)",
            "workload": f"B={B} H={H} L={L} d={D} bf16",
            "fwd_ms": t_f * 1e3, "bwd_ms": t_b * 1e3,
            "fwd_roofline": roof(bf, t_f), "bwd_roofline": roof(bb, t_b)}


def measure_long_context(dn, dev):
    """Side measurement (outside the timed step): BASELINE configs[2], the
    long-context shape B=2 H=16 L=16384 (32 units on 148 SMs), fwd+bwd with
    the segment-parallel kernels and with one CTA per unit."""
    import torch
    stream = torch.cuda.current_stream(dev)
    B, Hh, Ll, D = 2, 16, 16384, 128
    g = torch.Generator(device=dev).manual_seed(13)
    mk = lambda: torch.randn((B, Hh, Ll, D), device=dev, generator=g).to(torch.bfloat16)
    q, k, v, dO = mk(), mk(), mk(), mk()
    beta = torch.rand((B, Hh, Ll), device=dev, generator=g).to(torch.bfloat16)
    o = torch.empty_like(v)
    grads = (torch.empty_like(q), torch.empty_like(k), torch.empty_like(v),
             torch.empty_like(beta))
    res = {"workload": f"B={B} H={Hh} L={Ll} d={D} chunk=64 bf16 fwd+bwd"}
    for seg in (True, False):
        d = dn.make_desc(B, Hh, Ll, D, D, 64, torch.bfloat16, segments=seg)
        ws = dn.alloc_workspace(d, dev)

        def step():
            dn.deltanet_fwd(q, k, v, beta, workspace=ws, want_hT=False, out=o, segments=seg)
            dn.deltanet_bwd(q, k, v, beta, dO, workspace=ws, want_dh0=False, out=grads,
                            segments=seg)
        step()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(5):
            step()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        t = e0.elapsed_time(e1) * 1e-3 / 5
        res["segmented" if seg else "one_cta_per_unit"] = {
            "ms_per_step": t * 1e3, "tokens_per_s": B * Ll / t,
            "launches": dn.deltanet_launch_count(d, 0) + dn.deltanet_launch_count(d, 1)}
    return res


def _timed(dev, fn, reps):
    import torch
    stream = torch.cuda.current_stream(dev)
    fn()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    return e0.elapsed_time(e1) * 1e-3 / reps


def measure_gated(dn, dev, q, k, v, beta, t_fwd_ungated, t_bwd_ungated):
    """Side measurement (outside the timed step) of Gated DeltaNet (SURVEY
    §8(f) f4): the tcgen05 gated forward and backward on the
    step's workload (gates g = -0.05 softplus(N(0,1)), dO ~ N(0,1)); the
    backward reads the forward's saved records like the ungated step."""
    import torch
    B, Hh, Ll, D = q.shape
    gen = torch.Generator(device=dev).manual_seed(17)
    gates = -0.05 * torch.nn.functional.softplus(
        torch.randn((B, Hh, Ll), device=dev, generator=gen))
    dO = torch.randn(v.shape, device=dev, generator=gen).to(v.dtype)
    o = torch.empty_like(v)
    d = dn.make_desc(B, Hh, Ll, D, D, 64, torch.bfloat16, gated=True)
    ws = dn.alloc_workspace(d, dev)
    t_f = _timed(dev, lambda: dn.deltanet_gated_fwd(q, k, v, beta, gates, workspace=ws, out=o,
                                                    want_hT=False), 5)
    t_b = _timed(dev, lambda: dn.deltanet_gated_bwd(q, k, v, beta, gates, dO, workspace=ws,
                                                    want_dh0=False), 5)
    wl = f"B={B} H={Hh} L={Ll} d={D} bf16 (the step's workload)"
    return {"fwd": {"workload": wl, "kernel": "tc_fwd_kernel<false, true> (tcgen05)",
                    "ms": t_f * 1e3, "tokens_per_s": B * Ll / t_f,
                    "vs_ungated_fwd": t_f / t_fwd_ungated,
                    "launches": dn.deltanet_launch_count(d, 0)},
            "bwd": {"workload": wl, "kernel": "tc_bwd_kernel<false, true> (tcgen05)",
                    "ms": t_b * 1e3, "tokens_per_s": B * Ll / t_b,
                    "vs_ungated_bwd": t_b / t_bwd_ungated,
                    "launches": dn.deltanet_launch_count(d, 1)},
            "fwd_bwd_tokens_per_s": B * Ll / (t_f + t_b)}


def measure_context_parallel(dn, dev, parts=2):
    """Side measurement (outside the timed step) of context parallelism
     on BASELINE configs[2] (B=2 H=16 L=16384), `parts`
    simulated ranks on this GPU: the per-rank kernels (transition, scan,
    fwd / bwd of its L/parts tokens from the scanned state) timed on the last
    part, against the whole sequence on one GPU.  The all-gather of the
    transitions (2 x 64 KB per unit per rank) is not included."""
    import torch
    B, Hh, Ll, D = 2, 16, 16384, 128
    Lp = Ll // parts
    g = torch.Generator(device=dev).manual_seed(19)
    mk = lambda L_: torch.randn((B, Hh, L_, D), device=dev, generator=g).to(torch.bfloat16)
    q, k, v, dO = mk(Lp), mk(Lp), mk(Lp), mk(Lp)
    beta = torch.rand((B, Hh, Lp), device=dev, generator=g).to(torch.bfloat16)
    d = dn.make_desc(B, Hh, Lp, D, D, 64, torch.bfloat16)
    ws = dn.alloc_workspace(d, dev)
    psi, hloc = dn.deltanet_fwd_transition(q, k, v, beta, workspace=ws)
    psi_all = torch.stack([psi] * parts)
    loc_all = torch.stack([hloc] * parts)
    o = torch.empty_like(v)
    grads = (torch.empty_like(q), torch.empty_like(k), torch.empty_like(v),
             torch.empty_like(beta))
    hs = torch.empty((B, Hh, D, D), dtype=torch.float32, device=dev)
    de = torch.empty_like(hs)
    dloc = torch.empty_like(hs)

    def rank_step():
        dn.deltanet_fwd_transition(q, k, v, beta, psi=psi, hloc=hloc, workspace=ws)
        dn.deltanet_state_scan(psi_all, loc_all, parts - 1, out=hs)
        dn.deltanet_fwd(q, k, v, beta, h0=hs, workspace=ws, want_hT=False, out=o)
        dn.deltanet_bwd_transition(q, k, v, beta, dO, workspace=ws, dhloc=dloc)
        dn.deltanet_state_scan(psi_all, loc_all, parts - 1, reverse=True, out=de)
        dn.deltanet_bwd(q, k, v, beta, dO, h0=hs, dhT=de, workspace=ws, want_dh0=False,
                        out=grads)
    t_rank = _timed(dev, rank_step, 5)
    t_tr = _timed(dev, lambda: dn.deltanet_fwd_transition(q, k, v, beta, psi=psi, hloc=hloc, workspace=ws), 5)
    t_btr = _timed(dev, lambda: dn.deltanet_bwd_transition(q, k, v, beta, dO, workspace=ws,
                                                           dhloc=dloc), 5)
    return {"workload": f"B={B} H={Hh} L={Ll} d={D}, {parts} parts of {Lp} tokens",
            "per_rank_ms": t_rank * 1e3,
            "fwd_transition_ms": t_tr * 1e3, "bwd_transition_ms": t_btr * 1e3,
            "transition_launches": [dn.deltanet_launch_count(d, 5),
                                    dn.deltanet_launch_count(d, 6)],
            "projected_tokens_per_s": parts * B * Lp / t_rank,
            "note": "per-rank kernel time of one simulated rank; excludes the NCCL all-gather"}


def _free_port():
    import socket
    s_ = socket.socket()
    s_.bind(("127.0.0.1", 0))
    p = s_.getsockname()[1]
    s_.close()
    return p


def relaunch_distributed(n):
    """--gpus N > 1 outside torchrun: run this script under
    torch.distributed.run with N local ranks and return its exit code."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr", "127.0.0.1",
           "--master-port", str(_free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def _synthetic_rows(dev, rows, Hh, Ll, Dd, seed0):
    """Seeded inputs of the paper's distributions (DESIGN.md input recipe:
    q, k ~ SiLU(N(0,1)), v, dO ~ N(0,1), beta ~ sigmoid(N(0,1))), generated on
    the device one batch row at a time (seed0 + b), so a row's data does not
    depend on how the batch is sharded; timing-only records."""
    import torch
    f = torch.nn.functional
    parts = {n: [] for n in ("q", "k", "v", "beta", "dO")}
    for b in rows:
        g = torch.Generator(device=dev).manual_seed(seed0 + b)
        rn = lambda *shape: torch.randn(shape, device=dev, generator=g)
        parts["q"].append(f.silu(rn(1, Hh, Ll, Dd)))
        parts["k"].append(f.silu(rn(1, Hh, Ll, Dd)))
        parts["v"].append(rn(1, Hh, Ll, Dd))
        parts["beta"].append(torch.sigmoid(rn(1, Hh, Ll)))
        parts["dO"].append(rn(1, Hh, Ll, Dd))
    return [torch.cat(parts[n], 0).to(torch.bfloat16).contiguous()
            for n in ("q", "k", "v", "beta", "dO")]


def _time_steps(dev, step, reps, warm=2):
    import torch
    import torch.distributed as dist
    stream = torch.cuda.current_stream(dev)
    for _ in range(warm):
        step.step()
    torch.cuda.synchronize(dev)
    if dist.is_initialized():
        dist.barrier()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        step.step()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    return e0.elapsed_time(e1) * 1e-3 / reps


def measure_strong_scaling(dp, dev, ws, rank, reps=5):
    """BASELINE configs[4] as stated: B=64 H=16 L=4096 in total over the N
    ranks (shard_rows: 64/N batch rows = 1024/N units per GPU), fwd+bwd,
    device time max over ranks.  At N=1 this is the single-GPU B=64 record
    (1024 units, ~6.9 waves of 148 SMs) against which the 8-GPU shard
    (128 units, 0.86 of a wave) is compared (SURVEY §8(e) strong-scaling
    risk).  Not the headline: every rank runs it after the timed step."""
    B_total = 64
    rows = dp.shard_rows(B_total, ws, rank)
    q, k, v, beta, dO = _synthetic_rows(dev, rows, H, L, D, 4000)
    step = dp.ShardedStep(q, k, v, beta, dO, B_total=B_total, chunk=C)
    t, = dp.max_over_ranks([_time_steps(dev, step, reps)], dev)
    ff, fb, _, _ = per_token_head(D, D, C, 2)
    units = len(rows) * H
    del step, q, k, v, beta, dO
    return {"workload": f"B={B_total} total (BASELINE configs[4]) H={H} L={L} d={D} chunk={C} "
                        f"bf16 fwd+bwd, {len(rows)} rows = {units} units per GPU",
            "scaling": "strong", "n_gpus": ws, "ms_per_step": t * 1e3,
            "tokens_per_s": B_total * L / t, "units_per_gpu": units,
            "sm_waves_per_gpu": units / 148.0,
            "tc_peak_frac_per_gpu": (ff + fb) * units * L / t / 1634.4e12,
            "data": "synthetic, seeded per batch row on the device (timing only)"}


def measure_1p3b(dn, dp, dev, reps=10):
    """BASELINE configs[1]: the 1.3B-shaped layer B=8 H=16 d=128 L=2048 C=64
    (the paper's 2K x 8 training setting), fwd+bwd on one
    GPU (side record, rank 0)."""
    B = 8
    Ll = 2048
    q, k, v, beta, dO = _synthetic_rows(dev, range(B), H, Ll, D, 1000)
    step = dp.ShardedStep(q, k, v, beta, dO, B_total=B, chunk=C, local=True)  # rank 0 alone
    import torch
    stream = torch.cuda.current_stream(dev)
    for _ in range(2):
        step.step()
    torch.cuda.synchronize(dev)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    tf = tb = 0.0
    for _ in range(reps):
        ev[0].record(stream)
        step.fwd()
        ev[1].record(stream)
        step.bwd()
        ev[2].record(stream)
        torch.cuda.synchronize(dev)
        tf += ev[0].elapsed_time(ev[1]) * 1e-3 / reps
        tb += ev[1].elapsed_time(ev[2]) * 1e-3 / reps
    ff, fb, _, _ = per_token_head(D, D, C, 2)
    t = tf + tb
    return {"workload": f"B={B} H={H} L={Ll} d={D} chunk={C} bf16 fwd+bwd (BASELINE configs[1])",
            "ms_per_step": t * 1e3, "ms_fwd": tf * 1e3, "ms_bwd": tb * 1e3,
            "tokens_per_s": B * Ll / t,
            "tc_peak_frac": (ff + fb) * B * H * Ll / t / 1634.4e12}


def measure_head_dims(dn, dev, peaks, reps=20):
    """BASELINE configs[3] (head_dim 256: B=4 H=8 L=4096) and the d_head = 64
    column of fig:kernel_speed (B=8 H=16 L=4096), fwd+bwd
    on the split tcgen05 kernels, side records (rank 0).
    Roofline: at d = 256 the layer is tensor-bound on paper (AI ~300 flop/B
    above the ridge), at d = 64 HBM-bound."""
    import torch
    out = {}
    for name, (Bb, Hh, Ll, Dd) in (("hd256", (4, 8, 4096, 256)), ("d64", (8, 16, 4096, 64))):
        q, k, v, beta, dO = _synthetic_rows(dev, range(Bb), Hh, Ll, Dd, 3000)
        o, hT, ws = dn.deltanet_fwd(q, k, v, beta)
        dn.deltanet_bwd(q, k, v, beta, dO, workspace=ws)
        torch.cuda.synchronize(dev)
        stream = torch.cuda.current_stream(dev)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        tf, tb = [], []
        for _ in range(reps):
            ev[0].record(stream)
            dn.deltanet_fwd(q, k, v, beta, workspace=ws)
            ev[1].record(stream)
            dn.deltanet_bwd(q, k, v, beta, dO, workspace=ws)
            ev[2].record(stream)
            torch.cuda.synchronize(dev)
            tf.append(ev[0].elapsed_time(ev[1]) * 1e-3)
            tb.append(ev[1].elapsed_time(ev[2]) * 1e-3)
        med = lambda x: sorted(x)[len(x) // 2]
        t_f, t_b = med(tf), med(tb)
        t = t_f + t_b
        ff, fb, bf, bb = per_token_head(Dd, Dd, C, 2)
        n = Bb * Hh * Ll
        flops, byts = (ff + fb) * n, (bf + bb) * n
        t_tc, t_hbm = flops / (peaks["tf_burst"] * 1e12), byts / (peaks["hbm_gbs"] * 1e9)
        bound = "tensor" if t_tc >= t_hbm else "hbm"
        roof = ({"bound": "tensor", "achieved": flops / t / 1e12, "peak": peaks["tf_burst"],
                 "unit": "TFLOP/s", "frac": t_tc / t} if bound == "tensor" else
                {"bound": "hbm", "achieved": byts / t / 1e9, "peak": peaks["hbm_gbs"],
                 "unit": "GB/s", "frac": t_hbm / t})
        roof["floor_ms"] = max(t_tc, t_hbm) * 1e3
        d = dn.make_desc(Bb, Hh, Ll, Dd, Dd, C, torch.bfloat16)
        out[name] = {"workload": f"B={Bb} H={Hh} L={Ll} d={Dd} chunk={C} bf16 fwd+bwd",
                     "kernel_path": {2: "tcgen05 split", 1: "tcgen05 fused"}.get(
                         dn.deltanet_path(d), "simt"),
                     "launches": dn.deltanet_launch_count(d, 0) + dn.deltanet_launch_count(d, 1),
                     "ms_per_step": t * 1e3, "ms_fwd": t_f * 1e3, "ms_bwd": t_b * 1e3,
                     "tokens_per_s": Bb * Ll / t, "tc_peak_frac": flops / t / 1634.4e12,
                     "roofline": roof}
        del q, k, v, beta, dO, o, ws
        torch.cuda.empty_cache()
    return out


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def run_reference(args, ws, rank):
    """--impl reference: the fp64 oracle (the only 'reference' this paper
    has) timed on the host cores on a bounded sample of the same workload."""
    if rank != 0:
        return
    import numpy as np
    import oracle
    import synth
    cfg = synth.CONFIGS["sharded"]
    nthreads = oracle.default_threads()
    n_units = max(1, min(nthreads, 16))
    units = [(u // H, u % H) for u in range(n_units)]
    inp = synth.make_inputs(cfg, units=units)

    def step():
        oracle.recurrent_fwd(inp["q"], inp["k"], inp["v"], inp["beta"], nthreads=nthreads)
        oracle.recurrent_bwd(inp["q"], inp["k"], inp["v"], inp["beta"], inp["dO"],
                             nthreads=nthreads)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    t = (time.perf_counter() - t0) / args.steps
    # tokens/s of the metric: a step covers all H heads of B*L tokens, so the
    # sampled n_units unit-sequences are n_units/H of a B=1 step.
    value = n_units * L / H / t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "deltanet_layer_fwd_bwd", "B_per_gpu": B_PER_RANK, "H": H,
                   "L": L, "Dk": D, "Dv": D, "chunk": C, "io": "bf16-rounded inputs, fp64 oracle"},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": nthreads, "kind": "oracle",
                         "sample": f"{n_units} of the {B_PER_RANK * H} (b,h) units per step, "
                                   f"full L={L}, fwd+bwd, fp64 C oracle"},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(budget_s=12.0):
    """Oracle as it stands on the host cores, bounded sample (rank 0, N=1)."""
    import oracle
    import synth
    cfg = synth.CONFIGS["sharded"]
    nthreads = oracle.default_threads()
    n_units = nthreads
    units = [(u // H, u % H) for u in range(n_units)]
    inp = synth.make_inputs(cfg, units=units)
    reps, t_tot = 0, 0.0
    while t_tot < budget_s and reps < 8:
        t0 = time.perf_counter()
        oracle.recurrent_fwd(inp["q"], inp["k"], inp["v"], inp["beta"], nthreads=nthreads)
        oracle.recurrent_bwd(inp["q"], inp["k"], inp["v"], inp["beta"], inp["dO"],
                             nthreads=nthreads)
        t_tot += time.perf_counter() - t0
        reps += 1
    t = t_tot / reps
    return {"value": n_units * L / H / t, "unit": "tokens/s", "cores": nthreads,
            "kind": "oracle",
            "sample": f"{n_units} (b,h) units x full L={L} fwd+bwd per rep, {reps} reps, "
                      f"{t_tot:.1f} s; scaled to tokens/s as units*L/H/t"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--force-simt", action="store_true")
    ap.add_argument("--no-recurrent", action="store_true",
                    help="skip the recurrent-form (SURVEY §8(f) f2) side measurement")
    ap.add_argument("--no-strong", action="store_true",
                    help="skip the configs[4] strong-scaling record (B=64 total)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_distributed(args.gpus))
    ws, rank, local = dist_env()
    if args.gpus != ws and rank == 0:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}; using {ws}", file=sys.stderr)

    if args.impl == "reference":
        return run_reference(args, ws, rank)

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2406_06484_b200 as dn
    from paper_2406_06484_b200 import data_parallel as dp
    import synth

    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs CUDA devices (no CPU path)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)
    dn.load_library()

    cfg = synth.CONFIGS["sharded"]
    B_total = B_PER_RANK * ws          # weak scaling: 8 batch rows per rank
    rows = dp.shard_rows(B_total, ws, rank)
    host = synth.make_inputs(cfg, b_range=rows)
    td = torch.bfloat16
    q, k, v, beta, dO = (torch.from_numpy(host[f]).to(td).to(dev).contiguous()
                         for f in ("q", "k", "v", "beta", "dO"))
    desc = dn.make_desc(B_PER_RANK, H, L, D, D, C, td, l2norm=True, save_states=True,
                        force_simt=args.force_simt)
    ops = None
    if args.force_simt:
        from types import SimpleNamespace
        ops = SimpleNamespace(
            fwd=lambda *a_, **kw: dn.deltanet_fwd(*a_, force_simt=True, **kw),
            bwd=lambda *a_, **kw: dn.deltanet_bwd(*a_, force_simt=True, **kw),
            alloc=lambda q_, v_, c_: dn.alloc_workspace(desc, dev))
    step = dp.ShardedStep(q, k, v, beta, dO, B_total=B_total, chunk=C, ops=ops)
    o, grads = step.o, step.grads
    path = dn.deltanet_path(desc)
    n_launch = dn.deltanet_launch_count(desc, 0) + dn.deltanet_launch_count(desc, 1)
    stream = torch.cuda.current_stream(dev)
    fwd, bwd = step.fwd, step.bwd

    clocks = ClockSampler(dev)
    clocks.start()
    for _ in range(args.warmup):
        fwd()
        bwd()
    torch.cuda.synchronize(dev)
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    clocks.begin()
    for i in range(args.steps):
        ev[i][0].record(stream)
        fwd()
        ev[i][1].record(stream)
        bwd()
        ev[i][2].record(stream)
    clocks.poll_until(ev[-1][2])
    torch.cuda.synchronize(dev)
    clocks.end()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    t_fwd = sum(e[0].elapsed_time(e[1]) for e in ev) / args.steps * 1e-3
    t_bwd = sum(e[1].elapsed_time(e[2]) for e in ev) / args.steps * 1e-3
    t_total = ev[0][0].elapsed_time(ev[-1][2]) * 1e-3
    t_step = t_total / args.steps
    t_step, t_fwd, t_bwd = dp.max_over_ranks([t_step, t_fwd, t_bwd], dev)

    tokens_per_step = B_PER_RANK * ws * L
    value = tokens_per_step / t_step
    peaks = load_peaks()
    s = 2
    ff, fb, bf, bb = per_token_head(D, D, C, s)
    th = B_PER_RANK * H * L  # token-heads per rank per step
    # dominant kernel call and its binding roofline
    dom = ("bwd", t_bwd, fb * th, bb * th) if t_bwd >= t_fwd else ("fwd", t_fwd, ff * th, bf * th)
    name, t_k, F_k, B_k = dom
    long_region = t_total > 1.0
    tf_peak = peaks["tf_sustained"] if long_region else peaks["tf_burst"]
    t_tc, t_hbm = F_k / (tf_peak * 1e12), B_k / (peaks["hbm_gbs"] * 1e9)
    if t_hbm >= t_tc:
        roof = {"bound": "hbm", "achieved": B_k / t_k / 1e9, "peak": peaks["hbm_gbs"],
                "unit": "GB/s"}
    else:
        roof = {"bound": "tensor", "achieved": F_k / t_k / 1e12, "peak": tf_peak,
                "unit": "TFLOP/s"}
    roof["frac"] = roof["achieved"] / roof["peak"]
    roof["traffic"] = None
    tj = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    kname = f"tc_{name}_kernel"
    if path == 1 and os.path.exists(tj):
        tjs = json.load(open(tj))
        tr = tjs.get(kname)
        if tr:  # DRAM bytes per launch of this kernel from the committed ncu capture
            from paper_2406_06484_b200.build import sources_sha
            cap = tr["dram_read_bytes"] + tr["dram_write_bytes"]
            fresh = tjs.get("sources_sha16") == sources_sha()
            # a capture of other kernel sources is not this kernel's traffic
            roof["traffic"] = cap if fresh else None
            roof["traffic_unit"] = "bytes/launch (ncu dram__bytes_read+write, profiles/)"
            roof["traffic_capture"] = {"bytes": cap, "sources_sha16": tjs.get("sources_sha16"),
                                       "benched_sources_sha16": sources_sha(),
                                       "stale": not fresh,
                                       "git_head_at_summary": tjs.get("git_head_at_summary")}
            roof["algorithmic_bytes_per_launch"] = B_k
    roof["kernel"] = f"deltanet_{name} ({'tcgen05' if path == 1 else 'simt'} path)"
    roof["peak_source"] = peaks["source"] + (" sustained" if roof["bound"] == "tensor" and long_region else "")
    roof["algorithmic_per_token_head"] = {"flops": F_k / th, "bytes": B_k / th}

    tc_frac = (ff + fb) * th * ws / t_step / (peaks["tf_burst"] * 1e12) / ws

    # ---- e2e through the public API with host buffers (pinned), per step:
    # H2D of q,k,v,beta,dO; fwd+bwd; D2H of o,dq,dk,dv,dbeta.
    e2e = None
    if not args.no_e2e:
        hin = [t.cpu().pin_memory() for t in (q, k, v, beta, dO)]
        hout = [torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
                for t in (o, *grads)]
        h2d = sum(t.numel() * t.element_size() for t in hin)
        d2h = sum(t.numel() * t.element_size() for t in hout)

        host_buf = [None]

        def e2e_step():
            # the library's host-buffer entry point: slabs of batch rows
            # pipelined H2D / fwd+bwd / D2H on three streams (deltanet_fwd_bwd_host)
            host_buf[0], _ = dn.deltanet_fwd_bwd_host(*hin, out=tuple(hout), slabs=E2E_SLABS,
                                                      chunk=C, dev_buffer=host_buf[0],
                                                      device=dev)

        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize(dev)
        if ws > 1:
            dist.barrier()
        n_e2e = max(3, min(args.steps, 20))
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        for _ in range(n_e2e):
            e2e_step()
        a1.record(stream)
        torch.cuda.synchronize(dev)
        t_e2e = a0.elapsed_time(a1) * 1e-3 / n_e2e
        if ws > 1:
            tt = torch.tensor([t_e2e], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t_e2e = tt.item()
        e2e = {"value": tokens_per_step / t_e2e, "unit": "tokens/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": t_e2e * 1e3, "steps": n_e2e,
               "api": f"deltanet_fwd_bwd_host (pinned host tensors, {E2E_SLABS} slabs, "
                      "H2D / compute / D2H overlapped on three streams)"}

    clk = clocks.stop()

    # ---- NCCL gather of outputs and gradients into the full [B,H,L,d]
    # layout (data_parallel.gather_rows; outside the timed step)
    gather = None
    if ws > 1:
        dist.barrier()
        torch.cuda.synchronize(dev)
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        full = step.gather()
        g1.record(stream)
        torch.cuda.synchronize(dev)
        tg, = dp.max_over_ranks([g0.elapsed_time(g1) * 1e-3], dev)
        recv = sum(t.numel() * t.element_size() for t in full)
        gather = {"ms": tg * 1e3, "bytes_received_per_gpu": recv,
                  "GBps": recv / tg / 1e9, "collective": "ncclAllGather (all_gather_into_tensor)",
                  "layout": [list(t.shape) for t in full]}
        del full

    strong = None
    if not args.no_strong and not args.force_simt:
        strong = measure_strong_scaling(dp, dev, ws, rank)

    base = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        base = cpu_baseline()
    rec = pro = lng = gat = cpx = cfg1 = hds = None
    if rank == 0 and not args.no_recurrent and not args.force_simt:
        cfg1 = measure_1p3b(dn, dp, dev)
        hds = measure_head_dims(dn, dev, peaks)
        rec = measure_recurrent(dn, dev, q, k, v, beta, t_fwd, peaks)
        pro = measure_prologue(dn, dev, B_PER_RANK, H, L, D, peaks)
        lng = measure_long_context(dn, dev)
        gat = measure_gated(dn, dev, q, k, v, beta, t_fwd, t_bwd)
        cpx = measure_context_parallel(dn, dev)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "bf16", "data": "synthetic",
            "config": {"workload": f"deltanet_layer_fwd_bwd B={B_PER_RANK}/GPU H={H} L={L} "
                                   f"d={D} chunk={C}",
                       "global_batch": B_PER_RANK * ws, "seq_len": L, "heads": H,
                       "head_dim": D, "chunk": C, "parallelism": f"dp{ws} (batch x head shards)",
                       "l2": "inputs exceed L2 (q,k,v,dO 134 MB each); no flush",
                       "kernel_path": "tcgen05" if path == 1 else "simt"},
            "ms_fwd": t_fwd * 1e3, "ms_bwd": t_bwd * 1e3,
            "tc_peak_frac": tc_frac,
            "roofline": roof,
            "cpu_baseline": base,
            "e2e": e2e,
            "gpu_launches": n_launch * args.steps,
            "clocks": clk,
        }
        if gather:
            line["gather"] = gather
        if strong:
            line["strong_scaling"] = strong
        if cfg1:
            line["config_1p3b"] = cfg1
        if hds:
            line["head_dims"] = hds
        if rec:
            line["recurrent"] = rec
        if pro:
            line["prologue"] = pro
        if lng:
            line["long_context"] = lng
        if gat:
            line["gated"] = gat
        if cpx:
            line["context_parallel"] = cpx
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
