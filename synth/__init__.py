"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic: it only draws random
numbers with the shapes and value distributions of the paper's workload
(DESIGN.md §Input recipe) and rounds them once to the I/O dtype, so the
oracle (fp64, exact upcast) and the GPU see bit-identical inputs.

Recipe (§3.3, §2.2 line 96):
  q_raw, k_raw ~ SiLU(N(0,1))   (pre-normalisation keys/queries)
  v            ~ N(0,1)
  beta         ~ sigmoid(N(0,1)) in (0,1)
  dO           ~ N(0,1)         (upstream gradient of the layer output)
Each (b, h) unit has its own counter-style seed
  seed(cfg, b, h) = 2406064840 + 1_000_003 * cfg + b * H + h
so any rank (or the oracle) can regenerate any unit alone.
Alternative key distributions for parity edge cases: "gaussian" (raw
N(0,1) keys), "identical" (all keys of a unit equal, beta=1).

Gated DeltaNet (f4, R23) log-gates, fp32, from a separate stream:
  g = -scale * softplus(N(0,1))      (alpha = e^g in (0, 1))
scale = 0.05 is a slow decay (mean alpha ~ 0.96), 1.0 a fast one.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

SEED_BASE = 2406064840


@dataclass(frozen=True)
class Config:
    """One workload row of BASELINE.json `configs`."""
    name: str
    B: int
    H: int
    L: int
    Dk: int
    Dv: int
    chunk: int
    dtype: str  # "bf16" | "fp32"
    index: int  # seed stream: BASELINE.json configs position (5 = north_star target)


CONFIGS = {
    "tiny": Config("tiny", 1, 1, 64, 16, 16, 16, "fp32", 0),
    "1.3b": Config("1.3b", 8, 16, 2048, 128, 128, 64, "bf16", 1),
    "target": Config("target", 8, 16, 4096, 128, 128, 64, "bf16", 5),
    "long": Config("long", 2, 16, 16384, 128, 128, 64, "bf16", 2),
    "hd256": Config("hd256", 4, 8, 4096, 256, 256, 64, "bf16", 3),
    "sharded": Config("sharded", 64, 16, 4096, 128, 128, 64, "bf16", 4),
}


def unit_seed(cfg_index: int, b: int, h: int, H: int) -> int:
    return SEED_BASE + 1_000_003 * cfg_index + b * H + h


def round_to_bf16(x: np.ndarray) -> np.ndarray:
    """Round fp32 values to the nearest bf16 (ties to even), returned as fp32
    holding exactly representable bf16 values.  Bit manipulation only."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    u = (u + 0x7FFF + lsb) & 0xFFFF0000
    out = u.astype(np.uint32).view(np.float32)
    nan = np.isnan(x)
    if nan.any():
        out = out.copy()
        out[nan] = np.nan
    return out


def _silu(x):
    return x / (1.0 + np.exp(-x))


def _sigmoid(x):
    return 1.0 / (1.0 + np.exp(-x))


def unit_inputs(cfg_index, b, h, H, L, Dk, Dv, dtype="bf16", keys="silu"):
    """Inputs of one (b, h) unit as fp32 arrays (bf16-exact when dtype=bf16):
    q [L,Dk], k [L,Dk], v [L,Dv], beta [L], dO [L,Dv]."""
    rng = np.random.Generator(np.random.Philox(unit_seed(cfg_index, b, h, H)))
    qr = rng.standard_normal((L, Dk), dtype=np.float32)
    kr = rng.standard_normal((L, Dk), dtype=np.float32)
    v = rng.standard_normal((L, Dv), dtype=np.float32)
    br = rng.standard_normal((L,), dtype=np.float32)
    dO = rng.standard_normal((L, Dv), dtype=np.float32)
    if keys == "silu":
        q, k = _silu(qr), _silu(kr)
    elif keys == "gaussian":
        q, k = qr, kr
    elif keys == "identical":
        q, k = _silu(qr), np.repeat(_silu(kr[:1]), L, axis=0)
    else:
        raise ValueError(keys)
    beta = _sigmoid(br).astype(np.float32)
    if keys == "identical":
        beta = np.ones_like(beta)
    out = [np.asarray(a, dtype=np.float32) for a in (q, k, v, beta, dO)]
    if dtype == "bf16":
        out = [round_to_bf16(a) for a in out]
    return tuple(out)


def make_inputs(cfg: Config, b_range=None, keys="silu", units=None):
    """Stacked inputs [B', H, L, d] for batch rows b_range (default all), or
    for an explicit list of (b, h) `units` (returned stacked as [n, 1, L, d])."""
    fields = ("q", "k", "v", "beta", "dO")
    if units is not None:
        parts = [unit_inputs(cfg.index, b, h, cfg.H, cfg.L, cfg.Dk, cfg.Dv,
                             cfg.dtype, keys) for (b, h) in units]
        return {f: np.stack([p[i] for p in parts])[:, None]
                for i, f in enumerate(fields)}
    if b_range is None:
        b_range = range(cfg.B)
    b_range = list(b_range)
    shapes = {"q": (cfg.L, cfg.Dk), "k": (cfg.L, cfg.Dk), "v": (cfg.L, cfg.Dv),
              "beta": (cfg.L,), "dO": (cfg.L, cfg.Dv)}
    out = {f: np.empty((len(b_range), cfg.H) + shapes[f], np.float32) for f in fields}
    for bi, b in enumerate(b_range):
        for h in range(cfg.H):
            p = unit_inputs(cfg.index, b, h, cfg.H, cfg.L, cfg.Dk, cfg.Dv,
                            cfg.dtype, keys)
            for i, f in enumerate(fields):
                out[f][bi, h] = p[i]
    return out


def custom_config(B, H, L, Dk, Dv, chunk, dtype, index=100, name="custom"):
    return Config(name, B, H, L, Dk, Dv, chunk, dtype, index)


def make_gates(cfg: Config, scale: float = 0.05, b_range=None):
    """Log-gates g [B', H, L] fp32 (seed stream: the unit seed + 7919)."""
    if b_range is None:
        b_range = range(cfg.B)
    b_range = list(b_range)
    out = np.empty((len(b_range), cfg.H, cfg.L), np.float32)
    for bi, b in enumerate(b_range):
        for h in range(cfg.H):
            rng = np.random.Generator(np.random.Philox(unit_seed(cfg.index, b, h, cfg.H) + 7919))
            z = rng.standard_normal(cfg.L, dtype=np.float32).astype(np.float64)
            out[bi, h] = (-scale * np.logaddexp(0.0, z)).astype(np.float32)
    return out
