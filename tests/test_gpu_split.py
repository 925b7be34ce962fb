"""GPU parity of the split tcgen05 path (chunk-parallel
prep, per-d_v-block state chains, chunk-parallel local gradients) against
the fp64 oracle on the same seeded inputs, normwise bf16 bar (tests/parity.py).
d = 256 is BASELINE configs[3]; d = 64 is fig:kernel_speed's other head dim
(PAPER.md P:208-213); d = 128 runs here only with force_split, checked
against the oracle and against the fused kernels."""
import numpy as np
import pytest
import torch

import synth
from parity import TOL, compare, run_gpu, run_oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2406_06484_b200 import build
    build.build()


def _case(B, H, L, D, index, keys="silu"):
    cfg = synth.custom_config(B, H, L, D, D, 64, "bf16", index=index)
    return cfg, synth.make_inputs(cfg, keys=keys)


def _states(B, H, D, seed):
    rng = np.random.default_rng(seed)
    h0 = (0.1 * rng.standard_normal((B, H, D, D))).astype(np.float32)
    dhT = rng.standard_normal((B, H, D, D)).astype(np.float32)
    return h0, dhT


@pytest.mark.parametrize("D", [64, 128, 256])
def test_split_multi_chunk_ragged(D):
    """Three chunks and a ragged tail, two units, nonzero h0 and dhT."""
    import paper_2406_06484_b200 as dn
    L = 3 * 64 + 17
    cfg, inp = _case(1, 2, L, D, index=600 + D)
    h0, dhT = _states(1, 2, D, D)
    assert dn.deltanet_path(dn.make_desc(1, 2, L, D, D, force_split=True)) == 2
    got = run_gpu(inp, "bf16", 64, h0=h0, dhT=dhT, force_split=True)
    ref = run_oracle(inp, h0=h0.astype(np.float64), dhT=dhT.astype(np.float64))
    compare(got, ref, TOL["bf16"])


@pytest.mark.parametrize("L", [1, 37, 64, 128, 64 * 9 + 5])
def test_split_lengths(L):
    """A single partial chunk, exact multiples of C, a longer chain (d = 256)."""
    cfg, inp = _case(1, 2, L, 256, index=620 + L % 89)
    got = run_gpu(inp, "bf16", 64)
    compare(got, run_oracle(inp), TOL["bf16"])


@pytest.mark.parametrize("D", [64, 256])
def test_split_recompute_and_no_l2(D):
    """Backward without the forward's saved records (it re-runs the forward
    kernels), and both directions without the in-kernel L2 normalisation on
    caller-normalised q, k."""
    L = 2 * 64 + 30
    cfg, inp = _case(2, 2, L, D, index=640 + D)
    got = run_gpu(inp, "bf16", 64, save_states=False)
    compare(got, run_oracle(inp), TOL["bf16"])
    for f in ("q", "k"):
        x = inp[f].astype(np.float64)
        inp[f] = (x / np.linalg.norm(x, axis=-1, keepdims=True)).astype(inp[f].dtype)
    got = run_gpu(inp, "bf16", 64, l2norm=False)
    compare(got, run_oracle(inp, l2norm=False), TOL["bf16"])


def test_split_zero_rows_eps():
    """Zero q / k rows take the eps branch of the L2 normalisation and its
    adjoint (R9) on the split kernels."""
    cfg, inp = _case(1, 2, 150, 256, index=660)
    inp["q"][0, 0, 5] = 0
    inp["k"][0, 1, 70] = 0
    inp["k"][0, 0, 9] = 0
    got = run_gpu(inp, "bf16", 64)
    compare(got, run_oracle(inp), TOL["bf16"])


def test_split_d128_matches_fused():
    """d = 128 through the split kernels and through the fused kernels: both
    within the bar of the oracle, and within twice the bar of each other."""
    cfg, inp = _case(2, 2, 5 * 64 + 3, 128, index=670)
    ref = run_oracle(inp)
    a = run_gpu(inp, "bf16", 64, force_split=True)
    b = run_gpu(inp, "bf16", 64)
    compare(a, ref, TOL["bf16"])
    compare(b, ref, TOL["bf16"])
    compare(a, b, 2 * TOL["bf16"])


def test_split_deterministic():
    cfg, inp = _case(2, 2, 4 * 64 + 11, 256, index=680)
    a = run_gpu(inp, "bf16", 64)
    b = run_gpu(inp, "bf16", 64)
    for k in a:
        if a[k] is not None:
            assert np.array_equal(a[k], b[k]), k


def test_split_hd256_full_config_all_units():
    """BASELINE configs[3] at full size (B=4 H=8 L=4096 d=256), in the
    launch configuration bench.py times, every one of its 32 units against
    the oracle (normwise per unit)."""
    import paper_2406_06484_b200 as dn
    cfg = synth.CONFIGS["hd256"]
    inp = synth.make_inputs(cfg)
    d = dn.make_desc(cfg.B, cfg.H, cfg.L, cfg.Dk, cfg.Dv, cfg.chunk, torch.bfloat16)
    assert dn.deltanet_path(d) == 2
    got = run_gpu(inp, "bf16", cfg.chunk)
    ref = run_oracle(inp)
    for b in range(cfg.B):
        for h in range(cfg.H):
            sub = {k: (None if v is None else v[b:b + 1, h:h + 1]) for k, v in got.items()}
            one = {k: (None if v is None else v[b:b + 1, h:h + 1]) for k, v in ref.items()}
            compare(sub, one, TOL["bf16"])
