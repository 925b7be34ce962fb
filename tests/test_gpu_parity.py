"""GPU parity: the CUDA path (through the C ABI) vs the fp64 oracle on the
same seeded inputs, element by element, normwise tolerance (tests/parity.py).
"""
import numpy as np
import pytest
import torch

import synth
from parity import TOL, compare, normwise, row_guard as _row_guard, run_gpu, run_oracle, to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2406_06484_b200 import build
    build.build()


def _case(B, H, L, Dk, Dv, C, dtype, keys="silu", index=200):
    cfg = synth.custom_config(B, H, L, Dk, Dv, C, dtype, index=index)
    return cfg, synth.make_inputs(cfg, keys=keys)


# ---------------------------------------------------------------- fp32 (SIMT)

def test_tiny_config_fp32():
    """BASELINE.json configs[0]: B=1 H=1 L=64 d=16 chunk=16, fp32, 1e-4."""
    cfg = synth.CONFIGS["tiny"]
    inp = synth.make_inputs(cfg)
    got = run_gpu(inp, "fp32", cfg.chunk)
    errs = compare(got, run_oracle(inp), TOL["fp32"])
    assert max(errs.values()) < 1e-5


@pytest.mark.parametrize("C", [16, 32, 64, 128])
@pytest.mark.parametrize("d", [16, 64, 128])
def test_fp32_shapes_ragged(C, d):
    """Several chunks and a ragged tail (L = 2C + 37), B=2, H=2, h0/dhT set."""
    L = 2 * C + 37
    cfg, inp = _case(2, 2, L, d, d, C, "fp32", index=300 + C + d)
    rng = np.random.default_rng(C * d)
    h0 = (0.1 * rng.standard_normal((2, 2, d, d))).astype(np.float32)
    dhT = rng.standard_normal((2, 2, d, d)).astype(np.float32)
    got = run_gpu(inp, "fp32", C, h0=h0, dhT=dhT)
    compare(got, run_oracle(inp, h0=h0.astype(np.float64), dhT=dhT.astype(np.float64)),
            TOL["fp32"])


def test_fp32_rectangular_heads_no_l2():
    cfg, inp = _case(1, 3, 90, 32, 64, 32, "fp32", keys="gaussian", index=401)
    # un-normalised gaussian keys would blow up the recurrence; scale them down
    for f in ("q", "k"):
        inp[f] = (inp[f] / np.sqrt(32)).astype(np.float32)
    got = run_gpu(inp, "fp32", 32, l2norm=False)
    compare(got, run_oracle(inp, l2norm=False), TOL["fp32"])


@pytest.mark.parametrize("save_states", [True, False])
def test_fp32_states_recompute(save_states):
    cfg, inp = _case(1, 2, 200, 64, 64, 64, "fp32", index=402)
    got = run_gpu(inp, "fp32", 64, save_states=save_states)
    compare(got, run_oracle(inp), TOL["fp32"])


def test_fp32_identical_keys_beta_one():
    """Adversarial UT case: all keys of a unit equal, beta = 1."""
    cfg, inp = _case(1, 2, 150, 32, 32, 64, "fp32", keys="identical", index=403)
    got = run_gpu(inp, "fp32", 64)
    compare(got, run_oracle(inp), TOL["fp32"])


def test_zero_rows_l2_eps():
    """Zero q/k rows under L2 normalisation stay finite (R9)."""
    cfg, inp = _case(1, 1, 64, 16, 16, 16, "fp32", index=404)
    inp["q"][0, 0, 5] = 0
    inp["k"][0, 0, 9] = 0
    got = run_gpu(inp, "fp32", 16)
    compare(got, run_oracle(inp), TOL["fp32"])


def test_empty_length():
    """L = 0: no tokens; hT = h0 and dh0 = dhT."""
    import paper_2406_06484_b200 as dn
    q = torch.zeros(2, 2, 0, 16, device="cuda")
    b = torch.zeros(2, 2, 0, device="cuda")
    h0 = torch.randn(2, 2, 16, 16, device="cuda")
    o, hT, ws = dn.deltanet_fwd(q, q, q, b, chunk=16, h0=h0)
    dhT = torch.randn_like(h0)
    g = dn.deltanet_bwd(q, q, q, b, q, chunk=16, h0=h0, dhT=dhT, workspace=ws)
    torch.cuda.synchronize()
    assert torch.equal(hT, h0) and torch.equal(g[4], dhT)


# ---------------------------------------------------------------- bf16

@pytest.mark.parametrize("force_simt", [False, True])
def test_bf16_multi_chunk_ragged(force_simt):
    """bf16, d=128, C=64: 5 chunks + ragged tail, several units."""
    cfg, inp = _case(2, 3, 4 * 64 + 45, 128, 128, 64, "bf16", index=500)
    got = run_gpu(inp, "bf16", 64, force_simt=force_simt)
    compare(got, run_oracle(inp), TOL["bf16"])


def test_bf16_with_initial_state():
    cfg, inp = _case(1, 2, 256, 128, 128, 64, "bf16", index=501)
    rng = np.random.default_rng(7)
    h0 = (0.2 * rng.standard_normal((1, 2, 128, 128))).astype(np.float32)
    dhT = rng.standard_normal((1, 2, 128, 128)).astype(np.float32)
    got = run_gpu(inp, "bf16", 64, h0=h0, dhT=dhT)
    compare(got, run_oracle(inp, h0=h0.astype(np.float64), dhT=dhT.astype(np.float64)),
            TOL["bf16"])


@pytest.mark.parametrize("keys", ["gaussian", "identical"])
@pytest.mark.parametrize("compensated", [False, True])
def test_bf16_key_distributions(keys, compensated):
    """Gaussian keys: the north_star bar.  "identical" (every key of a unit
    equal, beta = 1) is an adversarial case outside the paper's workload:
    T^{-1} is bidiagonal, U = T^{-1} V holds differences v_i - v_{i-1}, and the
    state update, the intra-chunk output and dQ = dA K_hat sum C bf16-rounded
    operands whose sum telescopes: ~sqrt(C) 2^-9 of the result (hT 0.021,
    dq 0.023 measured).  DELTANET_COMPENSATED carries the rounding error
    along the tokens (R19) and brings it under the north_star bar
    2e-2 (hT 0.008, dq 0.018); without it this case keeps the bar 3e-2."""
    import paper_2406_06484_b200 as dn
    cfg, inp = _case(1, 2, 192, 128, 128, 64, "bf16", keys=keys, index=502)
    got = run_gpu(inp, "bf16", 64, extra_flags=dn.DELTANET_COMPENSATED if compensated else 0)
    bar = TOL["bf16"] if (keys != "identical" or compensated) else 3e-2
    compare(got, run_oracle(inp), bar)


def test_bf16_deterministic():
    cfg, inp = _case(2, 2, 320, 128, 128, 64, "bf16", index=503)
    a = run_gpu(inp, "bf16", 64)
    b = run_gpu(inp, "bf16", 64)
    for k in a:
        if a[k] is not None:
            assert np.array_equal(a[k], b[k]), k


def _per_unit(got, ref, tol, B, H):
    """normwise per (b, h) unit (each unit's own max as the scale), plus the
    per-unit check of dbeta row by row of 64 tokens (see _row_guard)."""
    for b in range(B):
        for h in range(H):
            sub = {k: (None if v is None else v[b:b + 1, h:h + 1]) for k, v in got.items()}
            one = {k: (None if v is None else v[b:b + 1, h:h + 1]) for k, v in ref.items()}
            compare(sub, one, tol)


def test_bf16_target_full_size_all_units():
    """The bench workload (north_star target, B=8 H=16 L=4096) in the bench
    launch configuration: every one of the 128 units against the oracle,
    normwise per unit, and dbeta per 64-token window."""
    cfg = synth.CONFIGS["target"]
    inp = synth.make_inputs(cfg)
    got = run_gpu(inp, "bf16", cfg.chunk)
    ref = run_oracle(inp)
    _per_unit(got, ref, TOL["bf16"], cfg.B, cfg.H)
    _row_guard(got, ref, "dbeta", TOL["bf16"])


def test_bf16_1p3b_full_size_sampled_units():
    """BASELINE configs[1] (B=8 H=16 L=2048) at full size; units of the
    first, middle and last batch rows against the oracle."""
    cfg = synth.CONFIGS["1.3b"]
    inp = synth.make_inputs(cfg)
    got = run_gpu(inp, "bf16", cfg.chunk)
    units = [(0, 0), (0, 9), (cfg.B // 2, 5), (cfg.B - 1, cfg.H - 1)]
    for (b, h) in units:
        one = {f: inp[f][b:b + 1, h:h + 1] for f in inp}
        ref = run_oracle(one)
        sub = {k: (None if v is None else v[b:b + 1, h:h + 1]) for k, v in got.items()}
        compare(sub, ref, TOL["bf16"])
        _row_guard(sub, ref, "dbeta", TOL["bf16"])


def test_bf16_tc_zero_and_tiny_rows():
    """tcgen05 path, d = 128: q / k rows that are exactly zero or of norm
    ~1e-8 (below eps = 1e-6, reading R9: divided by eps, not by the norm)
    next to ordinary rows; every output against the oracle."""
    import paper_2406_06484_b200 as dn
    cfg, inp = _case(1, 2, 3 * 64 + 11, 128, 128, 64, "bf16", index=560)
    assert dn.deltanet_path(dn.make_desc(1, 2, cfg.L, 128, 128, 64, torch.bfloat16)) == 1
    for f, rows in (("q", (0, 70, 140)), ("k", (5, 64, 190))):
        for t in rows:
            inp[f][0, 0, t] = 0.0
            x = inp[f][0, 1, t].astype(np.float64)
            inp[f][0, 1, t] = synth.round_to_bf16((1e-8 * x / np.linalg.norm(x)).astype(np.float32))
    got = run_gpu(inp, "bf16", 64)
    ref = run_oracle(inp)
    compare(got, ref, TOL["bf16"])
    _row_guard(got, ref, "dbeta", TOL["bf16"])


# ------------------------------------------------- segment-parallel forward

def _segmented(B, H, L):
    import paper_2406_06484_b200 as dn
    d = dn.make_desc(B, H, L, 128, 128, 64, torch.bfloat16)
    return dn.deltanet_launch_count(d, 0) == 3


@pytest.mark.parametrize("save_states", [True, False])
def test_bf16_segmented_forward(save_states):
    """Few units, many chunks: the forward splits each unit's sequence into
    segments (pass 1: local end state + transition, pass 2: scan of the
    segment-start states, pass 3: the forward from those states; DESIGN.md
    §4.6).  h0 / dhT exercise the scan's start and the backward that reads
    pass 3's states (or recomputes them through the same segmented forward)."""
    L = 64 * 40 + 17
    assert _segmented(1, 2, L)
    cfg, inp = _case(1, 2, L, 128, 128, 64, "bf16", index=520)
    rng = np.random.default_rng(11)
    h0 = (0.2 * rng.standard_normal((1, 2, 128, 128))).astype(np.float32)
    dhT = rng.standard_normal((1, 2, 128, 128)).astype(np.float32)
    got = run_gpu(inp, "bf16", 64, h0=h0, dhT=dhT, save_states=save_states)
    compare(got, run_oracle(inp, h0=h0.astype(np.float64), dhT=dhT.astype(np.float64)),
            TOL["bf16"])


def test_bf16_segments_match_serial():
    """The segmented and the one-CTA-per-unit forward agree to the bf16 bar
    (both are bf16-rounded evaluations of the same exact recurrence)."""
    cfg, inp = _case(1, 3, 64 * 33, 128, 128, 64, "bf16", index=521)
    a = run_gpu(inp, "bf16", 64)
    b = run_gpu(inp, "bf16", 64, segments=False)
    compare({k: a[k] for k in ("o", "hT")}, {k: b[k] for k in ("o", "hT")}, TOL["bf16"])


def test_bf16_segment_prep_records_bitwise():
    """Segmented forward, pass 3 from pass 1's prep records (T', T'' images,
    s, 1/s) vs pass 3 redoing its prep (without saved
    states there are no prep records): identical operands, so o and hT are
    bitwise equal; a ragged tail and a nonzero h0 included."""
    import paper_2406_06484_b200 as dn
    cfg, inp = _case(1, 3, 64 * 40 + 23, 128, 128, 64, "bf16", index=527)
    dev = lambda x, dt=torch.bfloat16: to_dev(x, dt)
    q, k, v, b = (dev(inp[f]) for f in ("q", "k", "v", "beta"))
    h0n = (0.1 * np.random.default_rng(7).standard_normal((1, 3, 128, 128))).astype(np.float32)
    h0 = dev(h0n, torch.float32)
    d = dn.make_desc(1, 3, cfg.L, 128, 128, 64, torch.bfloat16)
    assert dn.deltanet_launch_count(d, 0) == 3, "expected the segmented forward"
    o1, h1, _ = dn.deltanet_fwd(q, k, v, b, h0=h0, save_states=True)
    o2, h2, _ = dn.deltanet_fwd(q, k, v, b, h0=h0, save_states=False)
    torch.cuda.synchronize()
    assert torch.equal(o1, o2) and torch.equal(h1, h2)
    ref = run_oracle(inp, h0=h0n.astype(np.float64))
    compare({"o": o1.float().cpu().numpy(), "hT": h1.cpu().numpy()},
            {"o": ref["o"], "hT": ref["hT"]}, TOL["bf16"])


def test_bf16_long_context_sampled_units():
    """BASELINE configs[2] (B=2 H=16 L=16384): 32 units, so the forward runs
    segmented; three sampled units against the oracle (fwd + bwd)."""
    cfg = synth.CONFIGS["long"]
    assert _segmented(cfg.B, cfg.H, cfg.L)
    inp = synth.make_inputs(cfg)
    got = run_gpu(inp, "bf16", cfg.chunk)
    for (b, h) in [(0, 0), (cfg.B - 1, cfg.H - 1), (1, 6)]:
        one = {f: inp[f][b:b + 1, h:h + 1] for f in inp}
        ref = run_oracle(one)
        sub = {k: (None if v is None else v[b:b + 1, h:h + 1]) for k, v in got.items()}
        compare(sub, ref, TOL["bf16"])


@pytest.mark.parametrize("name", ["hd256", "sharded"])
def test_bf16_remaining_configs_sampled_units(name):
    """BASELINE configs[3] (d=256, the split tcgen05 kernels; every unit is
    checked in test_gpu_split.py) and configs[4] (B=64: 1024 units, several
    waves) at full size on their default paths; two sampled units against
    the oracle."""
    import paper_2406_06484_b200 as dn
    cfg = synth.CONFIGS[name]
    units = [(0, 0), (cfg.B - 1, cfg.H - 1)]
    inp = synth.make_inputs(cfg)
    d = dn.make_desc(cfg.B, cfg.H, cfg.L, cfg.Dk, cfg.Dv, cfg.chunk, torch.bfloat16)
    assert dn.deltanet_path(d) == (2 if cfg.Dk == 256 else 1)
    got = run_gpu(inp, "bf16", cfg.chunk)
    for (b, h) in units:
        one = {f: inp[f][b:b + 1, h:h + 1] for f in inp}
        ref = run_oracle(one)
        sub = {k: (None if v is None else v[b:b + 1, h:h + 1]) for k, v in got.items()}
        compare(sub, ref, TOL["bf16"])


# ------------------------------------------------- tcgen05 edge cases

@pytest.mark.parametrize("L", [1, 37, 64, 128, 64 * 41 + 1])
def test_bf16_tc_lengths(L):
    """tcgen05 path: a single partial chunk, exact multiples of C, and (at
    64*41+1 with one unit) a segmented run whose last segment is short."""
    import paper_2406_06484_b200 as dn
    H = 1 if L > 1000 else 2
    assert dn.deltanet_path(dn.make_desc(1, H, L, 128, 128, 64, torch.bfloat16)) == 1
    cfg, inp = _case(1, H, L, 128, 128, 64, "bf16", index=530 + L % 97)
    got = run_gpu(inp, "bf16", 64)
    compare(got, run_oracle(inp), TOL["bf16"])


def test_bf16_tc_no_l2_unit_keys():
    """tcgen05 path without the in-kernel L2 normalisation (flag off) on keys
    and queries normalised by the caller: same result as the flag on."""
    cfg, inp = _case(2, 2, 300, 128, 128, 64, "bf16", index=540)
    for f in ("q", "k"):
        x = inp[f].astype(np.float64)
        x = x / np.maximum(np.linalg.norm(x, axis=-1, keepdims=True), 1e-6)
        inp[f] = synth.round_to_bf16(x.astype(np.float32))
    got = run_gpu(inp, "bf16", 64, l2norm=False)
    compare(got, run_oracle(inp, l2norm=False), TOL["bf16"])
