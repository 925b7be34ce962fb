import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import synth
from parity import run_gpu, run_oracle, compare, TOL
for D, L in ((64, 150), (256, 130), (128, 70)):
    cfg = synth.custom_config(1, 2, L, D, D, 64, "bf16", index=990 + D)
    inp = synth.make_inputs(cfg)
    got = run_gpu(inp, "bf16", 64, force_split=(D == 128))
    print(D, L, compare(got, run_oracle(inp), TOL["bf16"]))
