"""GPU parity of context parallelism (include/deltanet.h
deltanet_fwd_transition / deltanet_bwd_transition / deltanet_state_scan;
DESIGN.md §4.8) against the fp64 oracle (oracle/context.py, pinned in
tests/test_oracle_context.py), normwise (R16): 2e-2 for the bf16
path's transitions and outputs, 1e-5 for the fp32 scan.

The multi-part runs simulate P ranks on one GPU: the sequence is cut into
consecutive parts (interior parts with ragged tails, an empty part), each
part's transition is computed, the transitions are stacked as an all-gather
would stack them, and every part runs its forward / backward from the
scanned boundary state.  ``test_cp_over_nccl_world1`` drives the real
torch.distributed orchestration (NCCL, one rank)."""
import os
import socket

import numpy as np
import pytest
import torch

import oracle
import synth
from oracle import context as cpo
from parity import TOL, compare, run_oracle, to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2406_06484_b200 import build
    build.build()


def _inputs(B, H, L, index):
    return synth.make_inputs(synth.custom_config(B, H, L, 128, 128, 64, "bf16", index=index))


def _dev(inp):
    return {f: to_dev(inp[f], torch.bfloat16) for f in ("q", "k", "v", "beta", "dO")}


def _np(t):
    return t.float().cpu().numpy().astype(np.float64)


@pytest.mark.parametrize("L", [64, 300, 64 * 20])
def test_fwd_transition(L):
    import paper_2406_06484_b200 as dn
    inp = _inputs(2, 2, L, 700 + L)
    x = _dev(inp)
    psi, hloc = dn.deltanet_fwd_transition(x["q"], x["k"], x["v"], x["beta"])
    torch.cuda.synchronize()
    rpsi, rhloc = cpo.transition(inp["q"], inp["k"], inp["v"], inp["beta"])
    compare({"psi": _np(psi), "hloc": _np(hloc)}, {"psi": rpsi, "hloc": rhloc}, TOL["bf16"])


@pytest.mark.parametrize("saved", [True, False])
@pytest.mark.parametrize("L", [64, 300])
def test_bwd_transition(L, saved):
    import paper_2406_06484_b200 as dn
    inp = _inputs(2, 2, L, 720 + L)
    x = _dev(inp)
    ws = None
    if saved:  # records from a forward with an arbitrary h0 (X does not depend on it)
        h0 = to_dev(0.5 * np.random.default_rng(1).standard_normal((2, 2, 128, 128)),
                    torch.float32)
        _, _, ws = dn.deltanet_fwd(x["q"], x["k"], x["v"], x["beta"], h0=h0)
    dloc = dn.deltanet_bwd_transition(x["q"], x["k"], x["v"], x["beta"], x["dO"], workspace=ws)
    torch.cuda.synchronize()
    ref = cpo.bwd_transition(inp["q"], inp["k"], inp["v"], inp["beta"], inp["dO"])
    compare({"dhloc": _np(dloc)}, {"dhloc": ref}, TOL["bf16"])


def test_empty_sequence_transition():
    import paper_2406_06484_b200 as dn
    z = torch.empty((2, 3, 0, 128), dtype=torch.bfloat16, device="cuda")
    b = torch.empty((2, 3, 0), dtype=torch.bfloat16, device="cuda")
    psi, hloc = dn.deltanet_fwd_transition(z, z, z, b)
    dloc = dn.deltanet_bwd_transition(z, z, z, b, z)
    torch.cuda.synchronize()
    eye = torch.eye(128, device="cuda").expand(2, 3, 128, 128)
    assert torch.equal(psi, eye)
    assert torch.count_nonzero(hloc) == 0 and torch.count_nonzero(dloc) == 0


@pytest.mark.parametrize("reverse", [False, True])
def test_state_scan_fp32(reverse):
    import paper_2406_06484_b200 as dn
    rng = np.random.default_rng(3 + reverse)
    P, B, H = 5, 2, 3
    psi = 0.1 * rng.standard_normal((P, B, H, 128, 128)) + np.eye(128)
    loc = rng.standard_normal((P, B, H, 128, 128))
    edge = rng.standard_normal((B, H, 128, 128))
    f = lambda a: to_dev(a, torch.float32)
    for part in range(P):
        for e in (None, edge):
            got = dn.deltanet_state_scan(f(psi), f(loc), part, reverse=reverse,
                                         edge=None if e is None else f(e))
            torch.cuda.synchronize()
            ref = cpo.state_scan(psi, loc, part, reverse=reverse, edge=e)
            compare({"out": _np(got)}, {"out": ref}, 1e-5)
    # in place: out aliases edge
    ed = f(edge)
    dn.deltanet_state_scan(f(psi), f(loc), 3, reverse=reverse, edge=ed, out=ed)
    torch.cuda.synchronize()
    compare({"out": _np(ed)}, {"out": cpo.state_scan(psi, loc, 3, reverse, edge)}, 1e-5)


def _cp_run(x, cuts, h0=None, dhT=None):
    """The orchestration of context_parallel.cp_fwd / cp_bwd for P simulated
    ranks on one device (the all-gather is a torch.stack)."""
    import paper_2406_06484_b200 as dn
    parts = [{f: t[:, :, a:b].contiguous() for f, t in x.items()}
             for a, b in zip(cuts[:-1], cuts[1:])]
    P = len(parts)
    tr = [dn.deltanet_fwd_transition(p["q"], p["k"], p["v"], p["beta"]) for p in parts]
    psi_all = torch.stack([t[0] for t in tr])
    loc_all = torch.stack([t[1] for t in tr])
    outs, hs, wss = [], [], []
    for r, p in enumerate(parts):
        h_start = dn.deltanet_state_scan(psi_all, loc_all, r, edge=h0)
        o, hT, ws = dn.deltanet_fwd(p["q"], p["k"], p["v"], p["beta"], h0=h_start)
        outs.append(o)
        hs.append(h_start)
        wss.append(ws)
    dloc_all = torch.stack([dn.deltanet_bwd_transition(p["q"], p["k"], p["v"], p["beta"],
                                                       p["dO"], workspace=ws)
                            for p, ws in zip(parts, wss)])
    grads = []
    for r, p in enumerate(parts):
        dh_end = dn.deltanet_state_scan(psi_all, dloc_all, r, reverse=True, edge=dhT)
        grads.append(dn.deltanet_bwd(p["q"], p["k"], p["v"], p["beta"], p["dO"], h0=hs[r],
                                     dhT=dh_end, workspace=wss[r]))
    torch.cuda.synchronize()
    cat = lambda ts: _np(torch.cat(ts, dim=2))
    return {"o": cat(outs), "hT": _np(hT), "dq": cat([g[0] for g in grads]),
            "dk": cat([g[1] for g in grads]), "dv": cat([g[2] for g in grads]),
            "dbeta": cat([g[3] for g in grads]), "dh0": _np(grads[0][4])}


@pytest.mark.parametrize("cuts", [
    [0, 256, 512],                 # two equal parts
    [0, 100, 100, 457, 777, 1024],  # ragged interior parts and an empty part
])
def test_multi_part_matches_oracle(cuts):
    L = cuts[-1]
    inp = _inputs(2, 2, L, 740 + len(cuts))
    rng = np.random.default_rng(9)
    h0 = 0.3 * rng.standard_normal((2, 2, 128, 128))
    dhT = 0.3 * rng.standard_normal((2, 2, 128, 128))
    got = _cp_run(_dev(inp), cuts, h0=to_dev(h0, torch.float32), dhT=to_dev(dhT, torch.float32))
    compare(got, run_oracle(inp, h0=h0, dhT=dhT), TOL["bf16"])


def test_multi_part_matches_single_call():
    """Eight parts of 512 tokens against one uncut deltanet_fwd / deltanet_bwd
    call on the same device (both bf16 paths, so to the bf16 bar)."""
    import paper_2406_06484_b200 as dn
    L = 4096
    inp = _inputs(1, 4, L, 760)
    x = _dev(inp)
    got = _cp_run(x, list(range(0, L + 1, 512)))
    o, hT, ws = dn.deltanet_fwd(x["q"], x["k"], x["v"], x["beta"])
    g = dn.deltanet_bwd(x["q"], x["k"], x["v"], x["beta"], x["dO"], workspace=ws)
    torch.cuda.synchronize()
    ref = {"o": _np(o), "hT": _np(hT), "dq": _np(g[0]), "dk": _np(g[1]), "dv": _np(g[2]),
           "dbeta": _np(g[3]), "dh0": _np(g[4])}
    compare(got, ref, TOL["bf16"])
    # and the multi-part run against the oracle on two sampled units
    for h in (0, 3):
        one = {f: inp[f][:, h:h + 1] for f in inp}
        sub = {key: val[:, h:h + 1] for key, val in got.items()}
        compare(sub, run_oracle(one), TOL["bf16"])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_cp_over_nccl_world1():
    """context_parallel.cp_fwd / cp_bwd through a real NCCL process group of
    one rank: the gather is the NCCL all_gather_into_tensor path; with one part
    the result equals the plain call."""
    import torch.distributed as dist

    import paper_2406_06484_b200 as dn
    from paper_2406_06484_b200.context_parallel import cp_bwd, cp_fwd
    inp = _inputs(2, 2, 300, 780)
    x = _dev(inp)
    own = not dist.is_initialized()
    if own:
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}",
                                rank=0, world_size=1)
    try:
        o, hT, st = cp_fwd(x["q"], x["k"], x["v"], x["beta"])
        g = cp_bwd(x["q"], x["k"], x["v"], x["beta"], x["dO"], st)
        torch.cuda.synchronize()
    finally:
        if own:
            dist.destroy_process_group()
    got = {"o": _np(o), "hT": _np(hT), "dq": _np(g[0]), "dk": _np(g[1]), "dv": _np(g[2]),
           "dbeta": _np(g[3]), "dh0": _np(g[4])}
    compare(got, run_oracle(inp), TOL["bf16"])


def test_segmented_transitions_long_parts():
    """Parts long enough (and units few enough) that the transitions run the
    segment-parallel pass 1 plus the composition kernel (launch count 2):
    transitions against the oracle, and a 2-part run against the uncut oracle."""
    import paper_2406_06484_b200 as dn
    L = 8192
    inp = _inputs(1, 2, L, 790)
    x = _dev(inp)
    half = {f: t[:, :, L // 2:].contiguous() for f, t in x.items()}
    d = dn.make_desc(1, 2, L // 2, 128, 128)
    assert dn.deltanet_launch_count(d, 5) == 2 and dn.deltanet_launch_count(d, 6) == 2
    psi, hloc = dn.deltanet_fwd_transition(half["q"], half["k"], half["v"], half["beta"])
    _, _, ws = dn.deltanet_fwd(half["q"], half["k"], half["v"], half["beta"])
    dloc = dn.deltanet_bwd_transition(half["q"], half["k"], half["v"], half["beta"], half["dO"],
                                      workspace=ws)
    torch.cuda.synchronize()
    sl = {f: a[:, :, L // 2:] for f, a in inp.items()}
    rpsi, rhloc = cpo.transition(sl["q"], sl["k"], sl["v"], sl["beta"])
    rdloc = cpo.bwd_transition(sl["q"], sl["k"], sl["v"], sl["beta"], sl["dO"])
    compare({"psi": _np(psi), "hloc": _np(hloc), "dhloc": _np(dloc)},
            {"psi": rpsi, "hloc": rhloc, "dhloc": rdloc}, TOL["bf16"])
    got = _cp_run(x, [0, L // 2, L])
    compare(got, run_oracle(inp), TOL["bf16"])
