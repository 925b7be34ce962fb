"""Multi-process (gloo, world_size 2, CPU) test of the sharding / gather
logic bench.py uses on 8 B200: rank r owns batch rows [8r, 8r+8) of the
B=64 "sharded" config, the (b, h) units are independent (no collective in
the step), and an all-gather of the per-rank outputs reassembles exactly the
single-process result.  The fp64 oracle stands in for the kernel here (test
infrastructure); the GPU path is covered by tests/test_gpu_parity.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, B_per, cfg_kw, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = synth.custom_config(**cfg_kw)
    rows = range(rank * B_per, (rank + 1) * B_per)
    x = synth.make_inputs(cfg, b_range=rows)
    o, _ = oracle.recurrent_fwd(x["q"], x["k"], x["v"], x["beta"], nthreads=1)
    dq, dk, dv, db, _ = oracle.recurrent_bwd(x["q"], x["k"], x["v"], x["beta"], x["dO"],
                                            nthreads=1)
    outs = []
    for t in (o, dq, dk, dv, db):
        local = torch.from_numpy(np.ascontiguousarray(t))
        full = [torch.empty_like(local) for _ in range(world)]
        dist.all_gather(full, local)
        outs.append(torch.cat(full, 0).numpy())
    # timing protocol of bench.py: max over ranks
    t = torch.tensor([float(rank + 1)])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        out_q.put((outs, t.item()))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_gather_matches_single_process():
    world, B_per = 2, 2
    cfg_kw = dict(B=world * B_per, H=2, L=40, Dk=8, Dv=8, chunk=16, dtype="bf16", index=77)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, B_per, cfg_kw, q))
             for r in range(world)]
    for p in procs:
        p.start()
    outs, tmax = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert tmax == world  # max over ranks
    cfg = synth.custom_config(**cfg_kw)
    x = synth.make_inputs(cfg)
    o, _ = oracle.recurrent_fwd(x["q"], x["k"], x["v"], x["beta"], nthreads=1)
    ref = [o, *oracle.recurrent_bwd(x["q"], x["k"], x["v"], x["beta"], x["dO"], nthreads=1)[:4]]
    for a, b in zip(outs, ref):
        assert np.array_equal(a, b)


def test_rank_slab_seeds_are_unit_local():
    """Any rank regenerates its slab alone: rows [8r, 8r+8) of the B=64 config
    equal the corresponding rows of the full tensor."""
    cfg = synth.custom_config(4, 2, 24, 8, 8, 16, "bf16", index=78)
    full = synth.make_inputs(cfg)
    part = synth.make_inputs(cfg, b_range=range(2, 4))
    for f in full:
        assert np.array_equal(full[f][2:4], part[f])


# ---------------------------------------------------------------- context parallelism
def _oracle_ops():
    """The fp64 oracle behind the op signatures paper_2406_06484_b200.context_parallel
    drives (test infrastructure standing in for the CUDA kernels on CPU)."""
    from types import SimpleNamespace

    from oracle import context as cpo

    T = torch.from_numpy
    N = lambda t: None if t is None else t.numpy()

    def fwd_transition(q, k, v, beta, l2norm=True, workspace=None):
        psi, hloc = cpo.transition(q.numpy(), k.numpy(), v.numpy(), beta.numpy(), l2norm=l2norm)
        return T(psi), T(hloc)

    def state_scan(psi_all, loc_all, part, reverse=False, edge=None):
        return T(cpo.state_scan(psi_all.numpy(), loc_all.numpy(), part, reverse, N(edge)))

    def fwd(q, k, v, beta, h0=None, l2norm=True, save_states=True, workspace=None):
        o, hT = oracle.recurrent_fwd(q.numpy(), k.numpy(), v.numpy(), beta.numpy(), h0=N(h0),
                                     l2norm=l2norm, nthreads=1)
        return T(o), T(hT), torch.zeros(1)

    def bwd_transition(q, k, v, beta, dO, l2norm=True, workspace=None):
        return T(cpo.bwd_transition(q.numpy(), k.numpy(), v.numpy(), beta.numpy(), dO.numpy(),
                                    l2norm=l2norm))

    def bwd(q, k, v, beta, dO, h0=None, dhT=None, l2norm=True, workspace=None):
        g = oracle.recurrent_bwd(q.numpy(), k.numpy(), v.numpy(), beta.numpy(), dO.numpy(),
                                 h0=N(h0), dhT=N(dhT), l2norm=l2norm, nthreads=1)
        return tuple(T(x) for x in g)

    return SimpleNamespace(fwd_transition=fwd_transition, bwd_transition=bwd_transition,
                           state_scan=state_scan, fwd=fwd, bwd=bwd)


def _cp_worker(rank, world, port, cfg_kw, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2406_06484_b200.context_parallel import cp_bwd, cp_fwd
    cfg = synth.custom_config(**cfg_kw)
    x = synth.make_inputs(cfg)
    Lr = cfg.L // world
    sl = slice(rank * Lr, (rank + 1) * Lr)
    part = {f: torch.from_numpy(np.ascontiguousarray(x[f][:, :, sl], dtype=np.float64))
            for f in ("q", "k", "v", "beta", "dO")}
    rng = np.random.default_rng(11)
    h0 = torch.from_numpy(rng.standard_normal((cfg.B, cfg.H, cfg.Dk, cfg.Dv)))
    dhT = torch.from_numpy(rng.standard_normal((cfg.B, cfg.H, cfg.Dk, cfg.Dv)))
    ops = _oracle_ops()
    o, hT, st = cp_fwd(part["q"], part["k"], part["v"], part["beta"], h0=h0, ops=ops)
    dq, dk, dv, db, dhs = cp_bwd(part["q"], part["k"], part["v"], part["beta"], part["dO"], st,
                                 dhT=dhT, ops=ops)
    outs = []
    for t in (o, dq, dk, dv, db):
        full = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(full, t.contiguous())
        outs.append(torch.cat(full, 2).numpy())
    if rank == 0:
        out_q.put(("r0", outs, dhs.numpy(), h0.numpy(), dhT.numpy()))
    if rank == world - 1:
        out_q.put(("last", hT.numpy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_context_parallel_orchestration_matches_uncut_run(world):
    """cp_fwd / cp_bwd over `world` gloo ranks, each holding a consecutive part
    of the sequence, reproduce the uncut recurrence's o, grads, hT and dh0."""
    cfg_kw = dict(B=2, H=2, L=world * 12, Dk=8, Dv=8, chunk=16, dtype="fp32", index=79)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_cp_worker, args=(r, world, port, cfg_kw, q))
             for r in range(world)]
    for p in procs:
        p.start()
    got = dict((m[0], m[1:]) for m in (q.get(timeout=180), q.get(timeout=180)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    outs, dh0, h0, dhT = got["r0"]
    (hT,) = got["last"]
    cfg = synth.custom_config(**cfg_kw)
    x = {f: np.asarray(a, dtype=np.float64) for f, a in synth.make_inputs(cfg).items()}
    o, hT_ref = oracle.recurrent_fwd(x["q"], x["k"], x["v"], x["beta"], h0=h0, nthreads=1)
    g = oracle.recurrent_bwd(x["q"], x["k"], x["v"], x["beta"], x["dO"], h0=h0, dhT=dhT,
                             nthreads=1)
    for a, b in zip(outs, [o, *g[:4]]):
        np.testing.assert_allclose(a, b, rtol=1e-9, atol=1e-11)
    np.testing.assert_allclose(hT, hT_ref, rtol=1e-9, atol=1e-11)
    np.testing.assert_allclose(dh0, g[4], rtol=1e-9, atol=1e-11)
