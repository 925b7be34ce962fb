"""Multi-process (gloo, world_size 2, CPU) test of the sharding / gather
code bench.py uses on N B200 (paper_2406_06484_b200.data_parallel): rank r
owns the contiguous batch rows shard_rows(B, N, r) of the B=64 "sharded"
config, the (b, h) units are independent (no collective in the step), and
an all-gather of the per-rank outputs reassembles exactly the
single-process result.  The fp64 oracle stands in for the kernels here (test
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


def _dp_oracle_ops():
    """Stand-in for the CUDA calls ShardedStep makes (same signatures), on
    fp64 CPU tensors: the oracle.  Test infrastructure only."""
    from types import SimpleNamespace
    n = lambda t: t.numpy()

    def fwd(q, k, v, beta, *, chunk, workspace, want_hT, out):
        o, _ = oracle.recurrent_fwd(n(q), n(k), n(v), n(beta), nthreads=1)
        out.copy_(torch.from_numpy(o))

    def bwd(q, k, v, beta, dO, *, chunk, workspace, want_dh0, out):
        g = oracle.recurrent_bwd(n(q), n(k), n(v), n(beta), n(dO), nthreads=1)
        for t, a in zip(out, g[:4]):
            t.copy_(torch.from_numpy(a))
    return SimpleNamespace(fwd=fwd, bwd=bwd, alloc=lambda q, v, chunk: None)


def _worker(rank, world, port, B_total, cfg_kw, out_q):
    """One rank of bench.py's data-parallel step, through the package's own
    sharding code (paper_2406_06484_b200.data_parallel): its rows of the
    seeded inputs, the local fwd + bwd (oracle ops), the max-over-ranks
    timing rule, and the gather of outputs and gradients."""
    from paper_2406_06484_b200 import data_parallel as dp
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = synth.custom_config(**cfg_kw)
    rows = dp.shard_rows(B_total, world, rank)
    x = synth.make_inputs(cfg, b_range=rows)
    t = {f: torch.from_numpy(np.ascontiguousarray(x[f], dtype=np.float64))
         for f in ("q", "k", "v", "beta", "dO")}
    st = dp.ShardedStep(t["q"], t["k"], t["v"], t["beta"], t["dO"], B_total=B_total,
                        chunk=cfg.chunk, ops=_dp_oracle_ops())
    st.step()
    outs = [a.numpy() for a in st.gather()]
    tmax = dp.max_over_ranks([rank + 1.0, 10.0 * (rank + 1)], "cpu")
    if rank == 0:
        out_q.put((outs, tmax, st.world, [len(dp.shard_rows(B_total, world, r))
                                          for r in range(world)]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("B_total", [4, 5])
def test_shard_gather_matches_single_process(B_total):
    """2 gloo ranks: the gathered outputs and gradients have the full
    [B, H, L, d] layout and equal the single-process result bit for bit
    (B = 5: uneven slabs 3 + 2, padded in the gather)."""
    world = 2
    cfg_kw = dict(B=B_total, H=2, L=40, Dk=8, Dv=8, chunk=16, dtype="bf16", index=77)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, B_total, cfg_kw, q))
             for r in range(world)]
    for p in procs:
        p.start()
    outs, tmax, n_gpus, sizes = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert n_gpus == 2
    assert sizes == [(B_total + 1) // 2, B_total // 2]
    assert tmax == [2.0, 20.0]  # max over ranks, element-wise
    cfg = synth.custom_config(**cfg_kw)
    x = synth.make_inputs(cfg)
    o, _ = oracle.recurrent_fwd(x["q"], x["k"], x["v"], x["beta"], nthreads=1)
    ref = [o, *oracle.recurrent_bwd(x["q"], x["k"], x["v"], x["beta"], x["dO"], nthreads=1)[:4]]
    shapes = [(B_total, 2, 40, 8)] * 4 + [(B_total, 2, 40)]
    for a, b, shp in zip(outs, ref, shapes):
        assert a.shape == shp
        assert np.array_equal(a, b)


def test_shard_rows_cover_the_batch():
    from paper_2406_06484_b200.data_parallel import shard_rows
    for B in (1, 7, 8, 64):
        for world in (1, 2, 3, 8):
            rs = [shard_rows(B, world, r) for r in range(world)]
            assert [i for r in rs for i in r] == list(range(B))
            assert max(map(len, rs)) - min(map(len, rs)) <= 1
    assert shard_rows(64, 8, 3) == range(24, 32)   # configs[4] at 8 GPUs: 8 rows per rank


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
