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
