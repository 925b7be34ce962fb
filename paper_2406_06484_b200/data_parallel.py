"""Batch x head data parallelism across GPUs.

The (b, h) units of a DeltaNet layer are independent in the forward and the
backward (the chunk recurrence of PAPER.md §3.2, Eq. 8-9, runs per
head), so a step shards with no collective: rank r of a group owns the
contiguous batch rows ``shard_rows(B, world, r)`` -- one contiguous slab of
every [B, H, L, d] tensor -- and runs the ordinary library calls on it.
NCCL is used only to gather outputs and gradients back into the full
[B, H, L, d] layout (north_star: "NCCL used only to gather outputs and
gradients"); the gather is outside the step.

``ops`` exists so the CPU multi-process tests (tests/test_dist_cpu.py, gloo)
drive this exact code with a stand-in for the kernels; the default is the
CUDA library and there is no fallback.  bench.py times ``ShardedStep.step``
and reports ``gather`` separately.
"""
from __future__ import annotations

from types import SimpleNamespace

import torch
import torch.distributed as dist


def shard_rows(B: int, world: int, rank: int) -> range:
    """Contiguous batch rows of `rank`: the first B % world ranks get one
    row more (B need not be a multiple of world; a rank may get none)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("rank outside the group")
    base, extra = divmod(B, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def _cuda_ops():
    from . import alloc_workspace, deltanet_bwd, deltanet_fwd, make_desc

    def alloc(q, v, chunk):
        B, H, L, Dk = q.shape
        return alloc_workspace(make_desc(B, H, L, Dk, v.shape[-1], chunk, q.dtype,
                                         save_states=True), q.device)
    return SimpleNamespace(fwd=deltanet_fwd, bwd=deltanet_bwd, alloc=alloc)


class ShardedStep:
    """One rank's share of a data-parallel fwd+bwd step.  q, k, v, beta, dO
    are this rank's rows (``shard_rows``) of the global [B_total, H, L, d]
    tensors, already on the rank's device.  ``step()`` runs deltanet_fwd
    (saving the chunk states) + deltanet_bwd into preallocated outputs;
    ``gather()`` returns the full (o, dq, dk, dv, dbeta) on every rank."""

    def __init__(self, q, k, v, beta, dO, *, B_total: int, chunk: int = 64, group=None,
                 ops=None, local: bool = False):
        """local=True: a single-process step of the whole batch even inside a
        process group (side measurements on one rank)."""
        self.ops = ops if ops is not None else _cuda_ops()
        self.q, self.k, self.v, self.beta, self.dO = q, k, v, beta, dO
        self.B_total, self.chunk, self.group = B_total, chunk, group
        dist_on = dist.is_initialized() and not local
        self.world = dist.get_world_size(group) if dist_on else 1
        self.rank = dist.get_rank(group) if dist_on else 0
        self.local = not dist_on
        rows = shard_rows(B_total, self.world, self.rank)
        if q.shape[0] != len(rows):
            raise ValueError(f"rank {self.rank} holds {q.shape[0]} rows, owns {len(rows)}")
        self.ws = self.ops.alloc(q, v, chunk) if q.shape[0] else None
        self.o = torch.empty_like(v)
        self.grads = (torch.empty_like(q), torch.empty_like(k), torch.empty_like(v),
                      torch.empty_like(beta))

    @property
    def tokens(self) -> int:
        """Tokens (batch rows x L) this rank processes per step."""
        return self.q.shape[0] * self.q.shape[2]

    def fwd(self):
        if self.q.shape[0]:
            self.ops.fwd(self.q, self.k, self.v, self.beta, chunk=self.chunk, workspace=self.ws,
                         want_hT=False, out=self.o)

    def bwd(self):
        if self.q.shape[0]:
            self.ops.bwd(self.q, self.k, self.v, self.beta, self.dO, chunk=self.chunk,
                         workspace=self.ws, want_dh0=False, out=self.grads)

    def step(self):
        self.fwd()
        self.bwd()

    def gather(self):
        """(o, dq, dk, dv, dbeta), each the full [B_total, ...] tensor."""
        if self.local:
            return (self.o, *self.grads)
        return tuple(gather_rows(t, self.B_total, self.group)
                     for t in (self.o, *self.grads))


def gather_rows(local: torch.Tensor, B_total: int, group=None) -> torch.Tensor:
    """All-gather the ranks' row slabs (``shard_rows`` order) into the full
    [B_total, ...] tensor.  Equal slabs go straight into the output with one
    collective (all_gather_into_tensor on NCCL); unequal ones are padded to
    the largest slab and trimmed."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return local
    world = dist.get_world_size(group)
    sizes = [len(shard_rows(B_total, world, r)) for r in range(world)]
    m = max(sizes)
    tail = tuple(local.shape[1:])
    if local.shape[0] < m:
        pad = torch.zeros((m - local.shape[0],) + tail, dtype=local.dtype, device=local.device)
        local = torch.cat([local, pad], 0)
    if dist.get_backend(group) == "nccl":
        full = torch.empty((world * m,) + tail, dtype=local.dtype, device=local.device)
        dist.all_gather_into_tensor(full, local.contiguous(), group=group)
        if all(s_ == m for s_ in sizes):
            return full  # already the [B_total, ...] layout, no copy
        parts = list(full.split(m, 0))
    else:
        parts = [torch.empty_like(local) for _ in range(world)]
        dist.all_gather(parts, local.contiguous(), group=group)
    if all(s == m for s in sizes):
        return torch.cat(parts, 0)
    return torch.cat([p[:s] for p, s in zip(parts, sizes)], 0)


def max_over_ranks(values, device, group=None):
    """Element-wise MAX over the group (the bench's timing rule: the slowest
    rank's device time)."""
    t = torch.tensor([float(x) for x in values], dtype=torch.float64, device=device)
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return t.tolist()


__all__ = ["shard_rows", "ShardedStep", "gather_rows", "max_over_ranks"]
