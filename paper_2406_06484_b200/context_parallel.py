"""Context parallelism across GPUs.

Rank r of a process group holds tokens [r*L_r, (r+1)*L_r) of every (b, h)
unit (the sequence is cut into consecutive parts, one per rank).  The parts
are stitched by the affine composition of the chunk state update (PAPER.md
§3.2 Eq. 8; include/deltanet.h "Context parallelism"):

  forward   1. (Psi_r, Hloc_r) = deltanet_fwd_transition(part r)      [1-2 launches]
            2. all-gather (Psi, Hloc) over the group                  [NCCL]
            3. H_start(r) = deltanet_state_scan(part r)               [1 launch]
            4. o_r = deltanet_fwd(part r, h0 = H_start(r))            [the usual kernels]
  backward  1. dHloc_r = deltanet_bwd_transition(part r, dO_r)        [1-2 launches]
            2. all-gather dHloc                                       [NCCL]
            3. dH_end(r) = deltanet_state_scan(part r, reverse)       [1 launch]
            4. grads_r = deltanet_bwd(part r, h0 = H_start(r), dhT = dH_end(r))

The exchange is O(P * B*H*Dk*(Dk+Dv)) fp32 bytes, independent of L; every
step except the all-gather is a CUDA kernel of libdeltanet.  ``ops`` exists
so the CPU multi-process tests (tests/test_dist_cpu.py, gloo) can drive this
exact orchestration with stand-in ops; the default is the CUDA library and
there is no fallback.
"""
from __future__ import annotations

from dataclasses import dataclass
from types import SimpleNamespace

import torch
import torch.distributed as dist


def _cuda_ops():
    from . import (alloc_workspace, deltanet_bwd, deltanet_bwd_transition, deltanet_fwd,
                   deltanet_fwd_transition, deltanet_state_scan, make_desc)

    def alloc(q, v, l2norm):  # one workspace for the transition, the fwd and the bwd
        B, H, L, Dk = q.shape
        return alloc_workspace(make_desc(B, H, L, Dk, v.shape[-1], 64, q.dtype, l2norm=l2norm),
                               q.device)
    return SimpleNamespace(fwd_transition=deltanet_fwd_transition,
                           bwd_transition=deltanet_bwd_transition,
                           state_scan=deltanet_state_scan, fwd=deltanet_fwd,
                           bwd=deltanet_bwd, alloc=alloc)


def _all_gather(x: torch.Tensor, group) -> torch.Tensor:
    """[P, *x.shape] (rank order).  One collective; the tensor variant on NCCL."""
    world = dist.get_world_size(group)
    if dist.get_backend(group) == "nccl":
        out = torch.empty((world,) + tuple(x.shape), dtype=x.dtype, device=x.device)
        dist.all_gather_into_tensor(out, x.contiguous(), group=group)
        return out
    parts = [torch.empty_like(x) for _ in range(world)]
    dist.all_gather(parts, x.contiguous(), group=group)
    return torch.stack(parts)


@dataclass
class CPState:
    """What the context-parallel forward keeps for its backward."""
    workspace: torch.Tensor
    h_start: torch.Tensor
    psi_all: torch.Tensor


def cp_fwd(q, k, v, beta, *, group=None, h0=None, l2norm=True, ops=None):
    """Forward of this rank's part.  h0 (the state before part 0) must be the
    same on every rank (or None).  Returns (o, hT, state); hT is the state
    after this rank's part (the sequence's final state on the last rank)."""
    ops = ops or _cuda_ops()
    r = dist.get_rank(group)
    ws = ops.alloc(q, v, l2norm) if hasattr(ops, "alloc") else None
    psi, hloc = ops.fwd_transition(q, k, v, beta, l2norm=l2norm, workspace=ws)
    both = _all_gather(torch.stack((psi, hloc)), group)  # [P, 2, B, H, D, D]
    psi_all, loc_all = both[:, 0].contiguous(), both[:, 1].contiguous()
    h_start = ops.state_scan(psi_all, loc_all, r, edge=h0)
    o, hT, ws = ops.fwd(q, k, v, beta, h0=h_start, l2norm=l2norm, save_states=True,
                        workspace=ws)
    return o, hT, CPState(ws, h_start, psi_all)


def cp_bwd(q, k, v, beta, dO, state: CPState, *, group=None, dhT=None, l2norm=True, ops=None):
    """Backward of this rank's part.  dhT (cotangent of the sequence's final
    state) must be the same on every rank (or None).  Returns
    (dq, dk, dv, dbeta, dh_start); dh_start of rank 0 is dl/dh0."""
    ops = ops or _cuda_ops()
    r = dist.get_rank(group)
    dloc = ops.bwd_transition(q, k, v, beta, dO, l2norm=l2norm, workspace=state.workspace)
    dloc_all = _all_gather(dloc, group)
    dh_end = ops.state_scan(state.psi_all, dloc_all, r, reverse=True, edge=dhT)
    return ops.bwd(q, k, v, beta, dO, h0=state.h_start, dhT=dh_end, l2norm=l2norm,
                   workspace=state.workspace)


__all__ = ["cp_fwd", "cp_bwd", "CPState"]
