"""Data-parallel replicas: one process per GPU, one NCCL all-reduce of the
weight gradients per iteration (the only collective of the path).

Every rank plans the identical schedule (the plan depends only on the net,
per-replica batch, pool and features -- parameters and their gradients live
outside the pool accounting, reference costmodel.py:3-6), so the collective
cannot perturb residency.  Gradients are summed over ranks and the SGD update
applies ``lr * grad / world``, i.e. the gradient of the global-batch mean loss.
Weights start identical on every rank (same init seed), so no broadcast is
needed; ``broadcast_parameters`` exists for externally supplied weights.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

__all__ = ["DPContext", "init", "average_gradients", "broadcast_parameters", "rank_seed"]


@dataclass
class DPContext:
    rank: int = 0
    world: int = 1
    local_rank: int = 0
    backend: str = "none"

    @property
    def active(self) -> bool:
        return self.world > 1


def init(backend: str | None = None) -> DPContext:
    """Initialise from torchrun's environment (RANK/WORLD_SIZE/LOCAL_RANK)."""
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world <= 1:
        return DPContext()
    if backend is None:
        backend = "nccl" if torch.cuda.is_available() else "gloo"
    if not dist.is_initialized():
        kw = {}
        if backend == "nccl":
            torch.cuda.set_device(local)
            kw["device_id"] = torch.device(f"cuda:{local}")
        dist.init_process_group(backend, **kw)
    return DPContext(rank=rank, world=world, local_rank=local, backend=backend)


def rank_seed(base: int, ctx: DPContext) -> int:
    """Per-rank data seed: each replica draws a different shard of the batch."""
    return base + 7919 * ctx.rank


def average_gradients(flat, ctx: DPContext, scale_in_update: bool = True):
    """Sum the flat fp32 gradient block over ranks (in place).

    With ``scale_in_update`` the 1/world factor is left to the fused SGD kernel
    (``Executor.apply_update(lr, 1/world)``); otherwise it is applied here.
    """
    if not ctx.active:
        return flat
    import torch.distributed as dist
    dist.all_reduce(flat, op=dist.ReduceOp.SUM)
    if not scale_in_update:
        flat.div_(ctx.world)
    if flat.is_cuda:
        # the executor's SGD kernel runs on its own stream, not torch's
        import torch
        torch.cuda.current_stream(flat.device).synchronize()
    return flat


def broadcast_parameters(flat, ctx: DPContext, src: int = 0):
    if ctx.active:
        import torch.distributed as dist
        dist.broadcast(flat, src)
    return flat
