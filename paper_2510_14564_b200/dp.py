"""Data parallelism over camera views.

Views are independent units with one real exchange per batch: every rank holds a full
replica of theta[59N], renders its share of the batch's views (views i with
i % world == rank), accumulates grad += over them through libbgs, then one SUM
all-reduce of grad[59N] (NCCL over NVLink 5 / NVSwitch on the GPU box; gloo in the CPU
tests) and the same deterministic Adam on every rank keeps the replicas bit-identical.

Host-side logic only (no compute): libbgs does every step of the path.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def views_for_rank(views, rank: int, world: int):
    """Round-robin split of the batch's views: rank r gets views r, r+G, r+2G, ..."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    return [v for i, v in enumerate(views) if i % world == rank]


def broadcast_params(theta: torch.Tensor, world: int, src: int = 0) -> None:
    """Replicas start identical (theta from rank `src`)."""
    if world > 1:
        dist.broadcast(theta, src)


def allreduce_grads(grad: torch.Tensor, world: int) -> None:
    """The batch's one exchange step: grad[59N] summed over ranks (R20: the caller scaled
    dL/dimage by 1/B, so the sum is the gradient of the batch-mean loss)."""
    if world > 1:
        dist.all_reduce(grad, op=dist.ReduceOp.SUM)
