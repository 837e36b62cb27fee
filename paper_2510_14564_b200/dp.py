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


# ---------------------------------------------------------------- sharded update (§8(e) 2)
# reduce-scatter of grad -> Adam on this rank's 1/G of theta -> all-gather of theta: the
# same link bytes as the all-reduce ((G-1)/G S each way), but each rank runs Adam over S/G
# elements only and keeps exp_avg / exp_avg_sq for its shard alone.


def shard_layout(total: int, world: int, align: int = 4) -> tuple[int, int]:
    """(shard, padded): each rank owns `shard` consecutive elements (a multiple of `align`,
    so every shard starts 16-byte aligned for the vectorised Adam); theta and grad are
    allocated with `padded` = world * shard >= total elements, the tail being padding."""
    if world < 1 or total < 0:
        raise ValueError(f"bad layout total={total} world={world}")
    per = -(-total // world)
    shard = -(-per // align) * align
    return shard, shard * world


def shard_range(rank: int, world: int, total: int, align: int = 4) -> tuple[int, int]:
    """[begin, end) of rank's shard in the padded layout."""
    shard, _ = shard_layout(total, world, align)
    return rank * shard, (rank + 1) * shard


def reduce_scatter_grads(grad_padded: torch.Tensor, rank: int, world: int) -> torch.Tensor:
    """Sum grad over ranks into this rank's shard, in place (NCCL in-place reduce-scatter:
    the output is the rank's own slice of the input).  Returns the shard view.  Only the
    shard is meaningful afterwards; the rest still holds this rank's partial sums."""
    shard = grad_padded.numel() // world
    out = grad_padded.narrow(0, rank * shard, shard)
    if world > 1:
        dist.reduce_scatter_tensor(out, grad_padded, op=dist.ReduceOp.SUM)
    return out


def all_gather_params(theta_padded: torch.Tensor, rank: int, world: int) -> None:
    """Every rank's updated shard of theta to every rank, in place (NCCL in-place
    all-gather), so the replicas are identical again."""
    if world > 1:
        shard = theta_padded.numel() // world
        dist.all_gather_into_tensor(theta_padded, theta_padded.narrow(0, rank * shard, shard))


# ---------------------------------------------------------------- overlapped all-reduce (§8(e) 1)
# The chain rule (a10) runs over the Gaussians in chunks; a chunk's gradient -- in each of
# theta's five segments the sub-range of its Gaussians -- is all-reduced on a communication
# stream while the next chunk computes, so the exchange hides behind a10 except for the last
# chunk.

SEGMENT_WIDTHS = (3, 3, 4, 1, 48)  # means, log_scales, quats, opacity logit, sh (theta layout)


def gaussian_chunks(n: int, chunks: int) -> list[tuple[int, int]]:
    """[begin, end) Gaussian ranges of ~equal size covering [0, n)."""
    if n < 0 or chunks < 1:
        raise ValueError(f"bad chunking n={n} chunks={chunks}")
    step = -(-n // chunks) if n else 0
    return [(b, min(n, b + step)) for b in range(0, n, step)] if n else []


def segment_slices(n: int, begin: int, end: int) -> list[tuple[int, int]]:
    """The theta elements of Gaussians [begin, end): one [lo, hi) per segment."""
    out, base = [], 0
    for w in SEGMENT_WIDTHS:
        out.append((base + w * begin, base + w * end))
        base += w * n
    return out


def allreduce_chunk(grad: torch.Tensor, n: int, begin: int, end: int, world: int, async_op: bool = False):
    """All-reduce (SUM) of the gradient elements of Gaussians [begin, end) -- five contiguous
    collectives; returns their work handles when async_op."""
    works = []
    if world > 1:
        for lo, hi in segment_slices(n, begin, end):
            w = dist.all_reduce(grad.narrow(0, lo, hi - lo), op=dist.ReduceOp.SUM, async_op=async_op)
            if async_op:
                works.append(w)
    return works
