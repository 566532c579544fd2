"""Multi-GPU host logic: frame sharding and max-over-ranks timing.

Frames are independent problems, so the path shards by frame
with no data-path collective: rank r of a world of P processes its own
contiguous block of frames.  torch.distributed (NCCL on GPUs, gloo in the CPU
tests) is used only for barriers, the max-over-ranks reduction of timings
and, optionally, gathering results to rank 0 outside the timed region.
"""
from __future__ import annotations

from typing import Tuple


def weak_shard(frames_per_rank: int, rank: int) -> Tuple[int, int]:
    """Weak scaling: every rank owns `frames_per_rank` frames; rank r's are
    global frames [r * n, (r + 1) * n) (frame f is the scene of seed + f)."""
    if frames_per_rank < 1 or rank < 0:
        raise ValueError("frames_per_rank >= 1 and rank >= 0 required")
    return rank * frames_per_rank, frames_per_rank


def strong_shard(total: int, world: int, rank: int) -> Tuple[int, int]:
    """Strong scaling: `total` frames split into contiguous near-equal blocks
    (the first total % world ranks get one extra frame)."""
    if not (0 <= rank < world) or total < 0:
        raise ValueError("0 <= rank < world and total >= 0 required")
    base, extra = divmod(total, world)
    first = rank * base + min(rank, extra)
    return first, base + (1 if rank < extra else 0)


def view_shard(views, world: int, rank: int):
    """Shard by peripheral view (24 views over 8 GPUs): views
    are independent once each rank has the whole frame (it recomputes the
    frame statistics itself, so h is identical everywhere).  Returns rank r's
    contiguous near-equal block of (index, baseline) pairs."""
    first, n = strong_shard(len(views), world, rank)
    return [(i, tuple(views[i])) for i in range(first, first + n)]


def max_over_ranks(value: float, device=None) -> float:
    """All-reduce MAX of a per-rank scalar (identity when not distributed)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_to_rank0(tensor, device=None):
    """Gather equally-shaped per-rank tensors to rank 0 (list on rank 0, None
    elsewhere); used outside timed regions only."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return [tensor]
    world = dist.get_world_size()
    if dist.get_rank() == 0:
        out = [tensor.new_empty(tensor.shape) for _ in range(world)]
        dist.gather(tensor, out, dst=0)
        return out
    dist.gather(tensor, None, dst=0)
    return None
