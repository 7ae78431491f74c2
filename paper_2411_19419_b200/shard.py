"""Batch sharding for the multi-GPU apply (BASELINE north_star: each GPU holds a
CSR replica and owns a contiguous batch slice; no collective on the hot path).

Only host logic lives here: which images a rank owns, and the max-over-ranks
reduction of device timings.  Works with any torch.distributed backend (NCCL on
the B200 box, gloo in the CPU tests)."""
from __future__ import annotations

from typing import Tuple


def batch_slice(total: int, rank: int, world: int) -> Tuple[int, int]:
    """(first image, image count) of `rank`'s contiguous slice; the first
    total % world ranks get one extra image."""
    if world < 1 or not 0 <= rank < world or total < 0:
        raise ValueError(f"batch_slice: bad arguments total={total} rank={rank} world={world}")
    base, extra = divmod(total, world)
    count = base + (1 if rank < extra else 0)
    start = rank * base + min(rank, extra)
    return start, count


def max_over_ranks(value: float, device=None) -> float:
    """All-reduce MAX of a per-rank scalar (e.g. elapsed ms); identity when
    torch.distributed is not initialised."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())
