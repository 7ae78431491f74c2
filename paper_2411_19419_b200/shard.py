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


def gather_outputs(Y_local, total: int, root: int = 0):
    """The optional final gather (BASELINE north_star: "NCCL over NVLink is
    used only for an optional final gather"): every rank's [count, rows]
    output slice (count = batch_slice(total, rank, world)[1]) is collected on
    `root` in batch order.  Slices are padded to the largest count so one
    collective moves them (over NVLink / NVSwitch with NCCL); returns the
    [total, rows] tensor on root and None elsewhere.  Identity when
    torch.distributed is not initialised."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return Y_local
    world, rank = dist.get_world_size(), dist.get_rank()
    start, count = batch_slice(total, rank, world)
    if Y_local.shape[0] != count:
        raise ValueError(f"gather_outputs: rank {rank} holds {Y_local.shape[0]} images, expected {count}")
    most = batch_slice(total, 0, world)[1]
    rows = Y_local.shape[1] if Y_local.dim() == 2 else 0
    send = Y_local
    if count < most:
        send = torch.zeros(most, rows, dtype=Y_local.dtype, device=Y_local.device)
        send[:count] = Y_local
    send = send.contiguous()
    dev = send.device
    if dist.get_backend() != "nccl":  # gloo gathers host tensors
        send = send.cpu()
    bufs = [torch.empty_like(send) for _ in range(world)] if rank == root else None
    dist.gather(send, gather_list=bufs, dst=root)
    if rank != root:
        return None
    return torch.cat([bufs[r][: batch_slice(total, r, world)[1]] for r in range(world)], dim=0).to(dev)
