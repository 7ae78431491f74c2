"""Multi-rank host logic on CPU with gloo (world_size 2): batch slices cover the
batch exactly once and the timing reduction is a true max over ranks."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2411_19419_b200.shard import batch_slice


def test_batch_slice_partition():
    for total in (0, 1, 7, 64, 256, 257):
        for world in (1, 2, 3, 4, 8):
            seen = []
            for r in range(world):
                s, c = batch_slice(total, r, world)
                seen += list(range(s, s + c))
            assert seen == list(range(total))
            counts = [batch_slice(total, r, world)[1] for r in range(world)]
            assert max(counts) - min(counts) <= 1
    with pytest.raises(ValueError):
        batch_slice(10, 2, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2411_19419_b200.shard import batch_slice, max_over_ranks, sum_over_ranks
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    start, count = batch_slice(256, rank, world)
    elapsed = 10.0 + rank * 5.0
    q.put((rank, start, count, max_over_ranks(elapsed), sum_over_ranks(count)))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_shards_and_max():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=10) for _ in range(world))
    assert [(r[1], r[2]) for r in res] == [(0, 128), (128, 128)]
    assert all(r[3] == 15.0 for r in res)  # max over ranks, seen identically by all
    assert all(r[4] == 256 for r in res)


def _gather_worker(rank, world, port, total, q):
    import torch
    import torch.distributed as dist
    from paper_2411_19419_b200.shard import batch_slice, gather_outputs
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    start, count = batch_slice(total, rank, world)
    # each image b's "output" row is b * 10 + column index
    Y = torch.arange(start, start + count, dtype=torch.float32)[:, None] * 10 + torch.arange(6.0)[None]
    out = gather_outputs(Y, total)
    q.put((rank, None if out is None else out.tolist()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("total", [7, 8])
def test_gloo_world2_final_gather(total):
    """The optional final gather puts every rank's slice on rank 0 in batch
    order (ragged slices included); other ranks get None."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, world, port, total, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = dict(q.get(timeout=10) for _ in range(world))
    assert res[1] is None
    want = [[b * 10.0 + c for c in range(6)] for b in range(total)]
    assert res[0] == want
