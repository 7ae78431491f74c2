"""NCCL sanity of the multi-GPU helpers (shard.py) with the NCCL backend at
world size = number of visible GPUs (1 on a gpurun box): init with device_id,
barrier, max/sum over ranks (float64 all-reduce) and the final gather."""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_19419_b200.shard import batch_slice, gather_outputs, max_over_ranks, sum_over_ranks  # noqa: E402

rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
local = int(os.environ.get("LOCAL_RANK", 0))
dev = torch.device("cuda", local)
torch.cuda.set_device(dev)
dist.init_process_group("nccl", device_id=dev)
dist.barrier()
assert max_over_ranks(1.5 + rank, dev) == 1.5 + world - 1
assert sum_over_ranks(2.0, dev) == 2.0 * world
total = 8 * world + 1
start, count = batch_slice(total, rank, world)
Y = torch.arange(start, start + count, dtype=torch.float32, device=dev)[:, None] * 10 + torch.arange(5.0, device=dev)
out = gather_outputs(Y, total)
if rank == 0:
    want = torch.arange(total, dtype=torch.float32, device=dev)[:, None] * 10 + torch.arange(5.0, device=dev)
    assert torch.equal(out, want)
    print(f"nccl smoke ok: world={world} backend={dist.get_backend()} nccl={torch.cuda.nccl.version()}")
dist.barrier()
dist.destroy_process_group()
