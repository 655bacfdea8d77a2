"""Run under torchrun: each rank repairs its shard of one logical buffer with
paper_2601_06349_b200.dist.repair_shard (NCCL halo gather + interior/edge
split on two streams) and rank 0 checks the gathered result against the CPU
oracle. Used by tests/test_gpu_dist.py at world size 1 (one GPU here); the
same script runs unchanged at world size 8."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
from paper_2601_06349_b200 import _lib  # noqa: E402
from paper_2601_06349_b200 import dist as pdist  # noqa: E402


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pdist.init_process_group_for_repair("nccl", device_id=dev)
    rank, world = dist.get_rank(), dist.get_world_size()
    ok = True
    for cfg, per_rank in ((4, 1 << 20), (1, (1 << 20) + 4097), (0, 8191), (1, 17)):
        total = per_rank * world
        x = _lib.gen_config(cfg, total, seed=cfg, first=rank * per_rank, count=per_rank,
                            shard_len=per_rank if cfg == 4 else 0, device=dev)
        for in_place in (True, False):
            for overlap in (True, False):
                src = x.clone()
                out = src if in_place else torch.empty_like(src)
                pdist.repair_shard(src, out, overlap=overlap)
                b = out.view(torch.uint8)  # NCCL has no 16-bit integer type
                parts = [torch.empty_like(b) for _ in range(world)]
                dist.all_gather(parts, b)
                if rank == 0:
                    got = torch.cat(parts).cpu().numpy().view(np.uint16)
                    full = O.gen_config(cfg, total, seed=cfg, shard_len=per_rank if cfg == 4 else 0)
                    good = bool((got == O.stencil(full)).all())
                    ok &= good
                    print(cfg, per_rank, in_place, overlap, "OK" if good else "MISMATCH", flush=True)
    dist.destroy_process_group()
    if rank == 0:
        print("ALL OK" if ok else "FAILED")
        sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
