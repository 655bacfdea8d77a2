"""Run under torchrun with 2+ processes (all on cuda:0 when only one GPU is
visible; the processes' kernels never wait on each other): PeerHalo maps the
neighbours' shards by CUDA IPC and every step is a single kernel per rank.
Rank 0 checks the gathered result against the CPU oracle."""
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
    dev = torch.device("cuda", local % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    ok = True
    for cfg, per_rank in ((4, 1 << 20), (1, (1 << 20) + 4097), (0, 8191), (1, 17)):
        total = per_rank * world
        x = _lib.gen_config(cfg, total, seed=cfg, first=rank * per_rank, count=per_rank,
                            shard_len=per_rank if cfg == 4 else 0, device=dev)
        for in_place in (True, False):
            shard = x.clone()
            torch.cuda.synchronize()
            halo = pdist.PeerHalo(shard)
            out = shard if in_place else torch.empty_like(shard)
            for _ in range(3):  # repeated in-place steps see their own / neighbours' rewrites: benign
                halo.repair(out)
            torch.cuda.synchronize()
            res = out.cpu().numpy().view(np.uint16).astype(np.int32)
            parts = [torch.zeros(per_rank, dtype=torch.int32) for _ in range(world)]
            dist.all_gather(parts, torch.from_numpy(res))
            if rank == 0:
                got = torch.cat(parts).numpy().astype(np.uint16)
                full = O.gen_config(cfg, total, seed=cfg, shard_len=per_rank if cfg == 4 else 0)
                good = bool((got == O.stencil(full)).all())
                ok &= good
                print(cfg, per_rank, in_place, "OK" if good else "MISMATCH", flush=True)
            dist.barrier()
            del halo
    dist.destroy_process_group()
    if rank == 0:
        print("ALL OK" if ok else "FAILED")
        sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
