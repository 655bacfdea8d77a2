"""CPU, world_size 2 (gloo): the one-process-per-GPU sharding logic of
paper_2601_06349_b200/dist.py — contiguous shards, a 2-unit all-gather halo
exchange, per-shard repair with halos — reproduces the whole-buffer oracle,
including empty / ragged shards and adversarial shard-edge patterns. The
per-shard compute is the CPU oracle here (no GPU); on the B200 it is the
sm_100a kernel (tests/test_gpu_parity.py covers that part)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2601_06349_b200 import dist as pdist


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, total, cuts, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x = O.gen_config(4, total, seed=4, shard_len=total // world)
        a, b = cuts[rank], cuts[rank + 1]
        shard = torch.from_numpy(x[a:b].view(np.int16).copy())

        def compute(s, out, left, right):
            res = O.stencil(s.numpy().view(np.uint16), left, right)
            out.copy_(torch.from_numpy(res.view(np.int16)))
            return out

        out = pdist.repair_shard(shard, torch.empty_like(shard), compute=compute, all_nonempty=False)
        sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(sizes, torch.tensor([out.numel()]))
        m = int(max(s.item() for s in sizes))
        padded = torch.zeros(m, dtype=torch.int32)  # gloo has no int16 collectives
        padded[: out.numel()] = out.to(torch.int32) & 0xFFFF
        parts = [torch.zeros(m, dtype=torch.int32) for _ in range(world)]
        dist.all_gather(parts, padded)
        if rank == 0:
            got = np.concatenate([p[: int(s.item())].numpy().astype(np.uint16) for p, s in zip(parts, sizes)])
            q.put(bool((got == O.stencil(x)).all()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cuts", [
    [0, 50_000, 100_000],            # equal shards, adversarial edge pattern at 50_000
    [0, 1, 100_000],                 # 1-unit shard
    [0, 0, 100_000],                 # empty shard on rank 0
    [0, 99_999, 100_000],
])
def test_two_rank_halo_exchange(cuts):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, 100_000, cuts, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    assert q.get(timeout=10) is True


def test_shard_bounds():
    for total in (0, 1, 7, 100, 2**32 + 5):
        for world in (1, 2, 3, 8):
            b = [pdist.shard_bounds(total, world, r) for r in range(world)]
            assert b[0][0] == 0 and b[-1][1] == total
            assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))
            assert max(e - s for s, e in b) - min(e - s for s, e in b) <= 1


def test_halos_from_edges_skips_empty():
    E = pdist.EMPTY
    edges = torch.tensor([[1, 2], [E, E], [3, 4], [E, E]], dtype=torch.int32)
    assert pdist.halos_from_edges(edges, 0) == (-1, 3)
    assert pdist.halos_from_edges(edges, 2) == (2, -1)
    assert pdist.halos_from_edges(edges, 1) == (2, 3)


def test_select_halos_matches_host_selection_with_empty_shards():
    """The device-side halo choice (no host sync) skips empty shards exactly
    like the host-side one; EMPTY reads as 0xFFFF, a non-surrogate, i.e.
    'outside'. D800 | empty | DC00 must pair across the empty shard."""
    E = pdist.EMPTY
    rng = np.random.default_rng(5)
    for _ in range(300):
        world = int(rng.integers(1, 9))
        e = [[int(a), int(b)] if rng.random() < 0.6 else [E, E]
             for a, b in rng.integers(0, 0x10000, size=(world, 2))]
        edges = torch.tensor(e, dtype=torch.int32)
        for r in range(world):
            sel = pdist.select_halos(edges, r).tolist()
            assert tuple(sel) == pdist.halos_from_edges(edges, r)
    edges = torch.tensor([[0x41, 0xD800], [E, E], [0xDC00, 0x41]], dtype=torch.int32)
    assert pdist.select_halos(edges, 0).tolist() == [E, 0xDC00]
    assert pdist.select_halos(edges, 2).tolist() == [0xD800, E]
    assert (E & 0xFFFF) == 0xFFFF and not O.stencil([0xFFFF, 0x41]).tolist() != [0xFFFF, 0x41]


def test_halo_pointer_offsets():
    edges = torch.zeros((4, 2), dtype=torch.int32)
    base = edges.data_ptr()
    assert pdist.halo_pointers(edges, 0) == (0, base + 8)
    assert pdist.halo_pointers(edges, 1) == (base + 4, base + 16)
    assert pdist.halo_pointers(edges, 3) == (base + 20, 0)


def _peerhalo_worker(rank, world, port, fail_rank, q):
    """PeerHalo's setup with the CUDA IPC pieces stubbed: when one rank cannot
    map its neighbours, every rank must raise (so callers fall back together)
    instead of the healthy ranks blocking in a barrier."""
    import torch.multiprocessing.reductions as R

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        def rebuild(*a):
            if rank == fail_rank:
                raise RuntimeError("cannot open IPC handle")
            return torch.zeros(4, dtype=torch.int16)

        R.reduce_tensor = lambda t: (rebuild, (None,) * 6 + (rank,) + (None,) * 8)
        torch.cuda.can_device_access_peer = lambda a, b: True
        torch.cuda.synchronize = lambda *a, **k: None
        shard = torch.zeros(8, dtype=torch.int16)
        try:
            h = pdist.PeerHalo(shard)
            q.put((rank, "ok", h.left_ptr != 0 or h.right_ptr != 0))
        except RuntimeError as e:
            q.put((rank, "raised", "PeerHalo setup failed" in str(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("fail_rank", [-1, 0, 1])
def test_peer_halo_setup_failure_is_collective(fail_rank):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_peerhalo_worker, args=(r, 2, port, fail_rank, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    if fail_rank < 0:
        assert res == [(0, "ok", True), (1, "ok", True)]
    else:
        assert res == [(0, "raised", True), (1, "raised", True)]
