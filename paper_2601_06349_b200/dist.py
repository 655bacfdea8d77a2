"""One-process-per-GPU sharding of one logical UTF-16 buffer (north star item 5).

The stencil needs exactly one unit on each side of a contiguous shard
(SURVEY.md §8e), so the only exchange step is 2 units per rank: every rank
contributes (first unit, last unit) of its shard to one tiny all-gather, and
the repair kernel reads its neighbours' units straight from the gathered
device tensor (u16m_to_well_formed_halo_ptr) — no host synchronisation inside
a step. Ordering is not required even in place: a neighbour's edge unit
yields the same decision whether it was read before or after that neighbour
rewrote it.

Host-side logic only; the compute call is injected so the same code runs with
NCCL + the sm_100a kernel (bench.py) and with gloo + the CPU oracle
(tests/test_dist_gloo.py).
"""
from __future__ import annotations

from typing import Optional

import torch
import torch.distributed as dist

EMPTY = -1  # sentinel for an empty shard's edge


def shard_bounds(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, as-equal-as-possible shard [start, end) of rank."""
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def edge_tensor(shard: torch.Tensor) -> torch.Tensor:
    """int32 [first, last] of a shard of int16/uint16 units (EMPTY if empty)."""
    if shard.numel() == 0:
        return torch.full((2,), EMPTY, dtype=torch.int32, device=shard.device)
    u = shard.view(torch.int16)
    return torch.stack([u[0], u[-1]]).to(torch.int32) & 0xFFFF


def gather_edges(shard: torch.Tensor, group=None, device: Optional[torch.device] = None) -> torch.Tensor:
    """[world, 2] int32 tensor of every rank's (first, last) unit."""
    world = dist.get_world_size(group)
    e = edge_tensor(shard)
    if device is not None:
        e = e.to(device)
    out = torch.empty(world * 2, dtype=torch.int32, device=e.device)
    dist.all_gather_into_tensor(out, e, group=group)
    return out.view(world, 2)


def halos_from_edges(edges: torch.Tensor, rank: int) -> tuple[int, int]:
    """(left, right) neighbour units for `rank`, skipping empty shards; -1 at
    the logical buffer's ends. Host values (synchronises if on device)."""
    e = edges.cpu().tolist()
    left = right = -1
    for r in range(rank - 1, -1, -1):
        if e[r][1] != EMPTY:
            left = e[r][1]
            break
    for r in range(rank + 1, len(e)):
        if e[r][0] != EMPTY:
            right = e[r][0]
            break
    return left, right


def select_halos(edges: torch.Tensor, rank: int) -> torch.Tensor:
    """int32 [left, right] on the edges' device, with no host sync: the last
    unit of the nearest NON-EMPTY shard before `rank` and the first unit of
    the nearest non-empty shard after it, EMPTY (-1) where there is none. The
    low 16 bits of EMPTY read as 0xFFFF, a non-surrogate, which the stencil
    treats exactly like "outside the buffer" — so the kernel can read both
    halos through pointers into this tensor unconditionally."""
    world = edges.shape[0]
    idx = torch.arange(world, device=edges.device)
    firsts, lasts = edges[:, 0], edges[:, 1]
    li = torch.where((idx < rank) & (lasts != EMPTY), idx, -1).max()
    ri = torch.where((idx > rank) & (firsts != EMPTY), idx, world).min()
    left = torch.where(li >= 0, lasts[li.clamp(min=0)], EMPTY)
    right = torch.where(ri < world, firsts[ri.clamp(max=world - 1)], EMPTY)
    return torch.stack([left, right]).to(torch.int32)


def halo_pointers(edges: torch.Tensor, rank: int) -> tuple[int, int]:
    """Device addresses of the neighbours' edge units inside the gathered
    int32 edges tensor (the low 16 bits of each little-endian int32 are the
    unit), 0 for none. Only valid when every shard is non-empty (an empty
    neighbour's EMPTY entry would hide the shard beyond it; see
    select_halos)."""
    world = edges.shape[0]
    base = edges.data_ptr()
    left = base + 4 * (2 * (rank - 1) + 1) if rank > 0 else 0
    right = base + 4 * (2 * (rank + 1)) if rank + 1 < world else 0
    return left, right


_side_streams: dict = {}


def _side_stream(device: torch.device) -> torch.cuda.Stream:
    """High-priority side stream: the gather + edge tiles must be scheduled
    ahead of the interior grid's pending CTAs, not after them."""
    if device not in _side_streams:
        lo, hi = torch.cuda.Stream.priority_range()
        _side_streams[device] = torch.cuda.Stream(device=device, priority=hi)
    return _side_streams[device]


def init_process_group_for_repair(backend: str = "nccl", **kw):
    """init_process_group with NCCL on high-priority streams (the halo gather
    then preempts the interior grid's queued CTAs instead of waiting for them)."""
    if backend == "nccl":
        opts = dist.ProcessGroupNCCL.Options()
        opts.is_high_priority_stream = True
        kw.setdefault("pg_options", opts)
    dist.init_process_group(backend, **kw)


def repair_shard(shard: torch.Tensor, out: Optional[torch.Tensor] = None, group=None, compute=None,
                 all_nonempty: bool = False, overlap: bool = True):
    """Repair this rank's shard of the logical buffer.

    Default (sm_100a kernel through the C ABI, every rank's shard non-empty):
    the interior tiles — everything except the shard's first and last
    8192-unit tiles, and the only part that needs no halo — start at once on
    the current stream, while a side stream all-gathers the edge units and
    then repairs the two edge tiles reading the neighbours' units straight
    from the gathered device tensor; the current stream joins the side
    stream. No host synchronisation inside the step. overlap=False runs
    gather -> whole-shard kernel serially. The halos are picked on the
    device from the gathered edges, skipping empty shards (select_halos);
    all_nonempty=True (the caller guarantees every rank's shard is
    non-empty) reads the neighbours' entries directly and saves those few
    tiny kernels.
    `compute(shard, out, left, right)` replaces the kernel (CPU tests; host
    halo values)."""
    rank = dist.get_rank(group)
    out = shard if out is None else out
    if compute is None:
        from . import _lib

        def pointers(edges):
            if all_nonempty:
                return edges, halo_pointers(edges, rank)
            sel = select_halos(edges, rank)
            return sel, (sel.data_ptr(), sel.data_ptr() + 4)

        if shard.numel() == 0:
            gather_edges(shard, group)  # every rank joins the collective
            return out
        main = torch.cuda.current_stream(shard.device)
        if not overlap:
            keep, (lp, rp) = pointers(gather_edges(shard, group))
            return _lib.to_well_formed_part(shard, out, _lib.PART_ALL, lp, rp)
        side = _side_stream(shard.device)
        side.wait_stream(main)
        _lib.to_well_formed_part(shard, out, _lib.PART_INTERIOR, stream=main)
        with torch.cuda.stream(side):
            keep, (lp, rp) = pointers(gather_edges(shard, group))
            _lib.to_well_formed_part(shard, out, _lib.PART_EDGES, lp, rp, stream=side)
        keep.record_stream(side)
        main.wait_stream(side)
        return out
    edges = gather_edges(shard, group)
    left, right = halos_from_edges(edges, rank)
    return compute(shard, out, left, right)


class PeerHalo:
    """Zero-collective halo access for one-process-per-GPU sharding.

    Every rank maps its nearest non-empty neighbours' shards once (CUDA IPC:
    peer memory over NVLink on a multi-GPU box, or the same GPU); a step is
    then ONE kernel launch per rank (u16m_to_well_formed_halo_ptr) whose two
    halo units are 2-byte loads straight from the neighbours' memory — no
    collective inside the step. A neighbour may be repairing its own shard in
    place at the same moment: the unit read is either its original value or
    its repaired value, and both give the same decision.
    The caller must make sure all ranks hold the same generation of the
    logical buffer (e.g. a barrier after refilling shards); this constructor
    ends with one.

    Uses torch's CUDA IPC plumbing (torch.multiprocessing.reductions) and
    all_gather_object, so it works with any backend (NCCL, gloo)."""

    def __init__(self, shard: torch.Tensor, group=None):
        from torch.multiprocessing.reductions import reduce_tensor

        self.rank = dist.get_rank(group)
        world = dist.get_world_size(group)
        self.shard = shard
        self._peers = []  # keep the mapped neighbour tensors alive
        self.left_ptr = self.right_ptr = 0
        if world == 1:
            dist.barrier(group=group)
            return
        rebuild, args = reduce_tensor(shard)
        metas = [None] * world
        dist.all_gather_object(metas, (args, int(shard.numel())), group=group)
        me = shard.device.index

        def open_on_my_device(a):
            # reduce_tensor's args[6] is the producer's device index, and torch
            # opens the IPC handle under that device, i.e. in the neighbour
            # GPU's context of this process, where this rank's kernels could
            # not dereference it. Opening it under THIS rank's device maps the
            # neighbour's memory into our own context (cudaIpcOpenMemHandle
            # with cudaIpcMemLazyEnablePeerAccess turns on NVLink peer access).
            a = list(a)
            owner = int(a[6])
            if owner != me and not torch.cuda.can_device_access_peer(me, owner):
                raise RuntimeError(f"cuda:{me} has no peer access to cuda:{owner}")
            a[6] = me
            return rebuild(*a)

        err = None
        try:
            for r in range(self.rank - 1, -1, -1):
                if metas[r][1] > 0:
                    t = open_on_my_device(metas[r][0])
                    self._peers.append(t)
                    self.left_ptr = t.data_ptr() + 2 * (t.numel() - 1)
                    break
            for r in range(self.rank + 1, world):
                if metas[r][1] > 0:
                    t = open_on_my_device(metas[r][0])
                    self._peers.append(t)
                    self.right_ptr = t.data_ptr()
                    break
        except Exception as e:  # noqa: BLE001 - reported on every rank below
            err = f"rank {self.rank}: {e!r}"
        # Agree before anyone proceeds: if one rank cannot map its neighbours,
        # every rank raises (callers fall back to the NCCL form together
        # instead of deadlocking in a barrier).
        errs = [None] * world
        dist.all_gather_object(errs, err, group=group)
        bad = [e for e in errs if e]
        if bad:
            self._peers.clear()
            self.left_ptr = self.right_ptr = 0
            raise RuntimeError("PeerHalo setup failed: " + "; ".join(bad))
        torch.cuda.synchronize(shard.device)
        dist.barrier(group=group)

    def repair(self, out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
        """Repair this rank's shard (in place when out is None)."""
        from . import _lib

        shard = self.shard
        out = shard if out is None else out
        if shard.numel() == 0:
            return out
        s = torch.cuda.current_stream(shard.device).cuda_stream if stream is None else stream
        _lib._check(_lib.raw().u16m_to_well_formed_halo_ptr(shard.data_ptr(), shard.numel(), out.data_ptr(),
                                                            self.left_ptr or None, self.right_ptr or None, s))
        return out
