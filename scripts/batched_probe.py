"""Decompose the batched (config 3) step on one GPU: the real CSR batch, the
same buffer as ONE string (no starts: tile machinery only), and the plain
copy kernel over the same bytes. Each timed call follows an L2 flush."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_06349_b200 import _lib  # noqa: E402

d, o = _lib.gen_c3(1 << 20)
n = d.numel()
one = torch.tensor([0, n], dtype=torch.int64, device="cuda")
out = torch.empty_like(d)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def timed(fn, reps=20):
    ts = []
    for _ in range(reps + 3):
        _lib.l2_flush(flush)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ts = sorted(ts[3:])
    return ts[len(ts) // 2] * 1e3


for name, fn in [
    ("c3 batch", lambda: _lib.to_well_formed_batched(d, o, out=out)),
    ("one string", lambda: _lib.to_well_formed_batched(d, one, out=out)),
    ("plain copy", lambda: _lib.to_well_formed(d, out=out)),
]:
    us = timed(fn)
    print(f"{os.environ.get('TAG', '')} {name:12s} {us:7.1f} us  {2 * n / us / 1e3:7.1f} GB/s in", flush=True)
