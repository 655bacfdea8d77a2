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


L = _lib.raw()
empties = torch.zeros((1 << 20) + 2, dtype=torch.int64, device="cuda")
empties[-1] = n  # 2^20 empty strings at 0, then one string over the whole buffer
odd = torch.empty(n + 8, dtype=torch.int16, device="cuda")[3:3 + n]  # out phase != in phase


def nolen(offs):  # the length-less entry (no buffer length: TMA producer-walk kernel)
    s = torch.cuda.current_stream().cuda_stream
    assert L.u16m_to_well_formed_batched(d.data_ptr(), offs.data_ptr(), offs.numel() - 1, out.data_ptr(), s) == 0


for name, fn in [
    ("c3 batch", lambda: _lib.to_well_formed_batched(d, o, out=out)),
    ("one string", lambda: _lib.to_well_formed_batched(d, one, out=out)),
    ("empties+one", lambda: _lib.to_well_formed_batched(d, empties, out=out)),
    ("c3 other-phase out", lambda: _lib.to_well_formed_batched(d, o, out=odd)),
    ("c3 no-length", lambda: nolen(o)),
    ("one no-length", lambda: nolen(one)),
    ("empties no-len", lambda: nolen(empties)),
    ("plain copy", lambda: _lib.to_well_formed(d, out=out)),
]:
    us = timed(fn)
    print(f"{os.environ.get('TAG', '')} {name:20s} {us:7.1f} us  {2 * n / us / 1e3:7.1f} GB/s in", flush=True)
