"""Codec-fused repair (u16m_fix_utf16_bytes) on 2^28 units, L2 flushed before
each call: same-phase output vs an output at another 16-byte phase, LE/BE,
with and without the replacement count."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_06349_b200 import _lib  # noqa: E402

n = 1 << 28
x = _lib.gen_config(1, n, seed=1)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
base = torch.empty(n + 16, dtype=torch.int16, device="cuda")


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


cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
L = _lib.raw()
s = torch.cuda.current_stream().cuda_stream
for big in (0, 1):
    for po in (0, 3):
        out = base[po:po + n]
        for c in (None, cnt):
            us = timed(lambda: L.u16m_fix_utf16_bytes(x.data_ptr(), n, out.data_ptr(), big,
                                                      c.data_ptr() if c is not None else None, s))
            print(f"{'BE' if big else 'LE'} out phase {po} count={c is not None}: {us:7.1f} us  {2 * n / us / 1e3:7.1f} GB/s in")
