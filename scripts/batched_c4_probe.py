"""Batched form at config-4 scale: 2^23 strings (config-3 length distribution, ~4.3e9 units, 8.6 GB)
through the length-aware and the length-less entry, against the plain copy of the same bytes."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_06349_b200 import _lib  # noqa: E402

L = _lib.raw()
data, offsets = _lib.gen_c3(1 << 23, seed=3)
n = data.numel()
out = torch.empty_like(data)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream().cuda_stream
S = offsets.numel() - 1


def run(name, fn):
    tot = 0.0
    for i in range(7):
        _lib.l2_flush(flush)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        assert fn() == 0
        b.record()
        torch.cuda.synchronize()
        if i >= 2:
            tot += a.elapsed_time(b)
    ms = tot / 5
    print(f"{name}: {ms * 1e3:.1f} us, {2 * n / ms / 1e6:.0f} GB/s input ({n} units, {S} strings)", flush=True)


run("plain copy", lambda: L.u16m_to_well_formed(data.data_ptr(), n, out.data_ptr(), s))
run("batched_n copy", lambda: L.u16m_to_well_formed_batched_n(data.data_ptr(), n, offsets.data_ptr(), S, out.data_ptr(), s))
run("batched (length-less) copy", lambda: L.u16m_to_well_formed_batched(data.data_ptr(), offsets.data_ptr(), S, out.data_ptr(), s))
run("batched_n in place", lambda: L.u16m_to_well_formed_batched_n(out.data_ptr(), n, offsets.data_ptr(), S, out.data_ptr(), s))
