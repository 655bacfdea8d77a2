"""Validation entry points at config-4 size (2^32 units = 8 GiB): count vs the
offsets scan with small limits, on the config-4 input and on its repaired
(well-formed) form. L2 flushed between reps, mean of 5."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_06349_b200 import _lib  # noqa: E402

L = _lib.raw()
n = 1 << 32
x = _lib.gen_config(4, n, seed=4, shard_len=n)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
offs = torch.zeros(1 << 20, dtype=torch.int64, device="cuda")
s = torch.cuda.current_stream().cuda_stream


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
    print(f"{name}: {ms * 1e3:.1f} us, {2 * n / ms / 1e6:.0f} GB/s, count={int(cnt.item())}", flush=True)


for label in ("config-4 input", "well-formed"):
    run(f"[{label}] count_unpaired", lambda: L.u16m_count_unpaired(x.data_ptr(), n, cnt.data_ptr(), s))
    run(f"[{label}] unpaired_offsets(limit=1)",
        lambda: L.u16m_unpaired_offsets(x.data_ptr(), n, 1, offs.data_ptr(), cnt.data_ptr(), s))
    run(f"[{label}] unpaired_offsets(limit=10)",
        lambda: L.u16m_unpaired_offsets(x.data_ptr(), n, 10, offs.data_ptr(), cnt.data_ptr(), s))
    run(f"[{label}] unpaired_offsets(limit=2^20)",
        lambda: L.u16m_unpaired_offsets(x.data_ptr(), n, 1 << 20, offs.data_ptr(), cnt.data_ptr(), s))
    _lib.to_well_formed_(x)
