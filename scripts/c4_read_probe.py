"""Config 4 (2^32 units): the read-only stream (u16m_count_unpaired, the same
kernel body with no stores) vs in-place repair vs copy, L2 flushed before
each call — how much of the in-place time is the read stream itself."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_06349_b200 import _lib  # noqa: E402

n = 1 << 32
x = _lib.gen_config(4, n, seed=4, shard_len=n)
w = torch.empty_like(x)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
L = _lib.raw()
s = torch.cuda.current_stream().cuda_stream


def timed(fn, prep=None, reps=8):
    ts = []
    for _ in range(reps + 2):
        if prep:
            prep()
        _lib.l2_flush(flush)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ts = sorted(ts[2:])
    return ts[len(ts) // 2] * 1e3


for _ in range(2):
    t_count = timed(lambda: L.u16m_count_unpaired(x.data_ptr(), n, cnt.data_ptr(), s))
    t_ip = timed(lambda: L.u16m_to_well_formed_in_place(w.data_ptr(), n, s), prep=lambda: w.copy_(x))
    t_cp = timed(lambda: L.u16m_to_well_formed(x.data_ptr(), n, w.data_ptr(), s))
    t_memcpy = timed(lambda: w.copy_(x))
    print(f"read-only count {t_count:8.1f} us ({2 * n / t_count / 1e3:6.1f} GB/s read) | in place {t_ip:8.1f} us | "
          f"copy {t_cp:8.1f} us | torch copy_ {t_memcpy:8.1f} us ({4 * n / t_memcpy / 1e3:6.1f} GB/s r+w)", flush=True)
