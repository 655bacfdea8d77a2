"""Read-only validation kernel (u16m_count_unpaired) on config 1 and config 4,
L2 flushed before each call."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_06349_b200 import _lib  # noqa: E402

flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
L = _lib.raw()
s = torch.cuda.current_stream().cuda_stream


def timed(fn, reps=10):
    ts = []
    for _ in range(reps + 2):
        _lib.l2_flush(flush)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ts = sorted(ts[2:])
    return ts[len(ts) // 2] * 1e3


for cfg, n in ((1, 1 << 28), (4, 1 << 32)):
    x = _lib.gen_config(cfg, n, seed=cfg, shard_len=n if cfg == 4 else 0)
    us = timed(lambda: L.u16m_count_unpaired(x.data_ptr(), n, cnt.data_ptr(), s))
    print(f"count c{cfg}: {us:8.1f} us  {2 * n / us / 1e3:7.1f} GB/s read",
          flush=True)
    del x
