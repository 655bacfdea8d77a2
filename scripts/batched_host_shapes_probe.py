"""Batched host form through pinned buffers for several batch shapes of the
same ~1 GB: where does the gap to the plain host path (same bytes) come from?"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_06349_b200 import _lib  # noqa: E402

L = _lib.raw()
n = 1 << 29
hin = torch.empty(n, dtype=torch.int16, pin_memory=True)
hin.copy_(_lib.gen_config(0, n, seed=1))
hout = torch.empty(n, dtype=torch.int16, pin_memory=True)


def rate(fn):
    fn()
    ts = []
    for _ in range(4):
        t = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t)
    return 2 * n / min(ts) / 1e9


print("plain host:", round(rate(lambda: _lib._check(L.u16m_to_well_formed_host(hin.data_ptr(), n, hout.data_ptr()))), 1))
for S in (1 << 20, 1 << 16, 1 << 10, 64, 16):
    offs = torch.from_numpy(np.linspace(0, n, S + 1).astype(np.int64)).pin_memory()
    r = rate(lambda: _lib._check(L.u16m_to_well_formed_batched_host(hin.data_ptr(), n, offs.data_ptr(), S,
                                                                    hout.data_ptr())))
    print(f"batched host, {S:8d} equal strings: {r:5.1f} GB/s", flush=True)
