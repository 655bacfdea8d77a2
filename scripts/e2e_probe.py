"""Probe the host-memory e2e path (u16m_to_well_formed_host) on this box:
zero-copy (pinned mapped buffers) vs the staged pipeline, in place and copy."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_06349_b200 import _lib  # noqa: E402

L = _lib.raw()
n = 1 << 28
cfg = int(os.environ.get("CFG", "1"))
x = _lib.gen_config(cfg, n, seed=cfg)
h = torch.empty(n, dtype=torch.int16, pin_memory=True)
h.copy_(x)
src = h.clone().pin_memory()
out = torch.empty_like(h).pin_memory()
ref = _lib.to_well_formed(x).cpu()
for mode in os.environ.get("MODES", "inplace,copy").split(","):
    times = []
    for i in range(8):
        if mode == "inplace":
            h.copy_(src)
        t = time.perf_counter()
        dst = h if mode == "inplace" else out
        st = L.u16m_to_well_formed_host(h.data_ptr(), n, dst.data_ptr())
        times.append(time.perf_counter() - t)
        assert st == 0
        assert torch.equal(dst, ref), "mismatch"
    best = min(times[2:])
    print(f"cfg{cfg}", mode,
          f"{2 * n / best / 1e9:.1f} GB/s best, {2 * n * 6 / sum(times[2:]) / 1e9:.1f} mean", flush=True)
