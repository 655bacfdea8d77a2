"""Host-path throughput with PAGEABLE host memory (what a C++ caller passing
std::vector spans gets) versus pinned, 512 MiB, config 1 content."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_06349_b200 import _lib  # noqa: E402

L = _lib.raw()
n = 1 << 28
src = _lib.gen_config(1, n, seed=1).cpu().numpy()
for kind in ("pageable", "pinned"):
    if kind == "pageable":
        a = np.empty(n, np.int16)
        o = np.empty(n, np.int16)
        pa, po = a.ctypes.data, o.ctypes.data
    else:
        ta = torch.empty(n, dtype=torch.int16).pin_memory()
        to = torch.empty(n, dtype=torch.int16).pin_memory()
        a, o = ta.numpy(), to.numpy()
        pa, po = ta.data_ptr(), to.data_ptr()
    for mode in ("copy", "inplace"):
        best = 0.0
        for _ in range(4):
            a[:] = src
            t = time.perf_counter()
            assert L.u16m_to_well_formed_host(pa, n, pa if mode == "inplace" else po) == 0
            best = max(best, 2 * n / (time.perf_counter() - t) / 1e9)
        print(f"{kind:8s} {mode:7s} {best:5.1f} GB/s", flush=True)
