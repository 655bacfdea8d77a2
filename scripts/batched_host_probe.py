"""The host-memory batched entry (u16m_to_well_formed_batched_host) on a
2 MB batch of 10 000 strings: C-call time, warm, pageable vs pinned."""
import ctypes
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_06349_b200 import _lib  # noqa: E402

L = _lib.raw()
for nstr, slen in ((10_000, 100), (1000, 100), (100_000, 100), (10_000, 4096)):
    n = nstr * slen
    x = np.random.default_rng(0).integers(0, 65536, n).astype(np.uint16)
    offs = np.arange(0, n + 1, slen, dtype=np.int64)
    for kind in ("pageable", "pinned"):
        if kind == "pinned":
            t = torch.from_numpy(x.view(np.int16).copy()).pin_memory()
            ptr = t.data_ptr()
        else:
            buf = x.copy()
            ptr = buf.ctypes.data
        ts = []
        for i in range(6):
            t0 = time.perf_counter()
            st = L.u16m_to_well_formed_batched_host(ctypes.c_void_p(ptr), n, ctypes.c_void_p(offs.ctypes.data), nstr,
                                                    ctypes.c_void_p(ptr))
            ts.append(time.perf_counter() - t0)
            assert st == 0
        print(f"{nstr:7d} strings x {slen:5d} units ({2 * n / 1e6:6.1f} MB) {kind:8s}: "
              f"{min(ts[1:]) * 1e3:7.3f} ms best, {np.median(ts[1:]) * 1e3:7.3f} ms median", flush=True)
