"""Pageable in-place host jobs: error-dense input (config 1: every chunk has
rewrites, every chunk is copied back) against clean text and text with a few
dirty chunks (clean chunks are not copied back). 2 GiB, best of 4."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_06349_b200 import _lib  # noqa: E402

L = _lib.raw()
n = 1 << 30
dense = _lib.gen_config(1, n, seed=1).cpu().numpy()
clean = _lib.gen_config(0, n, seed=0).cpu().numpy()
clean = np.frombuffer(_lib.fix_utf16le(clean.tobytes()), np.int16).copy()  # well-formed config-0 text
few = clean.copy()
few[:: n // 7] = np.int16(-10240)  # 0xD800: a lone high surrogate in 7 places
import torch  # noqa: E402

a = np.empty(n, np.int16)
ta = torch.empty(n, dtype=torch.int16).pin_memory()
pa = ta.numpy()
for name, src in (("error-dense (config 1)", dense), ("clean text", clean), ("7 lone surrogates", few)):
    best = 0.0
    for _ in range(5):
        pa[:] = src
        t = time.perf_counter()
        assert L.u16m_to_well_formed_host(ta.data_ptr(), n, ta.data_ptr()) == 0
        best = max(best, 2 * n / (time.perf_counter() - t) / 1e9)
    assert (pa == np.frombuffer(_lib.fix_utf16le(src.tobytes()), np.int16)).all()
    print(f"pinned in place, {name}: {best:5.1f} GB/s", flush=True)
for name, src in (("error-dense (config 1)", dense), ("clean text", clean), ("7 lone surrogates", few)):
    best = 0.0
    for _ in range(4):
        a[:] = src
        t = time.perf_counter()
        assert L.u16m_to_well_formed_host(a.ctypes.data, n, a.ctypes.data) == 0
        best = max(best, 2 * n / (time.perf_counter() - t) / 1e9)
    print(f"pageable in place, {name}: {best:5.1f} GB/s", flush=True)
