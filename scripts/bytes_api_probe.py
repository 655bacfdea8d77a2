"""Where the time goes in fix_utf16le on 512 MiB of Python bytes."""
import ctypes
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_06349_b200 import _lib  # noqa: E402

L = _lib.raw()
n = 1 << 28
bad = _lib.gen_config(1, n, seed=1).cpu().numpy().tobytes()
for rep in range(2):
    t0 = time.perf_counter()
    out = bytearray(2 * n)
    t1 = time.perf_counter()
    src = np.frombuffer(memoryview(bad), dtype=np.uint8)
    ob = (ctypes.c_char * (2 * n)).from_buffer(out)
    t2 = time.perf_counter()
    assert L.u16m_to_well_formed_host(src.ctypes.data, n, ctypes.addressof(ob)) == 0
    t3 = time.perf_counter()
    b = bytes(out)
    t4 = time.perf_counter()
    o2 = np.empty(2 * n, np.uint8)
    t5 = time.perf_counter()
    assert L.u16m_to_well_formed_host(src.ctypes.data, n, o2.ctypes.data) == 0
    t6 = time.perf_counter()
    assert L.u16m_to_well_formed_host(src.ctypes.data, n, o2.ctypes.data) == 0
    t7 = time.perf_counter()
    print(f"bytearray {1e3*(t1-t0):.1f} ms | setup {1e3*(t2-t1):.1f} | C call {1e3*(t3-t2):.1f} | bytes() {1e3*(t4-t3):.1f}"
          f" | np.empty {1e3*(t5-t4):.1f} | C call into fresh np {1e3*(t6-t5):.1f} | again {1e3*(t7-t6):.1f}", flush=True)
