"""Latency of small host-memory calls through the Python bytes API (a GPU
round trip per call: H2D, kernel, D2H, sync)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_06349_b200 as P  # noqa: E402

for n in (8, 256, 4096, 65536):
    s = ("ab\ud800" * (n // 3 + 1))[:n]
    P.fix_str(s)
    t = time.perf_counter()
    for _ in range(200):
        P.fix_str(s)
    dt = (time.perf_counter() - t) / 200
    b = s.encode("utf-16-le", "surrogatepass")
    t = time.perf_counter()
    for _ in range(200):
        P.is_well_formed_utf16le(b)
    dv = (time.perf_counter() - t) / 200
    print(f"{n:6d} units: fix_str {dt * 1e6:7.1f} us/call   is_well_formed {dv * 1e6:7.1f} us/call", flush=True)
import ctypes
import numpy as np
from paper_2601_06349_b200 import _lib
L = _lib.raw()
for n in (4096, 65536):
    s = ("ab\ud800" * (n // 3 + 1))[:n]
    b = s.encode("utf-16-le", "surrogatepass")
    def t(f, k=100):
        f(); t0 = time.perf_counter()
        for _ in range(k): f()
        return (time.perf_counter() - t0) / k * 1e6
    a = np.frombuffer(b, np.uint8); o = np.empty_like(a)
    print(n, "encode", round(t(lambda: s.encode("utf-16-le", "surrogatepass")), 1),
          "fix_utf16le", round(t(lambda: P.fix_utf16le(b)), 1),
          "C host call", round(t(lambda: L.u16m_to_well_formed_host(ctypes.c_void_p(a.ctypes.data), ctypes.c_size_t(n), ctypes.c_void_p(o.ctypes.data))), 1),
          "decode", round(t(lambda: P.fix_utf16le(b).decode("utf-16-le")), 1), flush=True)
texts = [("ab\ud800cd" * 20)] * 10000
P.fix_str_batch(texts)  # first call allocates the pinned staging buffers
t0 = time.perf_counter(); r1 = [P.fix_str(x) for x in texts[:500]]; t1 = time.perf_counter()
for _ in range(5):
    r2 = P.fix_str_batch(texts)
t2 = time.perf_counter()
print(f"10 000 strings of 100 units: one call each {(t1 - t0) / 500 * 1e6:.1f} us/string; "
      f"fix_str_batch {(t2 - t1) / 5 / 10000 * 1e6:.2f} us/string (warm)", flush=True)
