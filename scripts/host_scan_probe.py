"""Host-memory validation (u16m_unpaired_offsets_host via the Python bytes
API): a 512 MiB well-formed buffer is scanned to the end; config-1 data with
limit 10 stops in the first chunk. Input GB/s."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_06349_b200 as P  # noqa: E402
from paper_2601_06349_b200 import _lib  # noqa: E402

n = 1 << 28
x = _lib.gen_config(1, n, seed=1)
bad = x.cpu().numpy().tobytes()
good = _lib.to_well_formed(x).cpu().numpy().tobytes()
for name, fn in (("is_well_formed(clean 512 MiB)", lambda: P.is_well_formed_utf16le(good)),
                 ("unpaired_surrogate_offsets(C1, limit=10)", lambda: P.unpaired_surrogate_offsets(bad, 10)),
                 ("unpaired_surrogate_offsets(clean, limit=10)", lambda: P.unpaired_surrogate_offsets(good, 10))):
    best = 1e9
    for _ in range(4):
        t = time.perf_counter()
        fn()
        best = min(best, time.perf_counter() - t)
    print(f"{name:45s} {best * 1e3:8.2f} ms  {2 * n / best / 1e9:6.1f} GB/s", flush=True)
for name, fn in (("fix_utf16le(C1 512 MiB bytes)", lambda: P.fix_utf16le(bad)),
                 ("fix_utf16_bytes(C1, be)", lambda: P.fix_utf16_bytes(bad, "be"))):
    best = 1e9
    for _ in range(3):
        t = time.perf_counter()
        fn()
        best = min(best, time.perf_counter() - t)
    print(f"{name:45s} {best * 1e3:8.2f} ms  {2 * n / best / 1e9:6.1f} GB/s", flush=True)
