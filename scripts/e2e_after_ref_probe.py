"""When, after a large process exits, is the e2e (host-buffer) rate disturbed?
Run right after `bench.py --impl reference` (the driver's order): pins 8 GiB
in / 8 GiB out and times u16m_to_well_formed_host back to back for ~100 s,
printing the time since this process started and MemFree."""
import os
import sys
import time

T0 = time.perf_counter()
import torch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_06349_b200 import _lib  # noqa: E402

N = 1 << 32
SECS = float(sys.argv[1]) if len(sys.argv) > 1 else 100.0
L = _lib.raw()
hin = torch.empty(N, dtype=torch.int16, pin_memory=True)
hout = torch.empty(N, dtype=torch.int16, pin_memory=True)
print(f"pinned at t={time.perf_counter() - T0:.1f}s", flush=True)
data = _lib.gen_config(4, N, seed=4, shard_len=N)
hin.copy_(data)
torch.cuda.synchronize()
while time.perf_counter() - T0 < SECS:
    now = time.perf_counter() - T0
    t = time.perf_counter()
    _lib._check(L.u16m_to_well_formed_host(hin.data_ptr(), N, hout.data_ptr()))
    r = 2 * N / (time.perf_counter() - t) / 1e9
    free = [l for l in open("/proc/meminfo") if l.startswith("MemFree")][0].split()[1]
    print(f"t={now:5.1f}s e2e {r:5.1f} GB/s  MemFree {int(free) >> 20} GiB", flush=True)
