"""Is the e2e (host-buffer) rate disturbed by memory another process just
freed? Times u16m_to_well_formed_host over 8 GiB pinned in/out repeatedly for
~70 s; at t=15 s a helper process touches 48 GiB of ordinary memory and exits
at t=25 s (its pages are then returned to the VM host in the background:
free page reporting is on in this guest, page_reporting_order=11)."""
import os
import subprocess
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_06349_b200 import _lib  # noqa: E402

N = 1 << 32
L = _lib.raw()
data = _lib.gen_config(4, N, seed=4, shard_len=N)
hin = torch.empty(N, dtype=torch.int16, pin_memory=True)
hout = torch.empty(N, dtype=torch.int16, pin_memory=True)
hin.copy_(data)
helper = ("import numpy as np, time; a = np.ones(48 << 30, dtype=np.uint8); time.sleep(10); "
          "del a; print('helper freed', flush=True)")
t_start = time.perf_counter()
proc = None
while time.perf_counter() - t_start < 70:
    now = time.perf_counter() - t_start
    if proc is None and now > 15:
        proc = subprocess.Popen([sys.executable, "-c", helper])
    t = time.perf_counter()
    _lib._check(L.u16m_to_well_formed_host(hin.data_ptr(), N, hout.data_ptr()))
    r = 2 * N / (time.perf_counter() - t) / 1e9
    free = [l for l in open("/proc/meminfo") if l.startswith("MemFree")][0].split()[1]
    print(f"t={now:5.1f}s e2e {r:5.1f} GB/s  MemFree {int(free) >> 20} GiB", flush=True)
proc.wait()
