"""Timeline of the host pipeline model: per-chunk H2D / kernel / D2H with
CUDA events, to see where a 512 MiB in-place host job loses time against the
~48-50 GB/s full-duplex PCIe rate. Pure torch copies + the library's repair
kernel on device chunks (same structure as u16m_capi.cu host_pipeline)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_06349_b200 import _lib  # noqa: E402

L = _lib.raw()
n = 1 << 28
x = _lib.gen_config(1, n, seed=1)
h = torch.empty(n, dtype=torch.int16, pin_memory=True)
h.copy_(x)
src = h.clone().pin_memory()


def pipeline(chunk_mib, ring=8, kernel=True, restore=True):
    cu = chunk_mib << 19
    nchunks = (n + cu - 1) // cu
    bufs = [torch.empty(cu, dtype=torch.int16, device="cuda") for _ in range(ring)]
    sh, sc, sd = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    loaded = [torch.cuda.Event() for _ in range(nchunks)]
    done = [torch.cuda.Event() for _ in range(nchunks)]
    drained = [torch.cuda.Event(enable_timing=True) for _ in range(nchunks)]
    t0 = torch.cuda.Event(enable_timing=True)
    if restore:
        h.copy_(src)
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    t0.record(sh)
    for c in range(nchunks):
        k = c % ring
        a, b = c * cu, min(n, (c + 1) * cu)
        with torch.cuda.stream(sh):
            if c >= ring:
                sh.wait_event(drained[c - ring])
            bufs[k][: b - a].copy_(h[a:b], non_blocking=True)
            loaded[c].record(sh)
        with torch.cuda.stream(sc):
            sc.wait_event(loaded[c])
            if kernel:
                L.u16m_to_well_formed_halo(bufs[k].data_ptr(), b - a, bufs[k].data_ptr(), -1, -1,
                                           ctypes_stream(sc))
            done[c].record(sc)
        with torch.cuda.stream(sd):
            sd.wait_event(done[c])
            h[a:b].copy_(bufs[k][: b - a], non_blocking=True)
            drained[c].record(sd)
    torch.cuda.synchronize()
    wall = time.perf_counter() - w0
    ev = t0.elapsed_time(drained[-1]) / 1e3
    return 2 * n / wall / 1e9, 2 * n / ev / 1e9


def ctypes_stream(s):
    return s.cuda_stream


dsrc = src.cuda()
for rep in range(3):
    for how in ("none", "cpu", "cpu+sleep", "dma"):
        if how == "cpu" or how == "cpu+sleep":
            h.copy_(src)
        elif how == "dma":
            h.copy_(dsrc)
        if how == "cpu+sleep":
            time.sleep(0.2)
        torch.cuda.synchronize()
        t = time.perf_counter()
        L.u16m_to_well_formed_host(h.data_ptr(), n, h.data_ptr())
        print(f"library host path in place, restore={how:10s}: {2 * n / (time.perf_counter() - t) / 1e9:5.1f} GB/s",
              flush=True)
