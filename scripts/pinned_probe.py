"""Host-buffer e2e vs how the pinned host memory was allocated.

The driver's e2e (u16m_to_well_formed_host over pinned buffers, full-duplex
PCIe) varied 44-48 GB/s between back-to-back runs on one box. Hypothesis:
DMA to pinned memory backed by scattered 4 KiB pages pays IOMMU / page-walk
costs that 2 MiB pages avoid. This times the real host path over 8 GiB in +
8 GiB out for: torch pin_memory (cudaHostAlloc), anonymous mmap + cudaHostRegister
(4 KiB pages), mmap + MADV_HUGEPAGE (THP) + register, and MAP_HUGETLB + register."""
import ctypes
import mmap
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_06349_b200 import _lib  # noqa: E402

N = int(os.environ.get("PROBE_UNITS", str(1 << 32)))
NB = 2 * N


def sh(path):
    try:
        return open(path).read().strip()
    except OSError as e:
        return f"<{e.strerror}>"


print("THP enabled:", sh("/sys/kernel/mm/transparent_hugepage/enabled"))
print("THP defrag:", sh("/sys/kernel/mm/transparent_hugepage/defrag"))
print("nr_hugepages:", sh("/proc/sys/vm/nr_hugepages"))
print("iommu groups:", len(os.listdir("/sys/kernel/iommu_groups")) if os.path.isdir("/sys/kernel/iommu_groups") else "none")
print("cmdline:", sh("/proc/cmdline")[:300])
for l in open("/proc/meminfo"):
    if l.startswith(("MemFree", "AnonHugePages", "HugePages_Total", "Hugepagesize")):
        print(" ", l.strip())

cudart = torch.cuda.cudart()
keep = []


def alloc(kind):
    if kind == "torch_pin":
        t = torch.empty(N, dtype=torch.int16, pin_memory=True)
        return t, t.data_ptr()
    flags = mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS
    if kind == "hugetlb":
        flags |= 0x40000  # MAP_HUGETLB (2 MiB default size)
    m = mmap.mmap(-1, NB, flags=flags, prot=mmap.PROT_READ | mmap.PROT_WRITE)
    if kind == "thp":
        m.madvise(mmap.MADV_HUGEPAGE)
    a = np.frombuffer(m, dtype=np.int16)
    a[:] = 0  # fault every page in
    addr = a.ctypes.data
    r = cudart.cudaHostRegister(addr, NB, 0)
    if int(r) != 0:
        raise RuntimeError(f"cudaHostRegister failed: {r}")
    keep.append((m, addr))
    return torch.from_numpy(a), addr


def anon_huge():
    for l in open("/proc/meminfo"):
        if l.startswith("AnonHugePages"):
            return l.split(":")[1].strip()


L = _lib.raw()
data = _lib.gen_config(4, N, seed=4, shard_len=N)
res = {}
for kind in ("torch_pin", "anon4k", "thp", "hugetlb", "torch_pin"):
    try:
        t0 = time.perf_counter()
        hin, pin = alloc(kind)
        hout, pout = alloc(kind)
        ta = time.perf_counter() - t0
    except Exception as e:  # noqa: BLE001
        print(f"{kind}: allocation failed: {e}")
        continue
    hin.copy_(data)
    rates = []
    for i in range(6):
        t = time.perf_counter()
        _lib._check(L.u16m_to_well_formed_host(pin, N, pout))
        rates.append(NB / (time.perf_counter() - t) / 1e9)
    print(f"{kind:10s} alloc+fault {ta:5.1f} s  AnonHugePages {anon_huge():>12s}  e2e copy GB/s: "
          + " ".join(f"{r:5.1f}" for r in rates[1:]), flush=True)
    del hin, hout
    torch.cuda.synchronize()
    for m, addr in keep:
        cudart.cudaHostUnregister(addr)
    keep.clear()  # the mmaps are unmapped when the last numpy view is collected
