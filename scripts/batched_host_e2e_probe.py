import ctypes, time, sys, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np
from paper_2601_06349_b200 import _lib
L = _lib.raw()
data, offsets = _lib.gen_c3(1 << 20, seed=3)
n = data.numel(); S = offsets.numel() - 1
hin = torch.empty(n, dtype=torch.int16, pin_memory=True); hin.copy_(data)
hout = torch.empty(n, dtype=torch.int16, pin_memory=True)
for kind in ("pageable", "pinned"):
    hoff = offsets.cpu()
    if kind == "pinned": hoff = hoff.pin_memory()
    ts = []
    for i in range(6):
        t = time.perf_counter()
        _lib._check(L.u16m_to_well_formed_batched_host(hin.data_ptr(), n, hoff.data_ptr(), S, hout.data_ptr()))
        ts.append(time.perf_counter() - t)
    print(kind, "offsets:", [round(2 * n / x / 1e9, 1) for x in ts[1:]])
t = time.perf_counter(); _lib._check(L.u16m_to_well_formed_host(hin.data_ptr(), n, hout.data_ptr())); dt = time.perf_counter() - t
t = time.perf_counter(); _lib._check(L.u16m_to_well_formed_host(hin.data_ptr(), n, hout.data_ptr())); dt = time.perf_counter() - t
print("plain host same bytes:", round(2 * n / dt / 1e9, 1))
