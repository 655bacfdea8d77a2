"""Cost of pinning pageable host memory on the fly (cudaHostRegister /
cudaHostUnregister) per chunk size, and DMA rates from freshly registered
pages — would registering the caller's pageable buffer chunk by chunk beat
the bounce-buffer copies (28 GB/s) of the pageable host path?"""
import time

import numpy as np
import torch

cudart = torch.cuda.cudart()
total = 1 << 30
a = np.ones(total, dtype=np.uint8)
d = torch.empty(total, dtype=torch.uint8, device="cuda")
for chunk_mib in (4, 16, 32, 64, 256):
    cb = chunk_mib << 20
    t_reg = t_unreg = 0.0
    t0 = time.perf_counter()
    for off in range(0, total, cb):
        p = a.ctypes.data + off
        t = time.perf_counter()
        r = cudart.cudaHostRegister(p, cb, 0)
        t_reg += time.perf_counter() - t
        assert int(r) == 0, r
        src = torch.from_numpy(a[off:off + cb])
        d[off:off + cb].copy_(src, non_blocking=True)
        torch.cuda.synchronize()
        t = time.perf_counter()
        cudart.cudaHostUnregister(p)
        t_unreg += time.perf_counter() - t
    wall = time.perf_counter() - t0
    print(f"chunk {chunk_mib:4d} MiB: register {total / t_reg / 1e9:6.1f} GB/s, unregister {total / t_unreg / 1e9:7.1f} GB/s, "
          f"serial register+H2D+unregister {total / wall / 1e9:5.1f} GB/s", flush=True)
