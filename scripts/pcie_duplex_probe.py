"""PCIe duplex probe: does spreading H2D / D2H over several streams (copy
engines) raise the full-duplex rate above one stream per direction?"""
import time

import torch

n = 512 << 20
h = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")


def run(k_h2d, k_d2h, reps=4, same_host=False):
    sh = [torch.cuda.Stream() for _ in range(k_h2d)]
    sd = [torch.cuda.Stream() for _ in range(k_d2h)]
    dst = h if same_host else h2
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        for i, s in enumerate(sh):
            a, b = i * n // k_h2d, (i + 1) * n // k_h2d
            with torch.cuda.stream(s):
                d[a:b].copy_(h[a:b], non_blocking=True)
        for i, s in enumerate(sd):
            a, b = i * n // k_d2h, (i + 1) * n // k_d2h
            with torch.cuda.stream(s):
                dst[a:b].copy_(d2[a:b], non_blocking=True)
    torch.cuda.synchronize()
    return reps * n / (time.perf_counter() - t) / 1e9


for _ in range(2):
    for kh, kd in [(1, 0), (2, 0), (4, 0), (0, 1), (0, 2), (1, 1), (2, 2), (4, 4), (2, 1), (1, 2)]:
        print(f"h2d streams {kh} d2h streams {kd}: {run(kh, kd):6.1f} GB/s each way", flush=True)
    print(f"1+1 same host buffer: {run(1, 1, same_host=True):6.1f} GB/s each way", flush=True)
print("async engines:", torch.cuda.get_device_properties(0))
