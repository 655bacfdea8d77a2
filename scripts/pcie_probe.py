"""PCIe H2D / D2H / duplex bandwidth probe (pinned memory), for the e2e design."""
import time

import torch

n = 512 << 20
h = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for name, fn in [
    ("h2d", lambda: d.copy_(h, non_blocking=True)),
    ("d2h", lambda: h.copy_(d, non_blocking=True)),
]:
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    print(name, 5 * n / (time.perf_counter() - t) / 1e9, "GB/s")
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5):
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
print("duplex each-way", 5 * n / (time.perf_counter() - t) / 1e9, "GB/s")
# chunked duplex like the pipeline
for chunk_mb in (4, 16, 64):
    c = chunk_mb << 20
    streams = [torch.cuda.Stream() for _ in range(4)]
    torch.cuda.synchronize()
    t = time.perf_counter()
    for rep in range(3):
        for i, off in enumerate(range(0, n, c)):
            with torch.cuda.stream(streams[i % 4]):
                d[off:off + c].copy_(h[off:off + c], non_blocking=True)
                h2[off:off + c].copy_(d[off:off + c], non_blocking=True)
    torch.cuda.synchronize()
    print(f"pipeline chunk {chunk_mb} MiB: input rate", 3 * n / (time.perf_counter() - t) / 1e9, "GB/s")
