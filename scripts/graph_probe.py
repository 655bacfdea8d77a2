"""Does a CUDA-graph launch shorten the event-timed step of a small job
(config 0, 32 MiB copy) versus a direct launch? L2 flushed before every rep."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_06349_b200 as P  # noqa: E402
from paper_2601_06349_b200 import _lib  # noqa: E402

n = 1 << 24
x = _lib.gen_config(0, n, seed=0)
out = torch.empty_like(x)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    P.to_well_formed(x, out=out)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        P.to_well_formed(x, out=out)
    torch.cuda.synchronize()


def timed(fn, reps=30):
    ts = []
    with torch.cuda.stream(s):
        for _ in range(reps):
            _lib.l2_flush(flush)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            fn()
            b.record(s)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


for _ in range(3):
    d = timed(lambda: P.to_well_formed(x, out=out))
    r = timed(lambda: g.replay())
    print(f"C0 direct {d:.1f} us ({2 * n / d / 1e3:.0f} GB/s)  graph {r:.1f} us ({2 * n / r / 1e3:.0f} GB/s)")
