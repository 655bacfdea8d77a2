"""Copy repair throughput when `out` has a different 16-byte phase than `in`
(the general kernel's per-unit store path) vs the same phase. 2^28 units."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_06349_b200 as P  # noqa: E402
from paper_2601_06349_b200 import _lib  # noqa: E402

n = 1 << 28
x = _lib.gen_config(2, n + 16, seed=2)
o = torch.empty(n + 16, dtype=torch.int16, device="cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for pi, po in ((0, 0), (0, 1), (1, 0), (3, 6), (1, 1)):
    src, dst = x[pi:pi + n], o[po:po + n]
    best = 1e9
    for _ in range(10):
        _lib.l2_flush(flush)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        P.to_well_formed(src, out=dst)
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    print(f"in phase {pi} out phase {po}: {best * 1e3:7.1f} us  {2 * n / best / 1e6:7.0f} GB/s", flush=True)
