"""Same-phase copies whose start or end is not 16-byte aligned: how much the
edge tiles cost. 2^28-unit class jobs, L2 flushed."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_06349_b200 as P  # noqa: E402
from paper_2601_06349_b200 import _lib  # noqa: E402

N = 1 << 28
x = _lib.gen_config(2, N + 64, seed=2)
o = torch.empty(N + 64, dtype=torch.int16, device="cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for ph, n in ((0, N), (1, N), (1, N - 1), (0, N + 1), (0, N - 8), (0, N + 8), (0, N + 16384 * 8 * 0 + 8192)):
    src, dst = x[ph:ph + n], o[ph:ph + n]
    best = 1e9
    for _ in range(10):
        _lib.l2_flush(flush)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        P.to_well_formed(src, out=dst)
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    print(f"phase {ph} n {n - N:+d}: {best * 1e3:7.1f} us", flush=True)
