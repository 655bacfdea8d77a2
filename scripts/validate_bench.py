"""Throughput of the validation entry points (§8(f-1)) on config 1 data:
u16m_count_unpaired (read-only stream kernel) and u16m_unpaired_offsets
(limit 10, the CLI `check` call). Input GB/s, L2 flushed between reps."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_06349_b200 import _lib  # noqa: E402

L = _lib.raw()
n = 1 << 28
x = _lib.gen_config(1, n, seed=1)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
offs = torch.zeros(10, dtype=torch.int64, device="cuda")
alloffs = torch.zeros(n // 16, dtype=torch.int64, device="cuda")
clean = _lib.to_well_formed(x)  # well-formed input: nothing to report
s = torch.cuda.current_stream().cuda_stream
for name, fn in (("count_unpaired", lambda: L.u16m_count_unpaired(x.data_ptr(), n, cnt.data_ptr(), s)),
                 ("unpaired_offsets(limit=10)",
                  lambda: L.u16m_unpaired_offsets(x.data_ptr(), n, 10, offs.data_ptr(), cnt.data_ptr(), s)),
                 ("unpaired_offsets(limit=10), well-formed input",
                  lambda: L.u16m_unpaired_offsets(clean.data_ptr(), n, 10, offs.data_ptr(), cnt.data_ptr(), s)),
                 ("unpaired_offsets(all), well-formed input",
                  lambda: L.u16m_unpaired_offsets(clean.data_ptr(), n, n // 16, alloffs.data_ptr(), cnt.data_ptr(), s)),
                 ("unpaired_offsets(all, 8.3M offsets)",
                  lambda: L.u16m_unpaired_offsets(x.data_ptr(), n, n // 16, alloffs.data_ptr(), cnt.data_ptr(), s))):
    tot = 0.0
    for i in range(13):
        _lib.l2_flush(flush)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        assert fn() == 0
        b.record()
        torch.cuda.synchronize()
        if i >= 3:
            tot += a.elapsed_time(b)
    ms = tot / 10
    print(f"{name}: {ms * 1e3:.1f} us, {2 * n / ms / 1e6:.0f} GB/s input (read-only: 2 B/unit), count={int(cnt.item())}")
