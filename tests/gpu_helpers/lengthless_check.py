"""The length-less batched entry (u16m_to_well_formed_batched) on strings in a
tensor from the allocator PYTORCH_CUDA_ALLOC_CONF selects for this process,
starting 1 MiB into the tensor and spanning many 20 MiB pages when the
allocator maps expandable segments. Run by tests/test_gpu_parity.py."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
from paper_2601_06349_b200 import _lib  # noqa: E402


def main():
    n = 150 << 20  # units (300 MiB: 15 expandable-segment pages)
    t = torch.zeros(n + (1 << 20), dtype=torch.int16, device="cuda")
    x = O.gen_config(0, n, seed=5)
    view = t[(1 << 19):(1 << 19) + n]
    view.copy_(torch.from_numpy(x.view(np.int16)))
    lens = np.random.default_rng(1).integers(1, 4096, 200_000)
    offs = np.concatenate([[0], np.cumsum(lens)])
    offs = offs[offs <= n]
    offs[-1] = n
    d_off = torch.from_numpy(offs.astype(np.int64)).cuda()
    for inplace in (False, True):
        out = view if inplace else torch.empty_like(view)
        if inplace:
            view.copy_(torch.from_numpy(x.view(np.int16)))
        st = _lib.raw().u16m_to_well_formed_batched(view.data_ptr(), d_off.data_ptr(), d_off.numel() - 1,
                                                    out.data_ptr(), torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        assert st == 0, st
        got = out.cpu().numpy().view(np.uint16)
        exp = O.fix_batched(x, offs)
        bad = int((got != exp).sum())
        assert bad == 0, (os.environ.get("PYTORCH_CUDA_ALLOC_CONF"), inplace, bad)
    print("OK")


if __name__ == "__main__":
    main()
