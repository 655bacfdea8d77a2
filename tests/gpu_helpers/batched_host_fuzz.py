"""Random batches through the pipelined batched host form under the chunk
size U16M_PIPE_CHUNK_KIB selects (set it small so strings are cut by many
chunk edges): lengths, head/tail outside the strings, empty strings, pinned /
pageable, copy / in place — against the per-string oracle. Prints OK."""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
from paper_2601_06349_b200 import _lib  # noqa: E402

L = _lib.raw()
L.u16m_to_well_formed_batched_host.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_size_t,
                                               ctypes.c_void_p]


def main():
    rng = np.random.default_rng(int(os.environ.get("U16M_FUZZ_SEED", "11")))
    for it in range(int(os.environ.get("U16M_FUZZ_ITERS", "200"))):
        n = int(rng.integers(1, 200_000))
        x = rng.integers(0, 65536, n).astype(np.uint16)
        k = n // 20 + 1
        x[rng.integers(0, n, k)] = (0xD800 + rng.integers(0, 0x800, k)).astype(np.uint16)
        a = int(rng.integers(0, n + 1))
        b = int(rng.integers(a, n + 1))
        cuts = np.sort(rng.integers(a, b + 1, int(rng.integers(0, 200))))
        offs = np.maximum.accumulate(np.concatenate([[a], cuts, [b]]).astype(np.int64))
        e = O.fix_batched(x, offs)
        pinned, inplace = bool(it & 1), bool(it & 2)
        src = torch.from_numpy(x.view(np.int16).copy())
        if pinned:
            src = src.pin_memory()
        out = src if inplace else (torch.zeros_like(src).pin_memory() if pinned else torch.zeros_like(src))
        st = L.u16m_to_well_formed_batched_host(src.data_ptr(), n, offs.ctypes.data, offs.size - 1, out.data_ptr())
        assert st == 0, (it, st)
        got = out.numpy().view(np.uint16)
        assert (got == e).all(), (it, n, pinned, inplace, int((got != e).sum()))
    print("OK")


if __name__ == "__main__":
    main()
