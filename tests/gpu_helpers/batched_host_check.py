"""u16m_to_well_formed_batched_host under the chunk size this process's
U16M_PIPE_CHUNK_KIB selects: string-aligned pipeline chunks, the whole-buffer
fallback for a string longer than a chunk, all-empty batches, pinned and
pageable, copy and in place. Run by tests/test_gpu_parity.py."""
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


def check(x, offs, tag):
    n = x.size
    e = O.fix_batched(x, offs)
    for pinned in (False, True):
        for inplace in (False, True):
            src = torch.from_numpy(x.view(np.int16).copy())
            if pinned:
                src = src.pin_memory()
            out = src if inplace else (torch.empty_like(src).pin_memory() if pinned else torch.empty_like(src))
            st = L.u16m_to_well_formed_batched_host(src.data_ptr(), n, offs.ctypes.data, offs.size - 1, out.data_ptr())
            assert st == 0, (tag, st)
            got = out.numpy().view(np.uint16)
            assert (got == e).all(), (tag, pinned, inplace, int((got != e).sum()))


def main():
    rng = np.random.default_rng(5)
    n = 3_000_017
    x = O.gen_config(1, n, seed=7)
    # many short strings (and runs of empty ones), head and tail outside every string
    cuts = np.sort(np.concatenate([rng.integers(3, n - 5, 40_000), np.full(50, 1_000_000)]))
    check(x, np.concatenate([[3], cuts, [n - 5]]).astype(np.int64), "short strings")
    # strings longer than a chunk (cut by chunk edges: plain-kernel segments with real halos)
    check(x, np.array([0, 10, n - 10, n], np.int64), "long string")
    check(x, np.array([5, 5, n - 7], np.int64), "one long string, empty first")
    # long and short strings mixed, and strings cut exactly one unit into a chunk
    chunk = int(os.environ.get("U16M_PIPE_CHUNK_KIB", "32768")) * 512
    mix = np.sort(np.concatenate([rng.integers(0, n, 300), [chunk + 1, 2 * chunk - 1, 2 * chunk + 1]]))
    check(x, np.concatenate([[0], mix[mix < n], [n]]).astype(np.int64), "mixed lengths")
    # only empty strings
    check(x, np.full(1001, 12345, np.int64), "empty strings")
    # strings ending exactly on multiples of the chunk size
    edges = np.arange(0, n, max(1, chunk // 4), dtype=np.int64)
    check(x, np.concatenate([edges, [n]]).astype(np.int64), "chunk-aligned strings")
    print("OK")


if __name__ == "__main__":
    main()
