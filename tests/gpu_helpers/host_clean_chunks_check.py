"""Pageable in-place host jobs skip the copy-back of chunks without rewrites
(the caller's buffer already holds them). Mostly clean buffers with rewrites
in chosen chunks only — none, the first, the last, isolated middle ones, pairs
and lone surrogates straddling chunk edges — through the plain and the
byte-order-fused host entries (LE/BE, with and without the count), pageable
and pinned, in place and copy, against the oracle. The chunk size is this
process's U16M_PIPE_CHUNK_KIB. Run by tests/test_gpu_parity.py."""
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
chunk = int(os.environ.get("U16M_PIPE_CHUNK_KIB", "32768")) * 512


def run(x, tag):
    n = x.size
    e = O.fix_scalar(x) if n < 200_000 else O.stencil_mt(x)
    want = int((e != x).sum())
    for pinned in (False, True):
        for inplace in (True, False):
            def buf(a):
                t = torch.from_numpy(a.view(np.int16).copy())
                return t.pin_memory() if pinned else t
            # plain entry
            src = buf(x)
            out = src if inplace else buf(np.zeros_like(x))
            assert L.u16m_to_well_formed_host(src.data_ptr(), n, out.data_ptr()) == 0
            got = out.numpy().view(np.uint16)
            assert (got == e).all(), (tag, "plain", pinned, inplace, int((got != e).sum()))
            # byte-order-fused entry, with and without the count
            for be in (0, 1):
                xb = x.byteswap() if be else x
                for with_count in (True, False):
                    src = buf(xb)
                    out = src if inplace else buf(np.zeros_like(x))
                    cnt = ctypes.c_ulonglong(12345)
                    st = L.u16m_fix_utf16_bytes_host(src.data_ptr(), n, out.data_ptr(), be,
                                                     ctypes.byref(cnt) if with_count else None)
                    assert st == 0
                    got = out.numpy().view(np.uint16)
                    got = got.byteswap() if be else got
                    assert (got == e).all(), (tag, "codec", be, pinned, inplace)
                    if with_count:
                        assert cnt.value == want, (tag, cnt.value, want)


def main():
    rng = np.random.default_rng(11)
    n = 23 * chunk + 4321
    clean = rng.integers(0x20, 0x7F, n).astype(np.uint16)
    run(clean, "all clean")
    for dirty_chunks, tag in (([0], "first"), ([23], "ragged last"), ([22], "last full"), ([5], "one middle"),
                              ([3, 4, 11, 17], "several"), (list(range(24)), "all")):
        x = clean.copy()
        for c in dirty_chunks:
            lo, hi = c * chunk, min(n, (c + 1) * chunk)
            pos = rng.integers(lo, hi, 7)
            x[pos] = rng.integers(0xD800, 0xE000, 7).astype(np.uint16)
        run(x, tag)
    # surrogates exactly at chunk edges: valid pairs across an edge (both chunks stay clean),
    # a lone high as a chunk's last unit, a lone low as a chunk's first unit
    x = clean.copy()
    for c, kind in ((2, "pair"), (6, "lone_high"), (9, "lone_low"), (13, "high_high"), (19, "pair")):
        edge = c * chunk
        if kind == "pair":
            x[edge - 1], x[edge] = 0xD83D, 0xDE00
        elif kind == "lone_high":
            x[edge - 1] = 0xD800
        elif kind == "lone_low":
            x[edge] = 0xDC00
        else:
            x[edge - 1], x[edge] = 0xD800, 0xD801
    run(x, "chunk edges")
    print("OK")


if __name__ == "__main__":
    main()
