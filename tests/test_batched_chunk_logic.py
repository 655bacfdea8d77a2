"""CPU check of the chunk/segment rule the pipelined batched host path uses
(paper_2601_06349_b200/csrc/u16m_host.cu, u16m_to_well_formed_batched_host):
per fixed-size chunk, strings wholly inside go to the batched kernel and a
string cut by a chunk edge is repaired on its in-chunk segment with the real
neighbour unit as the halo on the cut side — restated here over the oracle
and compared with the per-string oracle on random batches and chunk sizes."""
import numpy as np

import oracle as O


def simulate(x, offs, chunk):
    n, S = x.size, offs.size - 1
    out = x.copy()
    for c0 in range(0, n, chunk):
        c1 = min(n, c0 + chunk)
        lo = int(np.searchsorted(offs, c0, "left"))
        hi = int(np.searchsorted(offs, c1, "right"))

        def plain(u0, u1, left, right):
            if u1 > u0:
                out[u0:u1] = O.stencil(x[u0:u1], left, right)

        if 1 <= lo <= S and offs[lo] > c0:
            e0 = int(offs[lo])
            if e0 > c1:
                plain(c0, c1, int(x[c0 - 1]), int(x[c1]))
                continue
            plain(c0, e0, int(x[c0 - 1]), -1)
        if hi >= 1 and hi - 1 > lo:
            sub = offs[lo:hi]
            out[sub[0]:sub[-1]] = O.fix_batched(x, sub)[sub[0]:sub[-1]]
        if 1 <= hi <= S and c0 <= offs[hi - 1] < c1:
            plain(int(offs[hi - 1]), c1, -1, int(x[c1]))
    return out


def test_chunk_segments_equal_per_string_repair():
    rng = np.random.default_rng(0)
    for t in range(400):
        n = int(rng.integers(1, 3000))
        x = rng.integers(0, 65536, n).astype(np.uint16)
        k = n // 5 + 1
        x[rng.integers(0, n, k)] = (0xD800 + rng.integers(0, 0x800, k)).astype(np.uint16)
        cuts = np.sort(rng.integers(0, n + 1, int(rng.integers(0, 30))))
        a = int(rng.integers(0, n + 1))
        b = int(rng.integers(a, n + 1))
        offs = np.maximum.accumulate(np.concatenate([[a], np.clip(cuts, a, b), [b]]).astype(np.int64))
        chunk = int(rng.integers(1, 400))
        assert (simulate(x, offs, chunk) == O.fix_batched(x, offs)).all(), (t, n, chunk)
