"""CUDA-graph capture of the stream-ordered device entry points.

A caller with many small jobs captures its launch-bound loop once and replays
it (no reference counterpart: the reference is synchronous CPU code,
proj/src/driver.cpp:135-147). Every stream-ordered C-ABI entry must therefore
be capturable: no synchronisation, no legacy-stream work and no host read-back
inside the call. Replays run on NEW contents of the same buffers and are
checked against the oracle, bit-exact."""
import ctypes

import numpy as np
import pytest
import torch

import oracle as O

pytestmark = pytest.mark.gpu


def _fill(t, x):
    t.copy_(torch.from_numpy(np.ascontiguousarray(x, np.uint16).view(np.int16)))


def _host(t):
    return t.cpu().numpy().view(np.uint16)


def _inputs(n, seed):
    rng = np.random.default_rng(seed)
    x = rng.integers(0, 1 << 16, n, dtype=np.uint16)
    # dense surrogates so that every tile holds rewrites and valid pairs
    m = rng.random(n) < 0.3
    x[m] = rng.integers(0xD800, 0xE000, int(m.sum()), dtype=np.uint16)
    return x


@pytest.mark.parametrize("n", [1, 777, 16384, 100003, (1 << 20) + 5])
def test_copy_inplace_count_in_one_graph(P, cuda, n):
    L = P._lib.raw()
    src = torch.empty(n, dtype=torch.int16, device=cuda)
    dst = torch.empty_like(src)
    inp = torch.empty_like(src)
    cnt = torch.zeros(1, dtype=torch.int64, device=cuda)
    _fill(src, _inputs(n, 1))
    side = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        # one eager pass first (lazy module load, device-property cache)
        P.to_well_formed(src, dst, stream=side)
        side.synchronize()
        with torch.cuda.graph(g, stream=side):
            s = side.cuda_stream
            P._lib._check(L.u16m_to_well_formed(src.data_ptr(), n, dst.data_ptr(), s))
            inp.copy_(src)
            P._lib._check(L.u16m_to_well_formed_in_place(inp.data_ptr(), n, s))
            cnt.zero_()
            P._lib._check(L.u16m_count_unpaired(src.data_ptr(), n, cnt.data_ptr(), s))
    for seed in (2, 3, 4):
        x = _inputs(n, seed)
        _fill(src, x)
        g.replay()
        torch.cuda.synchronize()
        e = O.fix_scalar(x)
        assert (_host(dst) == e).all()
        assert (_host(inp) == e).all()
        assert int(cnt.item()) == int((e != x).sum())


def test_halo_and_parts_in_a_graph(P, cuda):
    """The sharded primitives: halo values, device-side halo pointers, and the
    interior / edge split on two captured streams."""
    n = 70001
    L = P._lib.raw()
    whole = torch.empty(n + 2, dtype=torch.int16, device=cuda)
    shard = whole[1:-1]
    out_a = torch.empty(n, dtype=torch.int16, device=cuda)
    out_b = torch.empty_like(out_a)
    _fill(whole, _inputs(n + 2, 10))
    side = torch.cuda.Stream()
    other = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        P.to_well_formed(shard, out_a, stream=side)
        side.synchronize()
        with torch.cuda.graph(g, stream=side):
            lp, rp = whole.data_ptr(), whole.data_ptr() + 2 * (n + 1)
            P._lib._check(L.u16m_to_well_formed_halo_ptr(shard.data_ptr(), n, out_a.data_ptr(), lp, rp,
                                                         side.cuda_stream))
            other.wait_stream(side)
            P.to_well_formed_part(shard, out_b, P._lib.PART_INTERIOR, stream=side)
            with torch.cuda.stream(other):
                P.to_well_formed_part(shard, out_b, P._lib.PART_EDGES, lp, rp, stream=other)
            side.wait_stream(other)
    for seed in (11, 12):
        x = _inputs(n + 2, seed)
        x[0], x[1] = 0xD800, 0xDC00          # a pair straddling the left shard edge
        x[-2], x[-1] = 0xD801, 0x0041        # a lone high at the right edge
        _fill(whole, x)
        g.replay()
        torch.cuda.synchronize()
        e = O.fix_scalar(x)[1:-1]
        assert (_host(out_a) == e).all()
        assert (_host(out_b) == e).all()


def test_batched_and_offsets_scan_in_a_graph(P, cuda):
    """Entries that take stream-ordered workspace (the batched tile table, the
    offsets scan's tile counts) and launch programmatic dependents."""
    L = P._lib.raw()
    rng = np.random.default_rng(5)
    lens = rng.integers(0, 700, 3000)
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    n = int(off[-1])
    data = torch.empty(n, dtype=torch.int16, device=cuda)
    out = torch.empty_like(data)
    d_off = torch.from_numpy(off).to(cuda)
    cap = 4096
    offs = torch.empty(cap, dtype=torch.int64, device=cuda)
    cnt = torch.zeros(1, dtype=torch.int64, device=cuda)
    _fill(data, _inputs(n, 20))
    side = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        s = side.cuda_stream
        P._lib._check(L.u16m_to_well_formed_batched_n(data.data_ptr(), n, d_off.data_ptr(), len(lens),
                                                      out.data_ptr(), s))
        P._lib._check(L.u16m_unpaired_offsets(data.data_ptr(), n, cap, offs.data_ptr(), cnt.data_ptr(), s))
        side.synchronize()
        with torch.cuda.graph(g, stream=side):
            P._lib._check(L.u16m_to_well_formed_batched_n(data.data_ptr(), n, d_off.data_ptr(), len(lens),
                                                          out.data_ptr(), s))
            P._lib._check(L.u16m_unpaired_offsets(data.data_ptr(), n, cap, offs.data_ptr(), cnt.data_ptr(), s))
    for seed in (21, 22, 23):
        x = _inputs(n, seed)
        _fill(data, x)
        g.replay()
        torch.cuda.synchronize()
        assert (_host(out) == O.fix_batched(x, off)).all()
        want = O.unpaired_offsets(x, cap)
        k = int(cnt.item())
        assert k == len(want)
        assert offs[:k].cpu().tolist() == want


def test_codec_fused_in_a_graph(P, cuda):
    """Byte-order-fused repair with a device replacement count (CLI `fix` chain)."""
    L = P._lib.raw()
    n = 50021
    src = torch.empty(n, dtype=torch.int16, device=cuda)
    dst = torch.empty_like(src)
    cnt = torch.zeros(1, dtype=torch.int64, device=cuda)
    _fill(src, _inputs(n, 30))
    side = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        s = side.cuda_stream
        P._lib._check(L.u16m_fix_utf16_bytes(src.data_ptr(), n, dst.data_ptr(), 1, cnt.data_ptr(), s))
        side.synchronize()
        with torch.cuda.graph(g, stream=side):
            cnt.zero_()
            P._lib._check(L.u16m_fix_utf16_bytes(src.data_ptr(), n, dst.data_ptr(), 1, cnt.data_ptr(), s))
    for seed in (31, 32):
        x = _inputs(n, seed)
        _fill(src, x.byteswap())           # big-endian bytes in memory
        g.replay()
        torch.cuda.synchronize()
        e = O.fix_scalar(x)
        assert (_host(dst).byteswap() == e).all()
        assert int(cnt.item()) == int((e != x).sum())
