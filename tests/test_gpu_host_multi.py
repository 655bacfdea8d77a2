"""GPU: the host-memory form over several GPUs (u16m_to_well_formed_host_multi,
the call behind utf16mend::to_well_formed on host spans and Python
fix_utf16le). On a one-GPU box the devices are virtual (ids repeat): every
range runs its own pipeline thread on the same GPU, which exercises the range
split, the halo units read from host memory at every range edge and the
per-device locking exactly as distinct GPUs would."""
import ctypes

import numpy as np
import pytest
import torch

import oracle as O

pytestmark = pytest.mark.gpu


def _ids(*ids):
    return (ctypes.c_int * len(ids))(*ids)


def _multi(P, src, n, dst, ids):
    L = P._lib.raw()
    arr = _ids(*ids) if ids else None
    return L.u16m_to_well_formed_host_multi(src, n, dst, len(ids), arr)


@pytest.mark.parametrize("ids", [(0,), (0, 0), (0, 0, 0), (0, 0, 0, 0, 0, 0, 0, 0), ()])
def test_host_multi_c1_pinned_and_pageable(P, cuda, ids):
    n = (1 << 28) + 4099  # config 1 size, ragged: ranges end mid-vector
    x = P._lib.gen_config(1, n, seed=1)
    hx = x.cpu().numpy().view(np.uint16)
    e = O.stencil_mt(hx)
    pin = torch.empty(n, dtype=torch.int16, pin_memory=True)
    pin.copy_(x)
    pout = torch.empty(n, dtype=torch.int16, pin_memory=True)
    assert _multi(P, pin.data_ptr(), n, pout.data_ptr(), ids) == 0
    assert (pout.numpy().view(np.uint16) == e).all()
    assert _multi(P, pin.data_ptr(), n, pin.data_ptr(), ids) == 0        # in place
    assert (pin.numpy().view(np.uint16) == e).all()
    if len(ids) in (0, 3):
        pg = hx.copy()                                                   # pageable
        pgo = np.empty_like(pg)
        assert _multi(P, pg.ctypes.data, n, pgo.ctypes.data, ids) == 0
        assert (pgo == e).all()
        assert _multi(P, pg.ctypes.data, n, pg.ctypes.data, ids) == 0
        assert (pg == e).all()


def test_host_multi_range_edges_hold_pairs_and_lone_units(P, cuda):
    """Straddling pairs, H|x, x|L and H|H L placed on every possible range
    edge of a 4-way split (ranges are n/4 rounded down to 4096 units)."""
    n = (1 << 27) + 77
    g = 4
    x = O.gen_config(0, n, seed=9)
    for k in range(1, g):
        b = (n // g * k) & ~4095
        for d, pat in ((-3, [0xD800, 0xDC00]), (0, [0xD83D, 0xDE0A])):
            x[b + d - 1:b + d + 1] = pat
        x[b - 1], x[b] = 0xD800, 0xDC00                                   # H|L exactly on the edge
    e = O.stencil_mt(x)
    pin = torch.from_numpy(x.view(np.int16)).pin_memory()
    out = torch.empty_like(pin).pin_memory()
    assert _multi(P, pin.data_ptr(), n, out.data_ptr(), (0,) * g) == 0
    assert (out.numpy().view(np.uint16) == e).all()
    for k in range(1, g):                                                 # lone H|x and x|L on the edges
        b = (n // g * k) & ~4095
        x[b - 1], x[b] = (0xD800, 0x41) if k % 2 else (0x41, 0xDC00)
    e = O.stencil_mt(x)
    pin = torch.from_numpy(x.view(np.int16)).pin_memory()
    assert _multi(P, pin.data_ptr(), n, pin.data_ptr(), (0,) * g) == 0
    assert (pin.numpy().view(np.uint16) == e).all()


def test_host_multi_small_and_errors(P, cuda):
    L = P._lib.raw()
    x = np.array([0x41, 0xD800, 0xDC00, 0xDC00], np.uint16)
    out = np.zeros_like(x)
    assert _multi(P, x.ctypes.data, 4, out.ctypes.data, (0, 0)) == 0       # small: one device
    assert out.tolist() == [0x41, 0xD800, 0xDC00, 0xFFFD]
    assert _multi(P, x.ctypes.data, 0, out.ctypes.data, (0,)) == 0
    bad = _ids(torch.cuda.device_count())
    assert L.u16m_to_well_formed_host_multi(x.ctypes.data, 4, out.ctypes.data, 1, bad) == 1   # INVALID
    assert L.u16m_to_well_formed_host_multi(x.ctypes.data, 4, out.ctypes.data, -1, None) == 1
    assert L.u16m_to_well_formed_host_multi(x.ctypes.data, 4, x.ctypes.data + 2, 0, None) == 2  # ALIAS


@pytest.mark.slow
def test_host_multi_config4_full(P, cuda):
    """Config 4 (2^32 units, 8 GiB) from pinned host memory through the
    multi-device host form (4 virtual devices), copy and in place, exact over
    the whole buffer."""
    n = 1 << 32
    x = P._lib.gen_config(4, n, seed=4, shard_len=n)
    hin = torch.empty(n, dtype=torch.int16, pin_memory=True)
    hin.copy_(x)
    del x
    torch.cuda.empty_cache()
    e = O.stencil_mt(hin.numpy().view(np.uint16))
    hout = torch.empty(n, dtype=torch.int16, pin_memory=True)
    assert _multi(P, hin.data_ptr(), n, hout.data_ptr(), (0, 0, 0, 0)) == 0
    assert np.array_equal(hout.numpy().view(np.uint16), e)
    assert _multi(P, hin.data_ptr(), n, hin.data_ptr(), (0, 0, 0, 0)) == 0
    assert np.array_equal(hin.numpy().view(np.uint16), e)


def test_fix_utf16le_uses_every_device(P, cuda):
    """The bytes API goes through the multi-device host form: a job big enough
    for two ranges per visible device repairs exactly."""
    n = (1 << 26) * max(1, torch.cuda.device_count()) + 3
    x = O.gen_config(1, n, seed=21)
    assert np.frombuffer(P.fix_utf16le(x.tobytes()), np.uint16).tobytes() == O.stencil_mt(x).tobytes()


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="needs two distinct GPUs (NVLink peer loads between shards)")
def test_sharded_over_distinct_devices(P, cuda):
    """u16m_to_well_formed_sharded with every shard on its own GPU: the halo
    units are peer loads over NVLink (or a 2-byte peer copy)."""
    G = torch.cuda.device_count()
    Ls = 1 << 22
    x = O.gen_config(4, G * Ls, seed=4, shard_len=Ls)
    e = O.stencil_mt(x)
    shards = [torch.from_numpy(x[g * Ls:(g + 1) * Ls].view(np.int16).copy()).to(f"cuda:{g}") for g in range(G)]
    outs = [torch.empty_like(s) for s in shards]
    P.to_well_formed_sharded(shards, outs)
    assert (np.concatenate([o.cpu().numpy().view(np.uint16) for o in outs]) == e).all()
    P.to_well_formed_sharded(shards)
    assert (np.concatenate([s.cpu().numpy().view(np.uint16) for s in shards]) == e).all()
    devs = [g for g in range(G)]
    n = G * Ls
    pin = torch.from_numpy(x.view(np.int16)).pin_memory()
    out = torch.empty_like(pin).pin_memory()
    assert _multi(P, pin.data_ptr(), n, out.data_ptr(), tuple(devs)) == 0
    assert (out.numpy().view(np.uint16) == e).all()


@pytest.mark.parametrize("big", [False, True])
def test_codec_host_multi_ranges(P, cuda, big):
    """Byte-order-fused host repair over several (virtual) devices: every
    range edge reads its halo units from host memory in the job's byte order,
    and the replacement count is the sum over the ranges."""
    n = 3 * (1 << 25) + 4097  # three ranges of >= 32 Mi units, ragged
    x = O.gen_config(4, n, seed=31, shard_len=n // 3)
    e = O.stencil_mt(x)
    raw = (x.astype(">u2") if big else x).view(np.uint16)
    hin = torch.from_numpy(raw.view(np.int16).copy()).pin_memory()
    hout = torch.empty(n, dtype=torch.int16, pin_memory=True)
    L = P._lib.raw()
    cnt = ctypes.c_ulonglong(0)
    for ids in ((0, 0, 0), (0, 0)):
        assert L.u16m_fix_utf16_bytes_host_multi(hin.data_ptr(), n, hout.data_ptr(), int(big), ctypes.byref(cnt),
                                                 len(ids), _ids(*ids)) == 0
        h = hout.numpy().view(np.uint16)
        h = h.view(">u2").astype(np.uint16) if big else h
        assert np.array_equal(h, e) and cnt.value == int((x != e).sum()), ids
    # pageable input, in place
    buf = raw.copy()
    assert L.u16m_fix_utf16_bytes_host_multi(buf.ctypes.data, n, buf.ctypes.data, int(big), ctypes.byref(cnt), 3,
                                             _ids(0, 0, 0)) == 0
    h = buf.view(">u2").astype(np.uint16) if big else buf
    assert np.array_equal(h, e) and cnt.value == int((x != e).sum())
    assert L.u16m_fix_utf16_bytes_host_multi(hin.data_ptr(), n, hout.data_ptr(), 2, None, 1, _ids(0)) == 1


@pytest.mark.parametrize("pinned", [False, True])
def test_small_host_jobs_zero_copy(P, cuda, pinned):
    """Host jobs of at most 64 Ki units run the kernel on mapped pinned memory
    (the caller's, or the small staging buffer): plain repair copy / in place
    at odd phases, the byte-order-fused form with its count, and the
    validation scan (LE and BE) — all equal to the oracle."""
    L = P._lib.raw()
    rng = np.random.default_rng(17)
    for n in (1, 7, 8, 9, 4095, 65535, 65536):
        x = rng.integers(0, 65536, n).astype(np.uint16)
        x[rng.integers(0, n, max(1, n // 50))] = 0xD800
        e = O.stencil(x)
        for phase in (0, 1, 3):
            base = torch.zeros(n + 16, dtype=torch.int16)
            obase = torch.zeros(n + 16, dtype=torch.int16)
            if pinned:
                base, obase = base.pin_memory(), obase.pin_memory()
            src = base[phase:phase + n]
            src.copy_(torch.from_numpy(x.view(np.int16)))
            out = obase[(phase + 2) % 8:(phase + 2) % 8 + n]
            assert L.u16m_to_well_formed_host(src.data_ptr(), n, out.data_ptr()) == 0
            assert (out.numpy().view(np.uint16) == e).all(), (n, phase, "copy")
            for be in (False, True):
                raw = (x.astype(">u2") if be else x).view(np.uint16)
                src.copy_(torch.from_numpy(raw.view(np.int16).copy()))
                cnt = ctypes.c_ulonglong(0)
                assert L.u16m_fix_utf16_bytes_host(src.data_ptr(), n, src.data_ptr(), int(be), ctypes.byref(cnt)) == 0
                got = src.numpy().view(np.uint16)
                got = got.view(">u2").astype(np.uint16) if be else got
                assert (got == e).all() and cnt.value == int((x != e).sum()), (n, phase, be)
                src.copy_(torch.from_numpy(raw.view(np.int16).copy()))
                offs = (ctypes.c_ulonglong * 16)()
                found = ctypes.c_size_t(0)
                assert L.u16m_unpaired_offsets_bytes_host(src.data_ptr(), n, int(be), 16, offs,
                                                          ctypes.byref(found)) == 0
                exp = np.flatnonzero(x != e)[:16]
                assert found.value == exp.size and list(offs[:found.value]) == exp.tolist(), (n, phase, be)
