"""GPU parity: the sm_100a kernels (through the C ABI) against the CPU oracle
and the reference's golden vectors. Bit-exact everywhere (integer path)."""
import os
import numpy as np
import pytest
import torch

import oracle as O
from helpers import ALPHABET, boundary_sequences, concat_with_offsets, fuzz_inputs, sha

pytestmark = pytest.mark.gpu


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.uint16).view(np.int16).copy()).cuda()


def host(t):
    return t.cpu().numpy().view(np.uint16)


def gpu_copy(P, x):
    return host(P.to_well_formed(dev(x)))


def gpu_inplace(P, x):
    t = dev(x)
    P.to_well_formed_(t)
    return host(t)


def test_native_library_loaded(P, cuda):
    import os

    maps = open(f"/proc/{os.getpid()}/maps").read()
    assert P.lib_path() in maps


def test_mixed_sample_all_apis(P, cuda, golden):
    _, arr = golden
    x, e = arr["mixed_in"], arr["mixed_expected"]
    assert (gpu_copy(P, x) == e).all()
    assert (gpu_inplace(P, x) == e).all()
    assert np.frombuffer(P.fix_utf16le(x.tobytes()), np.uint16).tolist() == e.tolist()
    s = x.tobytes().decode("utf-16-le", "surrogatepass")
    assert P.fix_str(s) == e.tobytes().decode("utf-16-le")
    assert P.unpaired_surrogate_offsets(x.tobytes()) == [10, 21]
    assert not P.is_well_formed_utf16le(x.tobytes())
    assert P.is_well_formed_utf16le(e.tobytes())


def test_scalar_examples(P, cuda, golden):
    meta, _ = golden
    for ex in meta["scalar_examples"]:
        x = np.array(ex["in"], np.uint16)
        if x.size == 0:
            assert P.fix_utf16le(b"") == b""
            continue
        assert gpu_copy(P, x).tolist() == ex["out"]
        assert gpu_inplace(P, x).tolist() == ex["out"]


def test_boundary_exhaustive_individual(P, cuda, golden):
    """Every boundary-alphabet sequence of length <= 3 as its own launch, plus
    the stored length-4 golden outputs."""
    _, arr = golden
    for s in boundary_sequences(3):
        if s.size == 0:
            continue
        e = O.fix_scalar(s)
        assert (gpu_copy(P, s) == e).all()
        assert (gpu_inplace(P, s) == e).all()


def test_boundary4_and5_batched(P, cuda, golden):
    meta, arr = golden
    for L in (4, 5):
        seqs = list(boundary_sequences(L))
        data, offsets = concat_with_offsets(seqs)
        assert sha(data) == meta[f"boundary{L}_sha_in"]
        out = host(P.to_well_formed_batched(dev(data), torch.from_numpy(offsets).cuda()))
        assert sha(out) == meta[f"boundary{L}_sha_out"]
        if L == 4:
            assert (out == arr["boundary4_out"]).all()
        t = dev(data)
        P.to_well_formed_batched(t, torch.from_numpy(offsets).cuda(), out=t)  # in place
        assert sha(host(t)) == meta[f"boundary{L}_sha_out"]


def test_generate_kats(P, cuda, golden):
    meta, _ = golden
    for k in meta["generate_kats"]:
        x = np.frombuffer(P.generate_utf16le(k["n"], k["pair"], k["mismatch"], k["seed"]), np.uint16)
        assert sha(x) == k["sha_in"]
        assert sha(gpu_copy(P, x)) == k["sha_out"]
        assert sha(gpu_inplace(P, x)) == k["sha_out"]
        assert sha(np.frombuffer(P.fix_utf16le(x.tobytes()), np.uint16)) == k["sha_out"]
        assert P.count_unpaired(dev(x)) == k["changed"]


def test_fuzz_acceptance(P, cuda, golden):
    meta, arr = golden
    ins = fuzz_inputs(meta, arr, lambda n, p, m, s: np.frombuffer(P.generate_utf16le(n, p, m, s), np.uint16))
    assert sha(np.concatenate(ins)) == meta["fuzz"]["sha_in"]
    outs = [gpu_copy(P, x) if x.size else x for x in ins[:600]]
    outs_ip = [gpu_inplace(P, x) if x.size else x for x in ins[:600]]
    data, offsets = concat_with_offsets(ins)
    batched = host(P.to_well_formed_batched(dev(data), torch.from_numpy(offsets).cuda()))
    assert sha(batched) == meta["fuzz"]["sha_out"]
    assert (np.concatenate(outs) == batched[: offsets[600]]).all()
    assert (np.concatenate(outs_ip) == batched[: offsets[600]]).all()


@pytest.mark.parametrize("mode", ["copy", "inplace"])
def test_every_length_and_phase(P, cuda, mode):
    """Lengths 0..300 at every in/out 16-byte phase (edge vectors, the
    other-phase store path, tiles of one vector)."""
    rng = np.random.default_rng(11)
    base = torch.zeros(4096, dtype=torch.int16, device="cuda")
    obase = torch.zeros(4096, dtype=torch.int16, device="cuda")
    for n in list(range(0, 70)) + list(range(70, 301, 7)):
        x = rng.choice(ALPHABET, n)
        e = O.fix_scalar(x)
        for pi in range(8):
            po = (pi * 3 + n) % 8
            src = base[pi:pi + n]
            src.copy_(dev(x)) if n else None
            if mode == "copy":
                dst = obase[po + 16:po + 16 + n]
                guard = obase.clone()
                P.to_well_formed(src, out=dst)
                got = host(dst)
                # nothing outside [po+16, po+16+n) was touched
                diff = (obase != guard).nonzero().flatten().tolist()
                assert all(po + 16 <= i < po + 16 + n for i in diff)
            else:
                guard = base.clone()
                P.to_well_formed_(src)
                got = host(src)
                diff = (base != guard).nonzero().flatten().tolist()
                assert all(pi <= i < pi + n for i in diff)
            assert (got == e).all(), (n, pi, po)


def test_tile_boundaries_and_halos(P, cuda):
    rng = np.random.default_rng(5)
    for n in (8191, 8192, 8193, 8192 * 3 + 5, 1 << 20, 3_000_017):
        x = rng.choice(ALPHABET, n)
        e = O.stencil(x)
        assert (gpu_copy(P, x) == e).all(), n
        assert (gpu_inplace(P, x) == e).all(), n
        # explicit halos: every combination at both ends
        for left in (-1, 0x41, 0xD800, 0xDC00):
            for right in (-1, 0x41, 0xD800, 0xDC00):
                t = dev(x)
                out = torch.empty_like(t)
                P.to_well_formed_halo(t, out, left, right)
                assert (host(out) == O.stencil(x, left, right)).all()
                if n > 100_000:
                    break


def test_valid_pair_straddling_every_position(P, cuda):
    """proj/tests/test_generic_kernel.cpp:113-127, across warp/CTA tiles."""
    n = 2 * 8192 + 64
    for pos in list(range(0, 300)) + list(range(1000, 1100)) + list(range(8150, 8250)) + [n - 2]:
        x = np.full(n, 0x41, np.uint16)
        x[pos], x[pos + 1] = 0xD83D, 0xDE0A
        assert (gpu_copy(P, x) == x).all()
        assert (gpu_inplace(P, x) == x).all()


def test_every_unit_value_in_every_lane(P, cuda):
    """The SWAR classification on the GPU for all 65 536 unit values
    (proj/tests/test_surrogate.cpp:24-33 pins the predicates exhaustively):
    each value u appears as [u, DC00] (pairs iff H(u)) and [D800, u] (pairs
    iff L(u)), in 7-unit records so u visits every lane of a 16-byte vector."""
    u = np.arange(1 << 16, dtype=np.uint16)
    rec = np.empty((1 << 16, 7), np.uint16)
    rec[:, 0], rec[:, 1], rec[:, 2] = u, 0xDC00, 0x41
    rec[:, 3], rec[:, 4], rec[:, 5], rec[:, 6] = 0xD800, u, 0x41, 0x41
    x = rec.reshape(-1)
    e = O.fix_scalar(x)
    assert (gpu_copy(P, x) == e).all()
    assert (gpu_inplace(P, x) == e).all()
    assert (O.stencil(x) == e).all()
    # the 1-unit strings of the batched form see no neighbours at all
    offs = np.arange(u.size + 1, dtype=np.int64)
    z = P.to_well_formed_batched(dev(u), torch.from_numpy(offs).cuda())
    assert (host(z) == np.where((u & 0xF800) == 0xD800, 0xFFFD, u)).all()


def test_well_formed_in_place_identity(P, cuda):
    x = np.frombuffer(P.generate_utf16le(400_000, 0.05, 0.0, 77), np.uint16)
    assert P.is_well_formed_utf16le(x.tobytes())
    assert (gpu_inplace(P, x) == x).all()


def test_count_and_offsets(P, cuda):
    rng = np.random.default_rng(9)
    for n in (1, 31, 1000, 8193, 100_003, 2_000_000):
        x = rng.choice(ALPHABET, n)
        e = O.unpaired_offsets(x)
        t = dev(x)
        assert P.count_unpaired(t) == len(e)
        assert P.unpaired_offsets_device(t).cpu().tolist() == e
        for lim in (0, 1, 7, 1000):
            assert P.unpaired_offsets_device(t, lim).cpu().tolist() == e[:lim]
    assert P.unpaired_surrogate_offsets(O.u16([0x41, 0xDC00, 0x42, 0xD800]).tobytes(), 1) == [1]


def test_offsets_small_scan_threshold(P, cuda):
    """Buffers of up to 64 Ki units take the single-launch scan (one CTA walks
    the tiles), longer ones the count -> prefix -> emit chain: lengths on both
    sides of the switch and of the 16384-unit tile edges, every 16-byte phase,
    limits that stop inside the first, a middle and the last tile, dense and
    sparse rewrites, clean input."""
    rng = np.random.default_rng(77)
    big = rng.choice(ALPHABET, (1 << 16) + 64 + 8)
    sparse = np.full(big.size, 0x41, np.uint16)
    sparse[rng.integers(0, big.size, 40)] = 0xDC00
    for src in (big, sparse):
        t_all = dev(src)
        for n in (16383, 16384, 16385, 32768 + 5, 65535, 65536, 65537, 65536 + 64):
            for ph in (0, 1, 3, 7):
                x = src[ph:ph + n]
                e = O.unpaired_offsets(x)
                t = t_all[ph:ph + n]
                assert P.count_unpaired(t) == len(e)
                assert P.unpaired_offsets_device(t).cpu().tolist() == e, (n, ph)
                for lim in (1, 10, len(e) // 2, len(e), len(e) + 5):
                    assert P.unpaired_offsets_device(t, lim).cpu().tolist() == e[:lim], (n, ph, lim)
    clean = torch.full((65536,), 0x41, dtype=torch.int16, device="cuda")
    assert P.unpaired_offsets_device(clean, 10).numel() == 0
    # nothing is written past `limit` entries (guard region behind offsets_out), both paths
    L = P._lib.raw()
    s0 = torch.cuda.current_stream().cuda_stream
    for n in (50_000, 65536 + 64):
        x = big[:n]
        e = O.unpaired_offsets(x)
        t = dev(x)
        for lim in (1, 10, 333, len(e)):
            buf = torch.full((lim + 64,), -7, dtype=torch.int64, device="cuda")
            cnt = torch.full((3,), -7, dtype=torch.int64, device="cuda")
            assert L.u16m_unpaired_offsets(t.data_ptr(), n, lim, buf.data_ptr(), cnt[1:].data_ptr(), s0) == 0
            torch.cuda.synchronize()
            assert cnt.tolist() == [-7, min(lim, len(e)), -7]
            assert buf[:lim].tolist() == e[:lim] and (buf[lim:] == -7).all(), (n, lim)
    # the host scan of a short buffer (mapped pinned memory read by the same kernel)
    b = big[:50_001].tobytes()
    assert P.unpaired_surrogate_offsets(b) == O.unpaired_offsets(big[:50_001])
    assert P.unpaired_surrogate_offsets(b, 3) == O.unpaired_offsets(big[:50_001], 3)


def test_offsets_many_tiles(P, cuda):
    """unpaired offsets over more than one round of the single-CTA tile prefix
    (32768 tiles of 8192 units): lone surrogates planted at known places in an
    otherwise ASCII 2^28+ unit buffer, including the first and last unit."""
    n = (1 << 28) + 12_345
    rng = np.random.default_rng(5)
    pos = np.unique(np.concatenate([[0, n - 1, 8191, 8192, (1 << 28) - 1, 1 << 28],
                                    rng.integers(0, n, 5000)]))
    pos = pos[np.concatenate([[True], np.diff(pos) > 1])]   # no two adjacent: each stays lone
    t = torch.full((n,), 0x41, dtype=torch.int16, device="cuda")
    idx = torch.from_numpy(pos.astype(np.int64)).cuda()
    t[idx] = torch.tensor(np.where(pos % 2 == 0, 0xD800, 0xDC00).astype(np.uint16).view(np.int16)).cuda()
    assert P.count_unpaired(t) == pos.size
    assert P.unpaired_offsets_device(t).cpu().numpy().tolist() == pos.tolist()
    for lim in (1, 10, 4999):
        assert P.unpaired_offsets_device(t, lim).cpu().numpy().tolist() == pos[:lim].tolist()
    clean = torch.full((n,), 0x41, dtype=torch.int16, device="cuda")
    assert P.unpaired_offsets_device(clean, 10).numel() == 0


def test_batched_edges(P, cuda):
    rng = np.random.default_rng(21)
    # string-edge semantics: H|L across an edge must both become FFFD
    x = O.u16([0x41, 0xD800, 0xDC00, 0x42, 0xDC00, 0xD800])
    for offs in ([0, 2, 4, 6], [0, 6], [1, 1, 3, 5], [0, 1, 2, 3, 4, 5, 6], [2, 2]):
        o = np.array(offs, np.int64)
        got = host(P.to_well_formed_batched(dev(x), torch.from_numpy(o).cuda()))
        assert (got == O.fix_batched(x, o)).all(), offs
    # random strings with empties and long strings, unaligned start
    lens = rng.choice([0, 1, 2, 3, 7, 8, 9, 31, 100, 5000, 20000], 3000)
    offsets = np.zeros(lens.size + 1, np.int64)
    offsets[1:] = np.cumsum(lens) + 5
    offsets[0] = 5
    data = rng.choice(ALPHABET, int(offsets[-1]) + 9)
    e = O.fix_batched(data, offsets)
    got = host(P.to_well_formed_batched(dev(data), torch.from_numpy(offsets).cuda()))
    assert (got == e).all()
    assert (got[:5] == data[:5]).all() and (got[offsets[-1]:] == data[offsets[-1]:]).all()
    # strings covering only the middle of a large buffer: whole CTA tiles lie
    # before offsets[0] and after offsets[S] and must be left untouched
    data = rng.choice(ALPHABET, 300_001)
    for lo, hi in ((50_001, 150_003), (16_384, 32_768), (0, 299_990), (299_000, 300_001)):
        cuts = np.sort(rng.integers(lo, hi, 40))
        offsets = np.concatenate([[lo], cuts, [hi]]).astype(np.int64)
        e = O.fix_batched(data, offsets)
        t = dev(data)
        got = host(P.to_well_formed_batched(t, torch.from_numpy(offsets).cuda()))
        assert (got == e).all(), (lo, hi)
        assert (got[:lo] == data[:lo]).all() and (got[hi:] == data[hi:]).all()
        P.to_well_formed_batched(t, torch.from_numpy(offsets).cuda(), out=t)
        assert (host(t) == e).all(), (lo, hi, "in place")


def test_batched_tile_records(P, cuda):
    """Batched starts around the 2048-unit warp-tile records: starts exactly
    on tile boundaries (the start-after flag), 14-17 starts in one tile (the
    15-slot record and its overflow scan), strings spanning empty tiles,
    empty strings on boundaries, every buffer phase."""
    rng = np.random.default_rng(44)
    T = 2048
    for ph in range(8):
        for first in (0, 1, 7, 13):
            lens = []
            pos = first
            base = (first + ph) // 8 * 8 - ph   # warp tile 0 starts here
            while pos < 40 * T:
                kind = rng.integers(0, 6)
                if kind == 0:      # run to the next tile boundary (relative to base)
                    lens.append(int(T - (pos - base) % T))
                elif kind == 1:    # many tiny strings in one tile
                    lens += [int(rng.integers(0, 3)) for _ in range(int(rng.integers(13, 19)))]
                elif kind == 2:    # spans several tiles
                    lens.append(int(rng.integers(2, 5)) * T + int(rng.integers(-2, 3)))
                elif kind == 3:    # empty strings on a boundary
                    lens += [int(T - (pos - base) % T), 0, 0]
                else:
                    lens.append(int(rng.integers(1, 3000)))
                pos = first + sum(lens)
            offs = np.concatenate([[first], first + np.cumsum(lens)]).astype(np.int64)
            buf = rng.choice(ALPHABET, int(offs[-1]) + ph + 9)
            data = buf[ph:]
            e = O.fix_batched(data, offs)
            t = dev(buf)[ph:]
            got = host(P.to_well_formed_batched(t, torch.from_numpy(offs).cuda()))
            assert (got == e).all(), (ph, first)
            P.to_well_formed_batched(t, torch.from_numpy(offs).cuda(), out=t)
            assert (host(t) == e).all(), (ph, first, "in place")


def test_errors(P, cuda):
    t = torch.zeros(100, dtype=torch.int16, device="cuda")
    with pytest.raises(ValueError):
        P.to_well_formed(t[0:50], out=t[25:75])             # partial overlap
    with pytest.raises(ValueError):
        P.fix_utf16le(b"\x00\xd8\x41")                      # odd length
    with pytest.raises(ValueError):
        P.fix_utf16le(b"\x00\xd8", kernel="avx9000")        # unknown kernel
    assert P.fix_utf16le(b"\x00\xd8", kernel="bitmask") == b"\xfd\xff"
    with pytest.raises(ValueError):
        P.to_well_formed(torch.zeros(4, dtype=torch.int16))  # host tensor to device API


def test_host_pipeline_chunks(P, cuda):
    """u16m_to_well_formed_host: > 2 chunks, pinned and pageable, copy and in place."""
    n = (8 << 20) * 2 + 12345
    x = O.gen_config(1, n, seed=77)
    e = O.stencil_mt(x)
    assert np.frombuffer(P.fix_utf16le(x.tobytes()), np.uint16).tobytes() == e.tobytes()
    import ctypes
    L = P._lib.raw()
    pin = torch.from_numpy(x.view(np.int16)).pin_memory()
    outp = torch.empty_like(pin).pin_memory()
    assert L.u16m_to_well_formed_host(pin.data_ptr(), n, outp.data_ptr()) == 0
    assert (outp.numpy().view(np.uint16) == e).all()
    assert L.u16m_to_well_formed_host(pin.data_ptr(), n, pin.data_ptr()) == 0
    assert (pin.numpy().view(np.uint16) == e).all()
    # pageable memory, more chunks than pinned bounce buffers (5.3 x 32 MiB)
    m = (16 << 20) * 5 + 4321
    y = O.gen_config(1, m, seed=78)
    ey = O.stencil_mt(y)
    pg = y.view(np.int16).copy()
    pgo = np.empty_like(pg)
    assert L.u16m_to_well_formed_host(pg.ctypes.data, m, pgo.ctypes.data) == 0
    assert (pgo.view(np.uint16) == ey).all()
    assert L.u16m_to_well_formed_host(pg.ctypes.data, m, pg.ctypes.data) == 0
    assert (pg.view(np.uint16) == ey).all()


@pytest.mark.parametrize("chunk_kib", ["64", "1024"])
def test_host_pageable_inplace_skips_clean_chunks(cuda, chunk_kib):
    """Pageable in-place host jobs do not copy clean chunks back; results and
    replacement counts stay exact for every placement of the dirty chunks
    (helper process: the chunk size is read once per process)."""
    import subprocess
    import sys

    helper = os.path.join(os.path.dirname(os.path.abspath(__file__)), "gpu_helpers", "host_clean_chunks_check.py")
    env = {k: v for k, v in os.environ.items() if not k.startswith("U16M_")}
    env["U16M_PIPE_CHUNK_KIB"] = chunk_kib
    r = subprocess.run([sys.executable, helper], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout + r.stderr


def test_sharded_virtual(P, cuda):
    """u16m_to_well_formed_sharded with several shards on one GPU (device ids
    repeat), including empty shards and adversarial shard-edge patterns."""
    L = 1 << 16
    for G in (1, 2, 4, 7):
        total = G * L
        x = O.gen_config(4, total, seed=4, shard_len=L)
        e = O.stencil(x)
        shards = [dev(x[g * L:(g + 1) * L]) for g in range(G)]
        outs = [torch.empty_like(s) for s in shards]
        P.to_well_formed_sharded(shards, outs)
        assert (np.concatenate([host(o) for o in outs]) == e).all()
        P.to_well_formed_sharded(shards)  # in place
        assert (np.concatenate([host(s) for s in shards]) == e).all()
    # ragged + empty shards
    x = O.gen_config(4, 100_000, seed=4, shard_len=25_000)
    cuts = [0, 0, 1, 24_999, 25_001, 25_001, 60_000, 100_000]
    shards = [dev(x[a:b]) if b > a else torch.empty(0, dtype=torch.int16, device="cuda")
              for a, b in zip(cuts[:-1], cuts[1:])]
    P.to_well_formed_sharded(shards)
    assert (np.concatenate([host(s) for s in shards]) == O.stencil(x)).all()


def test_inplace_race_stress(P, cuda):
    """In-place vs copy on the worst-case error density, repeated, different
    sub-buffer offsets (changes the tile/warp-edge alignment every time)."""
    n = 1 << 22
    x = O.gen_config(1, n + 64, seed=1)
    e_full = None
    big = dev(x)
    for off in (0, 1, 3, 7, 8, 13, 31, 33):
        src = big[off:off + n]
        ref = P.to_well_formed(src)
        for rep in range(3):
            t = src.clone()
            P.to_well_formed_(t)
            assert torch.equal(t, ref)
        if off == 0:
            e_full = O.stencil_mt(x[:n])
            assert (host(ref) == e_full).all()


@pytest.mark.parametrize("cfg", [0, 1, 2, 4])
def test_device_generator_matches_oracle(P, cuda, cfg):
    total = 3_000_000
    shard = 1_000_000 if cfg == 4 else 0
    g = host(P._lib.gen_config(cfg, total, shard_len=shard))
    assert (g == O.gen_config(cfg, total, shard_len=shard)).all()
    w = host(P._lib.gen_config(cfg, total, first=123_457, count=777_777, shard_len=shard))
    assert (w == O.gen_config(cfg, total, first=123_457, count=777_777, shard_len=shard)).all()


def test_device_c3_generator_matches_oracle(P, cuda):
    d, o = P._lib.gen_c3(20_000)
    hd, ho = O.gen_c3(20_000)
    assert (o.cpu().numpy() == ho).all()
    assert (host(d) == hd).all()


# ---- BASELINE configs ---------------------------------------------------------
def test_config0_full(P, cuda):
    n = 1 << 24
    x = O.gen_config(0, n, seed=0)
    e = O.stencil_mt(x)
    t = dev(x)
    assert (host(P.to_well_formed(t)) == e).all()
    assert (host(P.to_well_formed_(t)) == e).all()


def _full_check(x_dev, y_dev, n, chunk=1 << 27):
    """Exact oracle parity over the WHOLE full-size result, streamed to the
    host in chunks extended by a one-unit halo on each side."""
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        lo, hi = max(0, a - 1), min(n, b + 1)
        e = O.stencil_mt(host(x_dev[lo:hi]))
        assert (host(y_dev[a:b]) == e[a - lo:a - lo + (b - a)]).all(), a


@pytest.mark.slow
def test_config1_full_inplace(P, cuda):
    n = 1 << 28
    x = P._lib.gen_config(1, n, seed=1)
    y = x.clone()
    P.to_well_formed_(y)
    _full_check(x, y, n)
    z = P.to_well_formed(x)
    assert torch.equal(y, z)                              # in place == copy
    assert P.count_unpaired(y) == 0                       # well-formed
    assert P.count_unpaired(x) == int((x != y).sum())     # minimality count
    assert torch.equal(P.to_well_formed(y), y)            # idempotence
    frac = (x != y).float().mean().item()
    assert 0.028 < frac < 0.034


@pytest.mark.slow
def test_config2_full_copy(P, cuda):
    n = 1 << 29
    rng = np.random.default_rng(2)
    x = P._lib.gen_config(2, n, seed=2)
    y = P.to_well_formed(x)
    _full_check(x, y, n)
    # every adversarial tile-boundary window (sampled) is exact
    for t in rng.integers(1, n // 256, 200):
        b = int(t) * 256
        a = b - 8
        xin = host(x[a:b + 8])
        assert (host(y[a:b + 8]) == O.stencil(xin, int(host(x[a - 1:a])[0]), int(host(x[b + 8:b + 9])[0]))).all()
    assert P.count_unpaired(y) == 0
    assert torch.equal(P.to_well_formed(y), y)


@pytest.mark.slow
def test_config3_full_batched(P, cuda):
    d, o = P._lib.gen_c3(1 << 20)
    ho = o.cpu().numpy()
    y = P.to_well_formed_batched(d, o)
    hd, hy = host(d), host(y)
    e = O.fix_batched(hd, ho)
    assert (hy == e).all()
    y2 = d.clone()
    P.to_well_formed_batched(y2, o, out=y2)
    assert torch.equal(y2, y)


@pytest.mark.slow
def test_config3_full_lengthless_entry(P, cuda):
    """Full config 3 through the north-star batched signature (no buffer
    length: u16m_to_well_formed_batched), copy and in place, against the
    oracle's per-string fix_scalar."""
    d, o = P._lib.gen_c3(1 << 20)
    L = P._lib.raw()
    s = torch.cuda.current_stream().cuda_stream
    out = torch.empty_like(d)
    assert L.u16m_to_well_formed_batched(d.data_ptr(), o.data_ptr(), o.numel() - 1, out.data_ptr(), s) == 0
    e = O.fix_batched(host(d), o.cpu().numpy())
    assert (host(out) == e).all()
    y = d.clone()
    assert L.u16m_to_well_formed_batched(y.data_ptr(), o.data_ptr(), o.numel() - 1, y.data_ptr(), s) == 0
    assert torch.equal(y, out)


def test_batched_negative_offsets_never_write_outside(P, cuda):
    """offsets[0] < 0 is a contract error: both batched entries clamp the
    extent to the buffer, so nothing before `in`/`out` is read or written
    (the clamp missed A < 0)."""
    L = P._lib.raw()
    s = torch.cuda.current_stream().cuda_stream
    guard = 64
    for ph in range(8):
        n = 50_000
        x = O.gen_config(1, n + 2 * guard, seed=ph)
        t = dev(x)
        for off in (np.array([-5, 100, 4000, n], np.int64), np.array([-(1 << 40), 7, n], np.int64)):
            o = torch.from_numpy(off).cuda()
            out = t.clone()
            base_in = t[guard + ph:]
            base_out = out[guard + ph:]
            assert L.u16m_to_well_formed_batched_n(base_in.data_ptr(), n, o.data_ptr(), o.numel() - 1,
                                                   base_out.data_ptr(), s) == 0
            assert L.u16m_to_well_formed_batched(base_in.data_ptr(), o.data_ptr(), o.numel() - 1,
                                                 base_out.data_ptr(), s) == 0
            torch.cuda.synchronize()
            assert torch.equal(out[:guard + ph], t[:guard + ph])          # nothing before the buffer
            clamped = off.copy()
            clamped[0] = 0
            seg = O.fix_batched(x[guard + ph:guard + ph + n], clamped)
            assert (host(out[guard + ph:guard + ph + n]) == seg).all()


@pytest.mark.slow
def test_config4_shards(P, cuda):
    """Config 4 on one GPU: 4 virtual shards of 2^26 units with adversarial
    shard edges (exact, whole buffer) and one full 2^32-unit shard (windows)."""
    L, G = 1 << 26, 4
    x = P._lib.gen_config(4, G * L, seed=4, shard_len=L)
    e = O.stencil_mt(host(x))
    shards = [x[g * L:(g + 1) * L].clone() for g in range(G)]
    outs = [torch.empty_like(s) for s in shards]
    P.to_well_formed_sharded(shards, outs)
    assert (np.concatenate([host(o) for o in outs]) == e).all()
    P.to_well_formed_sharded(shards)
    assert (np.concatenate([host(s) for s in shards]) == e).all()
    del x, shards, outs
    torch.cuda.empty_cache()
    n = 1 << 32
    x = P._lib.gen_config(4, n, seed=4, shard_len=n)
    y = P.to_well_formed(x)
    _full_check(x, y, n)
    assert P.count_unpaired(y) == 0


@pytest.mark.slow
def test_beyond_32bit_unit_indices(P, cuda):
    """A job of more than 2^32 units (8.6 GB): every unit index past 2^32 needs
    64-bit arithmetic in the kernels. Plain copy / in place / count / offsets
    and the batched form over strings lying on both sides of 2^32; exact
    against the oracle around 2^32 and over the tail, size-independent
    properties over the whole buffer."""
    free, _ = torch.cuda.mem_get_info()
    n = (1 << 32) + (1 << 21) + 5
    if free < 5 * 2 * n:
        pytest.skip("needs ~45 GB of free device memory")
    x = P._lib.gen_config(1, n, seed=33)                   # uniform units: rewrites everywhere
    y = P.to_well_formed(x)

    def window(a, b):
        lo, hi = max(0, a - 1), min(n, b + 1)
        e = O.stencil_mt(host(x[lo:hi]))
        return e[a - lo:a - lo + (b - a)]
    edge = (1 << 32) - (1 << 20)
    assert (host(y[edge:n]) == window(edge, n)).all()      # across 2^32 and to the ragged end
    assert (host(y[:1 << 20]) == window(0, 1 << 20)).all()
    rewrites = sum(int((x[a:a + (1 << 28)] != y[a:a + (1 << 28)]).sum()) for a in range(0, n, 1 << 28))
    assert P.count_unpaired(x) == rewrites
    assert P.count_unpaired(y) == 0
    # offsets: the last ones lie past 2^32
    tail_pos = (x[edge:] != y[edge:]).nonzero().flatten() + edge
    lim = rewrites - tail_pos.numel() + 1000
    offs = P.unpaired_offsets_device(x, limit=lim)
    assert offs.numel() == lim
    assert torch.equal(offs[-1000:], tail_pos[:1000])
    assert int(offs[-1]) > (1 << 32) - (1 << 20)
    del offs
    z = x.clone()
    P.to_well_formed_(z)
    for a in range(0, n, 1 << 28):
        assert torch.equal(z[a:a + (1 << 28)], y[a:a + (1 << 28)]), a   # in place == copy
    del z
    # batched: one long string up to just below 2^32, short strings across it, a long tail string
    cut = (1 << 32) - 3000
    lens = np.random.default_rng(5).integers(0, 700, 20)
    mids = cut + np.concatenate([[0], np.cumsum(lens)])
    offsets = np.concatenate([[7], mids, [n - 11]]).astype(np.int64)
    o = torch.from_numpy(offsets).cuda()
    w = torch.full_like(x, 0x1111)
    P.to_well_formed_batched(x, o, out=w)
    a = cut - (1 << 20)
    seg = host(x[a:n])
    seg_off = np.concatenate([[0], mids - a, [n - 11 - a]]).astype(np.int64)
    e = O.fix_batched(seg, seg_off)
    e[n - 11 - a:] = 0x1111                                # units in no string: not written
    got = host(w[a:n])
    assert (got[1:] == e[1:]).all()                        # (unit 0 of the window has its real predecessor)
    assert (host(w[:7]) == 0x1111).all()
    assert (host(w[7:1 << 20]) == O.fix_batched(host(x[7:(1 << 20) + 1]), np.array([0, (1 << 20) - 6], np.int64))[:(1 << 20) - 7]).all()


def test_parts_on_two_streams(P, cuda):
    """INTERIOR and EDGES parts run concurrently on two streams and together
    equal the whole-job repair (the overlap used by dist.repair_shard)."""
    rng = np.random.default_rng(31)
    for n in (5, 8192, 8193, 3 * 8192, 100_003, 1 << 20):
        x = O.gen_config(1, n, seed=n)
        left, right = 0xD812, 0xDC34
        hal = dev(np.array([left, right], np.uint16))
        lp, rp = hal.data_ptr(), hal.data_ptr() + 2
        e = O.stencil(x, left, right)
        for in_place in (False, True):
            t = dev(x)
            out = t if in_place else torch.empty_like(t)
            s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
            s1.wait_stream(torch.cuda.current_stream())
            s2.wait_stream(torch.cuda.current_stream())
            P.to_well_formed_part(t, out, P._lib.PART_INTERIOR, stream=s1)
            P.to_well_formed_part(t, out, P._lib.PART_EDGES, lp, rp, stream=s2)
            torch.cuda.synchronize()
            assert (host(out) == e).all(), (n, in_place)


def test_batched_entry_without_length(P, cuda, golden):
    """The north-star batched entry (no buffer length; persistent TMA kernel)
    and the length-aware one (tile table + one tile per CTA) agree with the
    oracle, including an offsets[S] beyond n that must be clamped."""
    meta, _ = golden
    seqs = list(boundary_sequences(5))
    data, offsets = concat_with_offsets(seqs)
    L = P._lib.raw()
    t = dev(data)
    o = torch.from_numpy(offsets).cuda()
    out = torch.empty_like(t)
    s = torch.cuda.current_stream().cuda_stream
    assert L.u16m_to_well_formed_batched(t.data_ptr(), o.data_ptr(), o.numel() - 1, out.data_ptr(), s) == 0
    assert sha(host(out)) == meta["boundary5_sha_out"]
    out2 = torch.empty_like(t)
    assert L.u16m_to_well_formed_batched_n(t.data_ptr(), t.numel(), o.data_ptr(), o.numel() - 1,
                                            out2.data_ptr(), s) == 0
    assert torch.equal(out, out2)
    # clamping: claim only the first half of the buffer
    half = t.numel() // 2
    keep = dev(np.full(t.numel() - half, 0x7777, np.uint16))
    buf = torch.cat([t[:half], keep])
    assert L.u16m_to_well_formed_batched_n(buf.data_ptr(), half, o.data_ptr(), o.numel() - 1, buf.data_ptr(), s) == 0
    torch.cuda.synchronize()
    assert (host(buf[half:]) == 0x7777).all()


def test_batched_other_phase_and_copy(P, cuda):
    """Batched copy into an output at every 16-byte phase relative to the
    input (shifted stores in the tile kernel) and into an aligned output."""
    rng = np.random.default_rng(41)
    lens = rng.choice([0, 1, 2, 3, 17, 300, 4095, 20000], 2000)
    offsets = np.zeros(lens.size + 1, np.int64)
    offsets[1:] = np.cumsum(lens) + 11
    offsets[0] = 11
    data = O.gen_config(1, int(offsets[-1]) + 13, seed=41)
    e = O.fix_batched(data, offsets)
    t = dev(data)
    o = torch.from_numpy(offsets).cuda()
    for shift in range(9):
        big = torch.full((t.numel() + 16,), 0x1234, dtype=torch.int16, device="cuda")
        out = big[shift:shift + t.numel()]
        out.copy_(t)
        P.to_well_formed_batched(t, o, out=out)
        got = host(out)
        assert (got == e).all(), shift


def test_batched_runs_of_empty_strings(P, cuda):
    """Long runs of equal offsets (empty strings) at the buffer start, on warp
    and CTA tile boundaries, mid-tile and at the end, through every batched
    entry: length-aware (tile table), length-less (TMA producer walk),
    mismatched in/out phase (general kernel) and in place."""
    rng = np.random.default_rng(77)
    L = P._lib.raw()
    s = torch.cuda.current_stream().cuda_stream
    for run in (1, 31, 32, 33, 100, 5000, 70_000):
        n = 60_000
        pts = sorted({0, 2048, 4096, 8192, 16384, 16385, 3001, 40_000, n} | set(int(v) for v in rng.integers(0, n, 20)))
        offs = []
        for p in pts:
            offs += [p] * (run if p in (0, 2048, 16384, 40_000, n) else 1 + int(rng.integers(0, 3)))
        offs = np.array(offs, np.int64)
        data = rng.choice(ALPHABET, n + 16)
        e = O.fix_batched(data, offs)
        t, o = dev(data), torch.from_numpy(offs).cuda()
        assert (host(P.to_well_formed_batched(t, o)) == e).all(), ("tiles", run)
        out = torch.empty_like(t)
        assert L.u16m_to_well_formed_batched(t.data_ptr(), o.data_ptr(), o.numel() - 1, out.data_ptr(), s) == 0
        assert (host(out) == e).all(), ("no-length", run)
        odd = torch.empty(n + 24, dtype=torch.int16, device="cuda")[3:3 + n + 16]
        P.to_well_formed_batched(t, o, out=odd)
        assert (host(odd)[: n] == e[: n]).all(), ("other phase", run)
        u = t.clone()
        P.to_well_formed_batched(u, o, out=u)
        assert (host(u) == e).all(), ("in place", run)


class _DLPackArray:
    """A minimal foreign device array: only the DLPack protocol (as CuPy or
    JAX arrays expose it)."""

    def __init__(self, t):
        self._t = t

    def __dlpack__(self, **kw):
        return self._t.__dlpack__(**kw)

    def __dlpack_device__(self):
        return self._t.__dlpack_device__()


def test_dlpack_producers_zero_copy(P, cuda):
    x = O.u16([0x41, 0xD800, 0x42, 0xDC00, 0xD83D, 0xDE0A, 0xDBFF])
    e = O.fix_scalar(x)
    t = dev(x)
    assert (host(P.to_well_formed(_DLPackArray(t))) == e).all()
    P.to_well_formed_(_DLPackArray(t))                     # repairs the producer's memory
    assert (host(t) == e).all()
    t = dev(x)
    assert P.count_unpaired(_DLPackArray(t)) == 3
    assert P.unpaired_offsets_device(_DLPackArray(t)).cpu().tolist() == [1, 3, 6]
    offs = torch.tensor([0, 2, 7], dtype=torch.int64, device="cuda")
    got = P.to_well_formed_batched(_DLPackArray(t), _DLPackArray(offs))
    assert (host(got) == O.fix_batched(x, np.array([0, 2, 7]))).all()


def test_host_scan_chunks(P, cuda):
    """u16m_unpaired_offsets_host (CLI check, is_well_formed, Python offsets on
    bytes): chunked over 32 MiB pieces with halos — a pair straddling a chunk
    edge is valid, lone units at chunk edges are found; pinned and pageable;
    early exit at `limit`."""
    import ctypes
    C = 16 << 20                       # default pipeline chunk in units
    n = 3 * C + 777
    x = np.full(n, 0x41, np.uint16)
    x[C - 1], x[C] = 0xD83D, 0xDE0A   # valid pair across the first chunk edge
    lone = [0, 5, 2 * C - 1, 2 * C, 3 * C + 776]
    for p_ in lone:
        x[p_] = 0xDC00 if p_ % 2 else 0xD800
    x[2 * C], x[2 * C - 1] = 0xDC00, 0xDC00  # L|L across the second edge: both lone
    exp = O.unpaired_offsets(x)
    assert exp == sorted(set(lone))
    assert P.unpaired_surrogate_offsets(x.tobytes()) == exp
    for lim in (1, 2, 3, 4, 5, 100):
        assert P.unpaired_surrogate_offsets(x.tobytes(), lim) == exp[:lim]
    assert not P.is_well_formed_utf16le(x.tobytes())
    assert P.is_well_formed_utf16le(O.fix_scalar(x).tobytes())
    L = P._lib.raw()
    pin = torch.from_numpy(x.view(np.int16)).pin_memory()
    out = np.zeros(10, np.uint64)
    cnt = ctypes.c_size_t(0)
    assert L.u16m_unpaired_offsets_host(pin.data_ptr(), n, 10, out.ctypes.data, ctypes.byref(cnt)) == 0
    assert out[: cnt.value].tolist() == exp


def test_batched_host_staged(P, cuda):
    """u16m_to_well_formed_batched_host (behind the C++ batched API on host
    spans): pageable and pinned buffers over several 32 MiB bounce chunks,
    copy and in place, strings crossing chunk edges."""
    import ctypes
    rng = np.random.default_rng(31)
    n = (16 << 20) * 3 + 999
    x = O.gen_config(1, n, seed=31)
    cuts = np.unique(np.concatenate([[5, n - 3, 16 << 20, (16 << 20) + 1], rng.integers(5, n - 3, 20000)]))
    offs = cuts.astype(np.int64)
    e = O.fix_batched(x, offs)
    L = P._lib.raw()
    L.u16m_to_well_formed_batched_host.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p,
                                                    ctypes.c_size_t, ctypes.c_void_p]
    src = x.view(np.int16).copy()
    out = np.empty_like(src)
    assert L.u16m_to_well_formed_batched_host(src.ctypes.data, n, offs.ctypes.data, offs.size - 1, out.ctypes.data) == 0
    assert (out.view(np.uint16) == e).all()
    assert L.u16m_to_well_formed_batched_host(src.ctypes.data, n, offs.ctypes.data, offs.size - 1, src.ctypes.data) == 0
    assert (src.view(np.uint16) == e).all()
    pin = torch.from_numpy(x.view(np.int16).copy()).pin_memory()
    assert L.u16m_to_well_formed_batched_host(pin.data_ptr(), n, offs.ctypes.data, offs.size - 1, pin.data_ptr()) == 0
    assert (pin.numpy().view(np.uint16) == e).all()
    bad = offs.copy()
    bad[3], bad[4] = bad[4], bad[3]
    assert L.u16m_to_well_formed_batched_host(src.ctypes.data, n, bad.ctypes.data, bad.size - 1, out.ctypes.data) == 1


def test_other_phase_copy_all_shifts(P, cuda):
    """Copies whose output starts at a different 16-byte phase than the input
    (the shifted-store kernel): every in/out phase pair, several CTA tiles,
    units at every warp/tile straddle, nothing outside the output touched."""
    rng = np.random.default_rng(17)
    n = 16384 * 3 + 4099
    x = rng.choice(ALPHABET, n)
    x[16384 * np.arange(1, 4) - 1] = 0xD800     # H right before tile starts
    x[2048 * np.arange(1, 20)] = 0xDC00          # L on warp-tile starts
    e = O.stencil(x)
    src_base = torch.zeros(n + 16, dtype=torch.int16, device="cuda")
    out_base = torch.zeros(n + 32, dtype=torch.int16, device="cuda")
    for pi in range(8):
        src = src_base[pi:pi + n]
        src.copy_(dev(x))
        for po in range(8):
            out_base.fill_(0x1234)
            dst = out_base[8 + po:8 + po + n]
            P.to_well_formed(src, out=dst)
            assert (host(dst) == e).all(), (pi, po)
            rest = torch.cat([out_base[:8 + po], out_base[8 + po + n:]])
            assert bool((rest == 0x1234).all()), (pi, po)


def test_python_batch_api(P, cuda):
    """fix_utf16le_batch / fix_str_batch: one GPU call, per-item semantics
    (no pairing across items), order kept, empties allowed."""
    rng = np.random.default_rng(8)
    items = []
    for i in range(3000):
        n = int(rng.choice([0, 1, 2, 3, 50, 700]))
        items.append(rng.choice(ALPHABET, n).astype(np.uint16).tobytes())
    items[5], items[6] = O.u16([0x41, 0xD800]).tobytes(), O.u16([0xDC00, 0x42]).tobytes()  # H | L across items
    got = P.fix_utf16le_batch(items)
    assert got == [O.fix_scalar(np.frombuffer(b, np.uint16)).tobytes() if b else b"" for b in items]
    assert got[5] == O.u16([0x41, 0xFFFD]).tobytes() and got[6] == O.u16([0xFFFD, 0x42]).tobytes()
    texts = ["ok", "", "a\ud800", "\udc00b", "\U0001F60A", "x😊y"]
    assert P.fix_str_batch(texts) == [P.fix_str(t) for t in texts]
    assert P.fix_utf16le_batch([]) == [] and P.fix_utf16le_batch([b"", b""]) == [b"", b""]


@pytest.mark.parametrize("conf", ["", "expandable_segments:True", "backend:cudaMallocAsync"])
def test_lengthless_entry_under_every_torch_allocator(cuda, conf):
    """The length-less batched entry sizes its grid from the allocation holding
    the strings; with VMM-mapped memory (expandable segments) that range is one
    20 MiB page, so it must take the bound-free kernel — exact either way."""
    import subprocess
    import sys

    helper = os.path.join(os.path.dirname(os.path.abspath(__file__)), "gpu_helpers", "lengthless_check.py")
    env = dict(os.environ, PYTORCH_CUDA_ALLOC_CONF=conf)
    r = subprocess.run([sys.executable, helper], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout + r.stderr


def test_concurrent_callers_on_their_own_streams(P, cuda):
    """SURVEY.md §8(b) threading contract: the library is re-entrant — host
    threads repairing on their own streams (device API) and through the host
    pipeline at the same time all get exact results."""
    import threading

    rng = np.random.default_rng(77)
    jobs = [rng.integers(0, 65536, int(rng.integers(1, 3_000_000))).astype(np.uint16) for _ in range(8)]
    exp = [O.stencil(x) for x in jobs]
    errors = []

    def device_worker(k):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for _ in range(5):
                    t = torch.from_numpy(jobs[k].view(np.int16).copy()).cuda(non_blocking=False)
                    y = P.to_well_formed(t, stream=s)
                    P.to_well_formed_(t, stream=s)
                    s.synchronize()
                    assert (y.cpu().numpy().view(np.uint16) == exp[k]).all()
                    assert (t.cpu().numpy().view(np.uint16) == exp[k]).all()
        except Exception as e:  # noqa: BLE001
            errors.append((k, repr(e)))

    def host_worker(k):
        try:
            for _ in range(5):
                got = np.frombuffer(P.fix_utf16le(jobs[k].tobytes()), np.uint16)
                assert (got == exp[k]).all()
        except Exception as e:  # noqa: BLE001
            errors.append((k, repr(e)))

    threads = [threading.Thread(target=device_worker if k % 2 else host_worker, args=(k,)) for k in range(8)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors


@pytest.mark.parametrize("chunk_kib", ["64", "1024", ""])
def test_batched_host_pipeline_chunks(cuda, chunk_kib):
    """The pipelined batched host path: chunks end on string boundaries (no
    halos), head / tail outside the strings copied on the host, and a string
    longer than a chunk falls back to the whole-buffer path — exact for every
    chunk size."""
    import subprocess
    import sys

    helper = os.path.join(os.path.dirname(os.path.abspath(__file__)), "gpu_helpers", "batched_host_check.py")
    env = {k: v for k, v in os.environ.items() if not k.startswith("U16M_")}
    if chunk_kib:
        env["U16M_PIPE_CHUNK_KIB"] = chunk_kib
    r = subprocess.run([sys.executable, helper], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout + r.stderr
