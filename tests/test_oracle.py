"""CPU: pin the oracle (oracle/) against the reference's golden vectors and,
when oracle/_ref was built here, against the reference's own code."""
import numpy as np
import pytest

import oracle as O
from helpers import ALPHABET, boundary_sequences, concat_with_offsets, fuzz_inputs, sha


def test_mixed_sample(golden):
    meta, arr = golden
    x, e = arr["mixed_in"], arr["mixed_expected"]
    assert x.size == 31
    assert (O.fix_scalar(x) == e).all()
    assert (O.stencil(x) == e).all()
    assert list(np.nonzero(x != e)[0]) == [10, 21]
    assert x[29] == 0xD83D and x[30] == 0xDE0A


def test_scalar_examples(golden):
    meta, _ = golden
    for ex in meta["scalar_examples"]:
        assert O.fix_scalar(ex["in"]).tolist() == ex["out"]
        assert O.stencil(ex["in"]).tolist() == ex["out"]


def test_alphabet(golden):
    assert (golden[1]["boundary_alphabet"] == ALPHABET).all()


def test_boundary4_stored(golden):
    _, arr = golden
    seqs = list(boundary_sequences(4))
    data, _ = concat_with_offsets(seqs)
    assert (data == arr["boundary4_in"]).all()
    out = np.concatenate([O.fix_scalar(s) for s in seqs])
    assert (out == arr["boundary4_out"]).all()


def test_boundary5_exhaustive(golden):
    meta, _ = golden
    seqs = list(boundary_sequences(5))
    assert len(seqs) == meta["boundary5_count"] == 37449
    data, offsets = concat_with_offsets(seqs)
    assert sha(data) == meta["boundary5_sha_in"]
    scan = O.fix_batched(data, offsets)
    assert sha(scan) == meta["boundary5_sha_out"]
    # the stencil (what the GPU computes) equals the consuming scan everywhere
    st = np.concatenate([O.stencil(s) for s in seqs])
    assert (st == scan).all()


def test_classification_all_units():
    x = np.arange(65536, dtype=np.uint16)
    # lone unit: H and L become FFFD, everything else survives
    out = np.array([O.stencil([u])[0] for u in range(0xD000, 0xE100)], np.uint16)
    sur = (np.arange(0xD000, 0xE100) >= 0xD800) & (np.arange(0xD000, 0xE100) <= 0xDFFF)
    assert (out[sur] == 0xFFFD).all()
    assert (out[~sur] == np.arange(0xD000, 0xE100)[~sur]).all()
    y = O.stencil(x)
    assert y.size == 65536


def test_generate_kats(golden):
    meta, _ = golden
    for k in meta["generate_kats"]:
        x = O.ref_generate(k["n"], k["pair"], k["mismatch"], k["seed"])
        assert sha(x) == k["sha_in"], k
        assert x[:16].tolist() == k["head_in"]
        y = O.fix_scalar(x)
        assert sha(y) == k["sha_out"]
        assert int((x != y).sum()) == k["changed"]


def test_fuzz(golden):
    meta, arr = golden
    ins = fuzz_inputs(meta, arr, O.ref_generate)
    assert sha(np.concatenate(ins)) == meta["fuzz"]["sha_in"]
    assert sha(np.concatenate([O.fix_scalar(x) for x in ins])) == meta["fuzz"]["sha_out"]


def test_properties_random():
    rng = np.random.default_rng(1)
    for t in range(300):
        n = int(rng.integers(0, 400))
        x = rng.choice(ALPHABET, n) if t % 2 else rng.integers(0, 65536, n).astype(np.uint16)
        y = O.fix_scalar(x)
        assert (O.stencil(x) == y).all()
        assert O.is_well_formed(y)
        assert (O.fix_scalar(y) == y).all()                   # idempotence
        ch = np.nonzero(x != y)[0]
        assert (y[ch] == 0xFFFD).all()                        # minimality
        assert ((x[ch] & 0xF800) == 0xD800).all()
        assert O.unpaired_offsets(x) == ch.tolist()
        assert O.is_well_formed(x) == (ch.size == 0)


def test_halo_sharding_is_exact():
    rng = np.random.default_rng(2)
    x = rng.choice(ALPHABET, 5000)
    full = O.stencil(x)
    cuts = [0, 1, 2, 777, 778, 2500, 4999, 5000]
    for a, b in zip(cuts[:-1], cuts[1:]):
        left = int(x[a - 1]) if a > 0 else -1
        right = int(x[b]) if b < x.size else -1
        assert (O.stencil(x[a:b], left, right) == full[a:b]).all()
    assert (O.stencil_mt(x, 4) == full).all()


def test_batched_oracle_edges():
    # H at the end of one string followed by L at the start of the next: both FFFD
    x = O.u16([0x41, 0xD800, 0xDC00, 0x42])
    assert O.fix_batched(x, [0, 2, 4]).tolist() == [0x41, 0xFFFD, 0xFFFD, 0x42]
    assert O.fix_batched(x, [0, 4]).tolist() == x.tolist()
    assert O.fix_batched(x, [1, 1, 3]).tolist() == [0x41, 0xD800, 0xDC00, 0x42]
    with pytest.raises(ValueError):
        O.fix_batched(x, [0, 3, 2])


def test_unpaired_offsets_kat():
    # proj/tests/test_surrogate.cpp:122-128
    x = [0x0041, 0xDC00, 0x0042, 0xD800]
    assert O.unpaired_offsets(x) == [1, 3]
    assert O.unpaired_offsets(x, 1) == [1]


@pytest.mark.parametrize("cfg", [0, 1, 2, 4])
def test_generator_windows_consistent(cfg):
    total = 200_000
    full = O.gen_config(cfg, total, shard_len=50_000 if cfg == 4 else 0)
    for first, count in ((0, 1), (4095, 2), (4096, 5000), (123_457, 50_001), (total - 3, 3)):
        w = O.gen_config(cfg, total, first=first, count=count, shard_len=50_000 if cfg == 4 else 0)
        assert (w == full[first:first + count]).all()


def test_generator_statistics():
    x = O.gen_config(0, 1 << 22)
    ascii_ = ((x >= 0x20) & (x <= 0x7E)).mean()
    assert 0.62 < ascii_ < 0.70   # 70% of characters; pairs take 2 units
    y = O.stencil(x)
    assert 0.005 < (x != y).mean() < 0.02
    c1 = O.gen_config(1, 1 << 22)
    h = ((c1 & 0xFC00) == 0xD800).mean()
    assert abs(h - 1 / 64) < 0.001
    c2 = O.gen_config(2, 1 << 22)
    assert 0.6 < ((c2 & 0xF800) == 0xD800).mean() < 0.7   # ~2/3 of units are pair halves
    for b in (256, 2048, 4096, 65536):                    # boundary patterns present
        k = (b // 256) % 5
        if k == 0:
            assert (c2[b - 1] & 0xFC00) == 0xD800 and (c2[b] & 0xFC00) == 0xDC00
    data, offs = O.gen_c3(4096)
    lens = np.diff(offs)
    assert lens.min() >= 1 and lens.max() <= 4095
    assert 300 < lens.mean() < 700
    out = O.fix_batched(data, offs)
    bad_strings = sum(int((data[a:b] != out[a:b]).any()) for a, b in zip(offs[:-1], offs[1:]))
    assert 0.15 < bad_strings / 4096 < 0.3


def test_c4_shard_edges():
    total, L = 4 * 65536, 65536
    x = O.gen_config(4, total, seed=4, shard_len=L)
    for k in range(1, 4):
        b = k * L
        kind = k % 5
        if kind == 0:
            assert (x[b - 1] & 0xFC00) == 0xD800 and (x[b] & 0xFC00) == 0xDC00
        if kind == 1:
            assert (x[b - 1] & 0xFC00) == 0xD800 and x[b] == 0x41
        if kind == 2:
            assert x[b - 1] == 0x42 and (x[b] & 0xFC00) == 0xDC00
        if kind == 3:
            assert (x[b - 1] & 0xFC00) == 0xD800 and (x[b] & 0xFC00) == 0xD800 and (x[b + 1] & 0xFC00) == 0xDC00


@pytest.mark.skipif(O.ref() is None, reason="oracle/_ref not built (reference tree absent)")
def test_oracle_vs_reference_build():
    rng = np.random.default_rng(3)
    kernels = O.ref_available_kernels()
    for t in range(400):
        n = int(rng.integers(0, 700))
        x = rng.choice(ALPHABET, n) if t % 2 else rng.integers(0, 65536, n).astype(np.uint16)
        e = O.fix_scalar(x)
        for k in kernels:
            assert (O.ref_to_well_formed(x, k) == e).all(), k
            assert (O.ref_to_well_formed(x, k, in_place=True) == e).all(), k
    for seed in range(10):
        a = O.ref_generate(10_000, 0.05, 0.05, seed)
        b = np.empty_like(a)
        O.ref().ref_generate(10_000, 0.05, 0.05, seed, O._p16(b))
        assert (a == b).all()


def test_in_place_race_is_benign_exhaustively():
    """SURVEY.md §0 fact 3, checked over every 5-unit class window: when a
    neighbour reads a unit either before or after that unit's own in-place
    rewrite (in any combination), every decision is unchanged. Classes:
    N (non-surrogate), H, L; edges are N."""
    import itertools

    vals = {"N": 0x41, "H": 0xD800, "L": 0xDC00}
    for w in itertools.product("NHL", repeat=5):
        x = np.array([vals[c] for c in w], np.uint16)
        truth = O.stencil(x)
        # every subset of units already rewritten when the neighbours look
        for mask in range(32):
            seen = x.copy()
            for i in range(5):
                if mask >> i & 1:
                    seen[i] = truth[i]
            # decisions of the three interior units from the mixed view
            for i in (1, 2, 3):
                u = int(x[i])
                prev_h = (int(seen[i - 1]) & 0xFC00) == 0xD800
                next_l = (int(seen[i + 1]) & 0xFC00) == 0xDC00
                r = u
                if (u & 0xFC00) == 0xD800 and not next_l:
                    r = 0xFFFD
                if (u & 0xFC00) == 0xDC00 and not prev_h:
                    r = 0xFFFD
                assert r == truth[i], (w, mask, i)
