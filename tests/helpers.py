"""Shared helpers for the test-suite (test infrastructure)."""
from __future__ import annotations

import hashlib

import numpy as np

ALPHABET = np.array([0x0041, 0xD7FF, 0xD800, 0xDBFF, 0xDC00, 0xDFFF, 0xE000, 0xFFFD], np.uint16)


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<u2").tobytes()).hexdigest()


def boundary_sequences(max_len: int):
    """All sequences over the reference's boundary alphabet
    (proj/tests/test_helpers.hpp:103-133): length ascending, then
    lexicographic (the order tests/golden/make_golden.py hashed them in)."""
    import itertools

    for L in range(max_len + 1):
        for t in itertools.product(range(8), repeat=L):
            yield ALPHABET[list(t)] if L else np.empty(0, np.uint16)


def concat_with_offsets(seqs):
    lens = [len(s) for s in seqs]
    offsets = np.zeros(len(seqs) + 1, np.int64)
    offsets[1:] = np.cumsum(lens)
    data = np.concatenate(seqs) if seqs else np.empty(0, np.uint16)
    return data.astype(np.uint16), offsets


def fuzz_inputs(meta, arrays, gen):
    """Regenerate the reference acceptance fuzz inputs (acceptance.cpp:37-45)."""
    fz = meta["fuzz"]
    out = []
    for i, n in enumerate(arrays["fuzz_n"]):
        pair = fz["pair_rates"][(i // 4) % 4]
        mis = fz["mismatch_rates"][i % 4]
        out.append(gen(int(n), pair, mis, fz["seed_base"] + i))
    return out
