"""Regenerate tests/golden/ from the reference's OWN compiled code.

Run in the dev container (needs /root/reference, builds oracle/_ref):

    python tests/golden/make_golden.py

Every expected output below is produced by the reference library
(oracle/_ref/libutf16mend_ref.so, built by oracle/Makefile from
/root/reference/proj/src), through its kernels and its test helpers:
  * mixed sample                 proj/tests/test_helpers.hpp:21-37
  * reference_fix stencil        proj/tests/test_helpers.hpp:42-53
  * boundary alphabet sweeps     proj/tests/test_helpers.hpp:103-133
  * fix_scalar examples          proj/tests/test_surrogate.cpp:57-66
  * generate() KATs              proj/src/datagen.cpp:44-74 with the seeds of
                                 proj/tests/test_bitmask_kernel.cpp:122-134,
                                 proj/tests/test_bytesplit_kernel.cpp:138-145,
                                 proj/tests/test_generic_kernel.cpp:148-157
  * fuzz configs                 proj/tests/acceptance.cpp:37-45
The GPU tests never read /root/reference: they load these fixtures.
"""
from __future__ import annotations

import hashlib
import itertools
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
FUZZ_MISMATCH = [0.0, 0.001, 0.01, 0.5]   # acceptance.cpp:37
FUZZ_PAIR = [0.0, 0.001, 0.02, 0.3]       # acceptance.cpp:38


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<u2").tobytes()).hexdigest()


def ref_fix(x: np.ndarray, kernel: str = "bitmask-emulated") -> np.ndarray:
    a = O.ref_to_well_formed(x, kernel)
    R = O.ref()
    b = np.empty_like(x)
    R.ref_reference_fix(O._p16(x), x.size, O._p16(b))
    assert (a == b).all()
    return a


def fuzz_cases(count: int):
    rng = np.random.default_rng(20240601)
    for i in range(count):
        n = int(rng.integers(0, 301))
        yield dict(n=n, pair=FUZZ_PAIR[(i // 4) % 4], mismatch=FUZZ_MISMATCH[i % 4], seed=0xF00D0000 + i)


def main() -> None:
    O.build(ref=True)
    R = O.ref()
    assert R is not None
    arrays: dict[str, np.ndarray] = {}
    meta: dict = {"generated_by": "tests/golden/make_golden.py", "reference_kernels": O.ref_available_kernels()}

    a = np.empty(31, np.uint16)
    b = np.empty(31, np.uint16)
    R.ref_mixed_sample(O._p16(a), O._p16(b))
    arrays["mixed_in"], arrays["mixed_expected"] = a, b
    alpha = np.empty(8, np.uint16)
    R.ref_boundary_alphabet(O._p16(alpha))
    arrays["boundary_alphabet"] = alpha

    ex = [[0x0048, 0x0069], [0xD800, 0x0041], [0xD83D, 0xDE0A], [0xDC00], [],
          [0xD800, 0xDC00, 0xDC00], [0x0041, 0xDC00, 0x0042, 0xD800]]
    meta["scalar_examples"] = [{"in": e, "out": [int(v) for v in ref_fix(O.u16(e))]} for e in ex]

    # exhaustive boundary sequences, length <= 4 stored, <= 5 hashed
    for maxlen, store in ((4, True), (5, False)):
        ins, outs, lens = [], [], []
        for L in range(maxlen + 1):
            for t in itertools.product(range(8), repeat=L):
                x = alpha[list(t)] if L else np.empty(0, np.uint16)
                ins.append(x)
                outs.append(ref_fix(x))
                lens.append(L)
        cin, cout = np.concatenate(ins), np.concatenate(outs)
        if store:
            arrays["boundary4_in"], arrays["boundary4_out"] = cin, cout
            arrays["boundary4_lens"] = np.asarray(lens, np.int32)
        meta[f"boundary{maxlen}_sha_in"], meta[f"boundary{maxlen}_sha_out"] = sha(cin), sha(cout)
        meta[f"boundary{maxlen}_count"] = len(lens)

    kats = []
    for n, pair, mis, seed in ((1_000_000, 0.001, 0.0, 3), (1_000_000, 0.001, 0.0, 4),
                               (4000, 0.05, 0.0, 77), (1_000_000, 0.001, 0.001, 6),
                               (1_000_000, 0.3, 0.5, 11)):
        x = np.empty(n, np.uint16)
        R.ref_generate(n, pair, mis, seed, O._p16(x))
        y = ref_fix(x)
        kats.append(dict(n=n, pair=pair, mismatch=mis, seed=seed, sha_in=sha(x), sha_out=sha(y),
                         changed=int((x != y).sum()), head_in=[int(v) for v in x[:16]]))
    meta["generate_kats"] = kats

    cases = list(fuzz_cases(3000))
    ins, outs = [], []
    for c in cases:
        x = np.empty(c["n"], np.uint16)
        R.ref_generate(c["n"], c["pair"], c["mismatch"], c["seed"], O._p16(x))
        ins.append(x)
        outs.append(ref_fix(x, "bitmask" if "bitmask" in meta["reference_kernels"] else "generic8"))
    arrays["fuzz_n"] = np.asarray([c["n"] for c in cases], np.int32)
    meta["fuzz"] = {"count": len(cases), "seed_base": 0xF00D0000, "pair_rates": FUZZ_PAIR,
                    "mismatch_rates": FUZZ_MISMATCH, "sha_in": sha(np.concatenate(ins)),
                    "sha_out": sha(np.concatenate(outs))}

    np.savez_compressed(os.path.join(OUT, "golden.npz"), **arrays)
    with open(os.path.join(OUT, "golden.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
