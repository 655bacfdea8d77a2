"""TEST INFRASTRUCTURE — numpy/ctypes front end for the CPU oracle.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may
import this package, and only as the checker or the timed CPU baseline. The
product (``paper_2601_06349_b200``) never imports it.

* ``liboracle.so`` — this repo's C restatement (``oracle.c``; citations there).
* ``_ref/libutf16mend_ref.so`` — the reference's own sources compiled by
  ``oracle/Makefile`` (present when built in the dev container; it travels to
  the GPU box as a built artefact). ``ref()`` returns None when absent.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(HERE, "liboracle.so")
_REF = os.path.join(HERE, "_ref", "libutf16mend_ref.so")

_u16p = ctypes.POINTER(ctypes.c_uint16)
_i64p = ctypes.POINTER(ctypes.c_int64)
_u64p = ctypes.POINTER(ctypes.c_uint64)
_sz = ctypes.c_size_t

_lib = None
_ref = None


def build(ref: bool | None = None) -> None:
    """Compile liboracle.so (and oracle/_ref when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)
    if ref is None:
        ref = os.path.isdir("/root/reference/proj")
    if ref:
        subprocess.run(["make", "-s", "-C", HERE, "ref", "-j8"], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            build(ref=False)
        L = ctypes.CDLL(_LIB)
        L.or_fix_scalar.argtypes = [_u16p, _u16p, _sz]
        L.or_stencil.argtypes = [_u16p, _sz, _u16p]
        L.or_stencil_halo.argtypes = [_u16p, _sz, _u16p, ctypes.c_int32, ctypes.c_int32]
        L.or_fix_batched.argtypes = [_u16p, _i64p, _sz, _u16p]
        L.or_fix_batched.restype = ctypes.c_int
        L.or_unpaired_offsets.argtypes = [_u16p, _sz, _sz, _u64p]
        L.or_unpaired_offsets.restype = _sz
        L.or_is_well_formed.argtypes = [_u16p, _sz]
        L.or_is_well_formed.restype = ctypes.c_int
        L.or_stencil_mt.argtypes = [_u16p, _sz, _u16p, ctypes.c_int]
        L.or_ref_generate.argtypes = [_sz, ctypes.c_double, ctypes.c_double, ctypes.c_uint64, _u16p]
        L.or_gen_config.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                    ctypes.c_uint64, ctypes.c_uint64, _u16p]
        L.or_gen_config.restype = ctypes.c_int
        L.or_gen_c3_offsets.argtypes = [ctypes.c_uint64, _sz, _i64p]
        L.or_gen_c3_content.argtypes = [ctypes.c_uint64, _sz, _i64p, _u16p]
        _lib = L
    return _lib


def ref():
    """The reference's own compiled code, or None if oracle/_ref was not built."""
    global _ref
    if _ref is None:
        if not os.path.exists(_REF):
            return None
        R = ctypes.CDLL(_REF)
        R.ref_to_well_formed.argtypes = [_u16p, _sz, _u16p, ctypes.c_char_p]
        R.ref_to_well_formed_in_place.argtypes = [_u16p, _sz, ctypes.c_char_p]
        R.ref_to_well_formed_mt.argtypes = [_u16p, _sz, _u16p, ctypes.c_int, ctypes.c_char_p]
        R.ref_reference_fix.argtypes = [_u16p, _sz, _u16p]
        R.ref_fix_scalar.argtypes = [_u16p, _sz, _u16p]
        R.ref_generate.argtypes = [_sz, ctypes.c_double, ctypes.c_double, ctypes.c_uint64, _u16p]
        R.ref_mixed_sample.argtypes = [_u16p, _u16p]
        R.ref_boundary_alphabet.argtypes = [_u16p]
        R.ref_unpaired_surrogate_offsets.argtypes = [_u16p, _sz, _sz, _u64p]
        R.ref_unpaired_surrogate_offsets.restype = _sz
        R.ref_default_kernel.argtypes = [ctypes.c_char_p, _sz]
        R.ref_available_kernels.argtypes = [ctypes.c_char_p, _sz]
        R.ref_parse_csv.argtypes = [ctypes.c_char_p, ctypes.c_char_p, _sz]
        _ref = R
    return _ref


def _p16(a: np.ndarray):
    assert a.dtype == np.uint16 and a.flags.c_contiguous
    return a.ctypes.data_as(_u16p)


def _p64(a: np.ndarray):
    assert a.dtype == np.int64 and a.flags.c_contiguous
    return a.ctypes.data_as(_i64p)


def u16(seq) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(seq, dtype=np.uint16))


# ---- repair -----------------------------------------------------------------
def fix_scalar(x) -> np.ndarray:
    x = u16(x)
    out = np.empty_like(x)
    lib().or_fix_scalar(_p16(out), _p16(x), x.size)
    return out


def stencil(x, left: int = -1, right: int = -1) -> np.ndarray:
    x = u16(x)
    out = np.empty_like(x)
    lib().or_stencil_halo(_p16(x), x.size, _p16(out), left, right)
    return out


def stencil_mt(x, threads: int | None = None) -> np.ndarray:
    x = u16(x)
    out = np.empty_like(x)
    lib().or_stencil_mt(_p16(x), x.size, _p16(out), threads or os.cpu_count() or 1)
    return out


def fix_batched(x, offsets) -> np.ndarray:
    x = u16(x)
    offsets = np.ascontiguousarray(np.asarray(offsets, dtype=np.int64))
    out = x.copy()
    rc = lib().or_fix_batched(_p16(x), _p64(offsets), offsets.size - 1, _p16(out))
    if rc != 0:
        raise ValueError("offsets must be non-decreasing and non-negative")
    return out


def unpaired_offsets(x, limit: int = 2**64 - 1) -> list[int]:
    x = u16(x)
    limit = min(limit, x.size)
    buf = np.empty(max(limit, 1), dtype=np.uint64)
    k = lib().or_unpaired_offsets(_p16(x), x.size, limit, buf.ctypes.data_as(_u64p))
    return [int(v) for v in buf[:k]]


def is_well_formed(x) -> bool:
    x = u16(x)
    return bool(lib().or_is_well_formed(_p16(x), x.size))


# ---- generators -------------------------------------------------------------
def ref_generate(n: int, pair_pct: float = 0.0, mismatch_pct: float = 0.0, seed: int = 0) -> np.ndarray:
    """Restatement of the reference's generate() (proj/src/datagen.cpp:44-74)."""
    out = np.empty(n, dtype=np.uint16)
    lib().or_ref_generate(n, pair_pct, mismatch_pct, seed, _p16(out))
    return out


def gen_config(cfg: int, total: int, seed: int | None = None, first: int = 0, count: int | None = None,
               shard_len: int = 0) -> np.ndarray:
    seed = cfg if seed is None else seed
    count = total - first if count is None else count
    out = np.empty(count, dtype=np.uint16)
    rc = lib().or_gen_config(cfg, seed, total, shard_len, first, count, _p16(out))
    if rc != 0:
        raise ValueError("bad generator arguments")
    return out


def gen_c3(num_strings: int, seed: int = 3) -> tuple[np.ndarray, np.ndarray]:
    offsets = np.empty(num_strings + 1, dtype=np.int64)
    lib().or_gen_c3_offsets(seed, num_strings, _p64(offsets))
    data = np.empty(int(offsets[-1]), dtype=np.uint16)
    lib().or_gen_c3_content(seed, num_strings, _p64(offsets), _p16(data))
    return data, offsets


# ---- reference (oracle/_ref) helpers ---------------------------------------
def ref_to_well_formed(x, kernel: str | None = None, in_place: bool = False) -> np.ndarray:
    R = ref()
    if R is None:
        raise RuntimeError("oracle/_ref not built")
    x = u16(x).copy()
    k = kernel.encode() if kernel else None
    if in_place:
        rc = R.ref_to_well_formed_in_place(_p16(x), x.size, k)
        out = x
    else:
        out = np.empty_like(x)
        rc = R.ref_to_well_formed(_p16(x), x.size, _p16(out), k)
    if rc != 0:
        raise ValueError(f"reference rejected kernel {kernel!r} (rc={rc})")
    return out


def ref_default_kernel() -> str:
    buf = ctypes.create_string_buffer(64)
    ref().ref_default_kernel(buf, 64)
    return buf.value.decode()


def ref_available_kernels() -> list[str]:
    buf = ctypes.create_string_buffer(512)
    ref().ref_available_kernels(buf, 512)
    return buf.value.decode().split(",")


def ref_parse_csv(path: str) -> list[tuple]:
    """Parse a CSV report with the reference's own parse_csv
    (proj/src/bench.cpp:172-203): [(impl, units, bytes, best_ns, mean_ns,
    gbps, margin_pct)], floats exact. Raises ValueError when it throws."""
    buf = ctypes.create_string_buffer(1 << 20)
    k = ref().ref_parse_csv(path.encode(), buf, 1 << 20)
    if k == -1:
        raise FileNotFoundError(path)
    if k < 0:
        raise ValueError("reference parse_csv threw")
    rows = []
    for line in buf.value.decode().splitlines():
        f = line.split("|")
        rows.append((f[0], int(f[1]), int(f[2]), int(f[3]), float(f[4]), float(f[5]), float(f[6])))
    return rows
