"""ctypes binding of libu16m.so (include/u16m.h, include/u16m_datagen.h).

Mirrors the reference's pybind11 module (proj/bindings/module.cpp:51-107):
same function names, same argument meaning, and the same errors —
``ValueError`` for an odd byte length (module.cpp:25-26) and for an unknown
kernel name (module.cpp:45), ``RuntimeError`` for device/CUDA failures. The
only route to compute is the C ABI; without the built library this module
raises ImportError (no eager/CPU fallback exists).
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
# U16M_LIBRARY: load another build of the same ABI (same-box A/B of kernel
# versions, scripts/ab_lib.sh); the default is the in-tree build.
_LIB_PATH = os.environ.get("U16M_LIBRARY") or os.path.join(_PKG, "libu16m.so")

if not os.path.exists(_LIB_PATH):
    raise ImportError(
        f"{_LIB_PATH} is missing: build it with `python paper_2601_06349_b200/_build.py` "
        "(or __graft_entry__.build()). There is no CPU fallback.")

_L = ctypes.CDLL(_LIB_PATH)
_u16p = ctypes.c_void_p
_vp = ctypes.c_void_p
_sz = ctypes.c_size_t
_st = ctypes.c_int

_L.u16m_to_well_formed.argtypes = [_u16p, _sz, _u16p, _vp]
_L.u16m_to_well_formed_in_place.argtypes = [_u16p, _sz, _vp]
_L.u16m_to_well_formed_batched.argtypes = [_u16p, _vp, _sz, _u16p, _vp]
_L.u16m_to_well_formed_batched_n.argtypes = [_u16p, _sz, _vp, _sz, _u16p, _vp]
_L.u16m_to_well_formed_halo.argtypes = [_u16p, _sz, _u16p, ctypes.c_int32, ctypes.c_int32, _vp]
_L.u16m_to_well_formed_halo_ptr.argtypes = [_u16p, _sz, _u16p, _vp, _vp, _vp]
_L.u16m_to_well_formed_part.argtypes = [_u16p, _sz, _u16p, _vp, _vp, ctypes.c_int, _vp]
_L.u16m_to_well_formed_sharded.argtypes = [ctypes.c_int, _vp, _vp, _vp, _vp]
_L.u16m_to_well_formed_host.argtypes = [_u16p, _sz, _u16p]
_L.u16m_count_unpaired.argtypes = [_u16p, _sz, _vp, _vp]
_L.u16m_unpaired_offsets.argtypes = [_u16p, _sz, _sz, _vp, _vp, _vp]
_L.u16m_status_string.argtypes = [_st]
_L.u16m_status_string.restype = ctypes.c_char_p
_L.u16m_last_error.restype = ctypes.c_char_p
_L.u16m_api_version.restype = ctypes.c_int
_L.u16m_launch_count.restype = ctypes.c_ulonglong
_L.u16m_gen_config.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                               ctypes.c_uint64, ctypes.c_uint64, _u16p, _vp]
_L.u16m_gen_c3_offsets.argtypes = [ctypes.c_uint64, _sz, _vp, ctypes.POINTER(ctypes.c_uint64)]
_L.u16m_gen_c3_content.argtypes = [ctypes.c_uint64, _sz, _vp, _u16p, _vp]
_L.u16m_generate_reference_mix.argtypes = [_sz, ctypes.c_double, ctypes.c_double, ctypes.c_uint64, _u16p]
_L.u16m_l2_flush.argtypes = [_vp, _sz, _vp]
_L.u16m_fix_utf16_bytes.argtypes = [_vp, _sz, _vp, ctypes.c_int, _vp, _vp]
_L.u16m_fix_utf16_bytes_host.argtypes = [_vp, _sz, _vp, ctypes.c_int, ctypes.POINTER(ctypes.c_ulonglong)]
_L.u16m_unpaired_offsets_host.argtypes = [_vp, _sz, _sz, _vp, ctypes.POINTER(ctypes.c_size_t)]
for _f in ("u16m_to_well_formed", "u16m_to_well_formed_in_place", "u16m_to_well_formed_batched",
           "u16m_to_well_formed_batched_n",
           "u16m_to_well_formed_halo", "u16m_to_well_formed_halo_ptr", "u16m_to_well_formed_sharded",
           "u16m_to_well_formed_host", "u16m_to_well_formed_part", "u16m_count_unpaired", "u16m_unpaired_offsets",
           "u16m_gen_config", "u16m_gen_c3_offsets", "u16m_gen_c3_content",
           "u16m_generate_reference_mix", "u16m_l2_flush", "u16m_fix_utf16_bytes",
           "u16m_fix_utf16_bytes_host", "u16m_unpaired_offsets_host"):
    getattr(_L, _f).restype = _st

OK, INVALID, ALIAS, NOT_DEVICE, CUDA, MISALIGNED, NO_DEVICE = range(7)

_L.u16m_kernel_names.argtypes = [ctypes.c_char_p, _sz]
_L.u16m_kernel_names.restype = ctypes.c_int
_L.u16m_default_kernel_name.argtypes = [ctypes.c_char_p, _sz]
_L.u16m_default_kernel_name.restype = ctypes.c_int
_L.u16m_select_kernel.argtypes = [ctypes.c_char_p, ctypes.c_char_p, _sz]
_L.u16m_select_kernel.restype = _st
_L.u16m_to_well_formed_host_multi.argtypes = [_u16p, _sz, _u16p, ctypes.c_int, _vp]
_L.u16m_to_well_formed_host_multi.restype = _st
_L.u16m_fix_utf16_bytes_host_multi.argtypes = [_vp, _sz, _vp, ctypes.c_int, ctypes.POINTER(ctypes.c_ulonglong),
                                               ctypes.c_int, _vp]
_L.u16m_fix_utf16_bytes_host_multi.restype = _st
_L.u16m_unpaired_offsets_bytes_host.argtypes = [_vp, _sz, ctypes.c_int, _sz, _vp, ctypes.POINTER(ctypes.c_size_t)]
_L.u16m_unpaired_offsets_bytes_host.restype = _st


class U16MError(RuntimeError):
    def __init__(self, status: int, detail: str):
        self.status = status
        super().__init__(f"{_L.u16m_status_string(status).decode()}: {detail}")


def _check(st: int) -> None:
    if st == OK:
        return
    detail = (_L.u16m_last_error() or b"").decode()
    msg = f"{_L.u16m_status_string(st).decode()}: {detail}"
    if st in (INVALID, ALIAS, MISALIGNED, NOT_DEVICE):
        raise ValueError(msg)
    raise U16MError(st, detail)


def lib_path() -> str:
    return _LIB_PATH


def api_version() -> int:
    return int(_L.u16m_api_version())


def launch_count() -> int:
    return int(_L.u16m_launch_count())


def raw():
    """The ctypes handle (bench / tests)."""
    return _L


# ---- device tensor API -------------------------------------------------------
def _units(t, name: str) -> torch.Tensor:
    """Validate a device buffer of code units. Any DLPack producer (CuPy,
    JAX, NumPy-on-device libraries, ...) is accepted zero-copy through
    torch.from_dlpack; the returned tensor aliases its memory."""
    if not isinstance(t, torch.Tensor) and hasattr(t, "__dlpack__"):
        t = torch.from_dlpack(t)
    if not isinstance(t, torch.Tensor):
        raise ValueError(f"{name} must be a CUDA tensor or a DLPack-exporting device array")
    if t.dtype not in (torch.int16, torch.uint16):
        raise ValueError(f"{name} must be an int16/uint16 tensor of UTF-16 code units")
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (use fix_utf16le for host bytes)")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t


def _stream(t: torch.Tensor, stream) -> int:
    if stream is None:
        return torch.cuda.current_stream(t.device).cuda_stream
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def to_well_formed(x: torch.Tensor, out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """out = repair(x) on the GPU (reference to_well_formed, driver.hpp:64-65)."""
    x = _units(x, "x")
    if out is None:
        out = torch.empty_like(x)
    out = _units(out, "out")
    if out.numel() != x.numel():
        raise ValueError("to_well_formed: input and output lengths differ")
    with torch.cuda.device(x.device):
        _check(_L.u16m_to_well_formed(x.data_ptr(), x.numel(), out.data_ptr(), _stream(x, stream)))
    return out


def to_well_formed_(x: torch.Tensor, stream=None) -> torch.Tensor:
    """In-place repair (reference to_well_formed_in_place, driver.hpp:68-69)."""
    x = _units(x, "x")
    with torch.cuda.device(x.device):
        _check(_L.u16m_to_well_formed_in_place(x.data_ptr(), x.numel(), _stream(x, stream)))
    return x


def to_well_formed_halo(x: torch.Tensor, out: Optional[torch.Tensor], left: int, right: int,
                        stream=None) -> torch.Tensor:
    """Repair one contiguous shard of a larger logical buffer; left/right are the
    neighbouring units (-1 at the logical buffer's ends). out=None: in place."""
    x = _units(x, "x")
    out = x if out is None else _units(out, "out")
    with torch.cuda.device(x.device):
        _check(_L.u16m_to_well_formed_halo(x.data_ptr(), x.numel(), out.data_ptr(), int(left), int(right),
                                           _stream(x, stream)))
    return out


PART_ALL, PART_EDGES, PART_INTERIOR = 0, 1, 2


def to_well_formed_part(x: torch.Tensor, out: Optional[torch.Tensor], part: int, left_ptr: int = 0,
                        right_ptr: int = 0, stream=None) -> torch.Tensor:
    """One part (PART_EDGES / PART_INTERIOR / PART_ALL) of a shard repair; halo
    units are read on the device from left_ptr / right_ptr (0 = buffer end)."""
    x = _units(x, "x")
    out = x if out is None else _units(out, "out")
    with torch.cuda.device(x.device):
        _check(_L.u16m_to_well_formed_part(x.data_ptr(), x.numel(), out.data_ptr(), left_ptr or None,
                                           right_ptr or None, int(part), _stream(x, stream)))
    return out


def to_well_formed_batched(data: torch.Tensor, offsets: torch.Tensor, out: Optional[torch.Tensor] = None,
                           stream=None) -> torch.Tensor:
    """Repair every string [offsets[s], offsets[s+1]) independently.

    Stream-ordered, no host sync. Units of `out` outside [offsets[0],
    offsets[-1]) are not written: with out=None (a clone of `data`) they hold
    the input, as in the host and C++ forms, which copy them; a caller-supplied
    `out` keeps whatever it held there."""
    data = _units(data, "data")
    if not isinstance(offsets, torch.Tensor) and hasattr(offsets, "__dlpack__"):
        offsets = torch.from_dlpack(offsets)
    if offsets.dtype != torch.int64 or not offsets.is_cuda or not offsets.is_contiguous():
        raise ValueError("offsets must be a contiguous int64 CUDA tensor")
    if offsets.numel() < 1:
        raise ValueError("offsets must have num_strings + 1 entries")
    if out is None:
        out = data.clone()
    out = _units(out, "out")
    if out.numel() != data.numel():
        raise ValueError("to_well_formed_batched: input and output lengths differ")
    with torch.cuda.device(data.device):
        _check(_L.u16m_to_well_formed_batched_n(data.data_ptr(), data.numel(), offsets.data_ptr(),
                                                offsets.numel() - 1, out.data_ptr(), _stream(data, stream)))
    return out


def to_well_formed_sharded(shards: Sequence[torch.Tensor], outs: Optional[Sequence[torch.Tensor]] = None):
    """One logical buffer = concatenation of `shards` (any CUDA devices of this
    process). outs=None: in place. Synchronous."""
    shards = [_units(s, "shard") for s in shards]
    outs = shards if outs is None else [_units(o, "out") for o in outs]
    n = len(shards)
    if len(outs) != n or any(o.numel() != s.numel() for o, s in zip(outs, shards)):
        raise ValueError("outs must match shards")
    for s in shards:
        torch.cuda.current_stream(s.device).synchronize()
    dev = (ctypes.c_int * n)(*[s.device.index for s in shards])
    ins = (ctypes.c_void_p * n)(*[s.data_ptr() for s in shards])
    lens = (ctypes.c_size_t * n)(*[s.numel() for s in shards])
    ous = (ctypes.c_void_p * n)(*[o.data_ptr() for o in outs])
    _check(_L.u16m_to_well_formed_sharded(n, ctypes.addressof(dev), ctypes.addressof(ins),
                                          ctypes.addressof(lens), ctypes.addressof(ous)))
    return list(outs)


def count_unpaired(x: torch.Tensor, stream=None) -> int:
    """Number of units repair would rewrite (0 <=> well-formed). Synchronises."""
    x = _units(x, "x")
    cnt = torch.zeros(1, dtype=torch.int64, device=x.device)
    with torch.cuda.device(x.device):
        _check(_L.u16m_count_unpaired(x.data_ptr(), x.numel(), cnt.data_ptr(), _stream(x, stream)))
    return int(cnt.item())


def unpaired_offsets_device(x: torch.Tensor, limit: Optional[int] = None, stream=None) -> torch.Tensor:
    """Ascending offsets (int64 CUDA tensor) of the units repair would rewrite."""
    x = _units(x, "x")
    cap = x.numel() if limit is None else max(0, min(int(limit), x.numel()))
    offs = torch.empty(max(cap, 1), dtype=torch.int64, device=x.device)
    cnt = torch.zeros(1, dtype=torch.int64, device=x.device)
    with torch.cuda.device(x.device):
        _check(_L.u16m_unpaired_offsets(x.data_ptr(), x.numel(), cap, offs.data_ptr(), cnt.data_ptr(),
                                        _stream(x, stream)))
    return offs[: int(cnt.item())]


# ---- reference-compatible bytes API (proj/bindings/module.cpp) ---------------
def _kernel_from_name(kernel: Optional[str]) -> None:
    """The reference's kernel validation (module.cpp:42-47 + driver.cpp:71-86):
    an unknown name, or an override this host does not support, raises
    ValueError with the reference's message. Every kernel id is served by the
    one sm_100a path."""
    if kernel is None:
        return
    buf = ctypes.create_string_buffer(64)
    if _L.u16m_select_kernel(kernel.encode(), buf, 64) != OK:
        raise ValueError((_L.u16m_last_error() or b"").decode())


def _check_bytes(data) -> memoryview:
    mv = memoryview(data).cast("B")
    if mv.nbytes % 2 != 0:
        raise ValueError("UTF-16 byte string must have an even length")
    return mv


def fix_utf16le(data, kernel: Optional[str] = None) -> bytes:
    """Return `data` (raw UTF-16LE code units) with every unpaired surrogate
    replaced by U+FFFD (module.cpp:54-64). Host memory is staged through the
    visible GPUs by u16m_to_well_formed_host_multi (the call behind the C++
    to_well_formed on host spans)."""
    mv = _check_bytes(data)
    _kernel_from_name(kernel)
    n = mv.nbytes // 2
    if n == 0:
        return b""
    src = _host_ptr(mv)                         # read in place, no Python-side copy
    out, addr = _new_bytes(mv.nbytes)
    _check(_L.u16m_to_well_formed_host_multi(src.ctypes.data, n, addr, 0, None))
    return out


def fix_str(text: str, kernel: Optional[str] = None) -> str:
    """Return `text` with every unpaired surrogate replaced by U+FFFD
    (proj/python/utf16mend/__init__.py:24-31)."""
    data = text.encode("utf-16-le", "surrogatepass")
    return fix_utf16le(data, kernel).decode("utf-16-le")


_L.u16m_to_well_formed_batched_host.argtypes = [_vp, _sz, _vp, _sz, _vp]
_L.u16m_to_well_formed_batched_host.restype = _st


def fix_utf16le_batch(items: Sequence) -> list[bytes]:
    """Repair many UTF-16LE byte strings with ONE GPU call (the batched form,
    u16m_to_well_formed_batched_host): each item is repaired on its own —
    units never pair across items — and the results come back in order.
    For many short strings this replaces one GPU round trip per string."""
    import itertools

    import numpy as np

    items = [b if type(b) is bytes else _check_bytes(b).tobytes() for b in items]
    if not items:
        return []
    ends = list(itertools.accumulate(map(len, items)))
    if any(e & 1 for e in ends):  # some item has an odd length
        for b in items:
            _check_bytes(b)
    total = ends[-1]
    if total == 0:
        return [b"" for _ in items]
    offsets = np.empty(len(items) + 1, dtype=np.int64)
    offsets[0] = 0
    offsets[1:] = ends
    offsets[1:] //= 2
    buf = bytearray().join(items)  # one contiguous, writable buffer
    addr = ctypes.addressof((ctypes.c_char * total).from_buffer(buf))
    _check(_L.u16m_to_well_formed_batched_host(addr, total // 2, offsets.ctypes.data, len(items), addr))
    raw = bytes(buf)
    return [raw[a:b] for a, b in zip(itertools.chain((0,), ends), ends)]


def fix_str_batch(texts: Sequence[str]) -> list[str]:
    """fix_str over many strings in one GPU call (see fix_utf16le_batch)."""
    out = fix_utf16le_batch([t.encode("utf-16-le", "surrogatepass") for t in texts])
    return [b.decode("utf-16-le") for b in out]


_PyBytes_FromStringAndSize = ctypes.pythonapi.PyBytes_FromStringAndSize
_PyBytes_FromStringAndSize.argtypes = [ctypes.c_void_p, ctypes.c_ssize_t]
_PyBytes_FromStringAndSize.restype = ctypes.py_object
_PyBytes_AsString = ctypes.pythonapi.PyBytes_AsString
_PyBytes_AsString.argtypes = [ctypes.py_object]
_PyBytes_AsString.restype = ctypes.c_void_p


def _new_bytes(nbytes: int):
    """A fresh, uninitialised `bytes` object and the address of its buffer, for
    the C ABI to write the result into before the object is returned (the
    reference's bindings also hand back bytes, module.cpp:54-64). Skips the
    zero-fill of a bytearray and the final bytes() copy — on a 512 MiB
    result those two passes cost 450 ms against 20 ms for the repair itself."""
    out = _PyBytes_FromStringAndSize(None, nbytes)
    return out, _PyBytes_AsString(out)


def _host_ptr(mv: memoryview):
    """A uint8 numpy view of the caller's bytes (zero-copy; `.ctypes.data` is
    the address the C ABI reads), copied only when not 2-byte aligned."""
    import numpy as np

    src = np.frombuffer(mv, dtype=np.uint8)
    return src.copy() if src.ctypes.data % 2 else src


def _host_offsets(data, limit: int) -> list[int]:
    """Chunked host-memory scan through the C ABI (u16m_unpaired_offsets_host):
    the bytes are read in place (no Python-side copy) and streamed to the GPU;
    the scan stops once `limit` offsets are found."""
    import numpy as np

    mv = _check_bytes(data)
    n = mv.nbytes // 2
    if n == 0 or limit <= 0:
        return []
    cap = min(int(limit), n)
    src = _host_ptr(mv)
    out = np.empty(cap, dtype=np.uint64)
    cnt = ctypes.c_size_t(0)
    _check(_L.u16m_unpaired_offsets_host(src.ctypes.data, n, cap, out.ctypes.data, ctypes.byref(cnt)))
    return out[: cnt.value].tolist()


def is_well_formed_utf16le(data) -> bool:
    """True if `data` contains no unpaired surrogate (module.cpp:66-70)."""
    return not _host_offsets(data, 1)


def is_well_formed_str(text: str) -> bool:
    return is_well_formed_utf16le(text.encode("utf-16-le", "surrogatepass"))


def unpaired_surrogate_offsets(data, limit: int = 2**64 - 1) -> list[int]:
    """Unit offsets that fixing would rewrite, capped at `limit` (module.cpp:72-78)."""
    return _host_offsets(data, limit)


def generate_utf16le(units: int, pair_pct: float = 0.0, mismatch_pct: float = 0.0, seed: int = 0) -> bytes:
    """Deterministic random UTF-16LE (the reference's generate(),
    proj/src/datagen.cpp:44-74, via module.cpp:80-93)."""
    if not (0.0 <= pair_pct <= 1.0 and 0.0 <= mismatch_pct <= 1.0):
        raise ValueError("pair_pct and mismatch_pct must be within [0, 1]")
    out = bytearray(2 * units)
    if units == 0:
        return bytes(out)
    buf = (ctypes.c_char * len(out)).from_buffer(out)
    _check(_L.u16m_generate_reference_mix(units, pair_pct, mismatch_pct, seed, ctypes.addressof(buf)))
    return bytes(out)


def fix_utf16_bytes(data, byte_order: str = "le") -> tuple[bytes, int]:
    """§8(f-3) codec fusion: repair raw UTF-16 bytes in their own byte order
    ("le" / "be") on the GPU without a swap pass; returns (bytes, number of
    replaced units). The CLI `fix` path (paper_2601_06349_b200/u16m); large
    inputs are spread over every visible GPU."""
    mv = _check_bytes(data)
    if byte_order not in ("le", "be"):
        raise ValueError("byte_order must be 'le' or 'be'")
    n = mv.nbytes // 2
    if n == 0:
        return b"", 0
    src = _host_ptr(mv)
    out, addr = _new_bytes(mv.nbytes)
    cnt = ctypes.c_ulonglong(0)
    _check(_L.u16m_fix_utf16_bytes_host(src.ctypes.data, n, addr, 1 if byte_order == "be" else 0,
                                        ctypes.byref(cnt)))
    return out, int(cnt.value)


def to_well_formed_bytes(x: torch.Tensor, out: Optional[torch.Tensor] = None, big_endian: bool = False,
                         count: bool = False, stream=None):
    """Device form of fix_utf16_bytes: x holds units as raw int16 words in the
    given byte order. Returns out, or (out, replacements) when count=True."""
    x = _units(x, "x")
    out = torch.empty_like(x) if out is None else _units(out, "out")
    cnt = torch.zeros(1, dtype=torch.int64, device=x.device) if count else None
    with torch.cuda.device(x.device):
        _check(_L.u16m_fix_utf16_bytes(x.data_ptr(), x.numel(), out.data_ptr(), 1 if big_endian else 0,
                                       cnt.data_ptr() if cnt is not None else None, _stream(x, stream)))
    return (out, int(cnt.item())) if count else out


def available_kernels() -> list[str]:
    """Names of every repair kernel selectable on this host (module.cpp:95-102),
    the reference's list; all of them run the one sm_100a path."""
    buf = ctypes.create_string_buffer(512)
    _L.u16m_kernel_names(buf, 512)
    return buf.value.decode().split(",")


def default_kernel() -> str:
    """Kernel the driver picks on this host (honours UTF16MEND_KERNEL), as the
    reference names it (module.cpp:104-106)."""
    buf = ctypes.create_string_buffer(64)
    _L.u16m_default_kernel_name(buf, 64)
    return buf.value.decode()


def backend() -> str:
    """The implementation every kernel name runs on."""
    return "cuda-sm100a"


# ---- device datagen (bench / tests) -----------------------------------------
def gen_config(cfg: int, total: int, seed: Optional[int] = None, first: int = 0, count: Optional[int] = None,
               shard_len: int = 0, out: Optional[torch.Tensor] = None, device="cuda", stream=None) -> torch.Tensor:
    seed = cfg if seed is None else seed
    count = total - first if count is None else count
    if out is None:
        out = torch.empty(count, dtype=torch.int16, device=device)
    with torch.cuda.device(out.device):
        _check(_L.u16m_gen_config(cfg, seed, total, shard_len, first, count, out.data_ptr(), _stream(out, stream)))
    return out


def gen_c3(num_strings: int, seed: int = 3, device="cuda") -> tuple[torch.Tensor, torch.Tensor]:
    offsets = torch.empty(num_strings + 1, dtype=torch.int64, device=device)
    total = ctypes.c_uint64(0)
    with torch.cuda.device(offsets.device):
        torch.cuda.current_stream().synchronize()
        _check(_L.u16m_gen_c3_offsets(seed, num_strings, offsets.data_ptr(), ctypes.byref(total)))
        data = torch.empty(int(total.value), dtype=torch.int16, device=device)
        _check(_L.u16m_gen_c3_content(seed, num_strings, offsets.data_ptr(), data.data_ptr(),
                                      _stream(data, None)))
    return data, offsets


def l2_flush(buf: torch.Tensor, stream=None) -> None:
    _check(_L.u16m_l2_flush(buf.data_ptr(), buf.numel() * buf.element_size(), _stream(buf, stream)))
