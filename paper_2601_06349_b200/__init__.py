"""utf16mend-b200: B200-native repair of ill-formed UTF-16 (sm_100a).

Python mirror of the reference's bindings (proj/python/utf16mend/__init__.py,
proj/bindings/module.cpp) with the same names, argument meaning and error
behaviour, plus zero-copy entry points for torch CUDA tensors. Every call
goes through the C ABI of ``libu16m.so`` (include/u16m.h) and runs on the
GPU; there is no CPU fallback — importing this package without the built
library raises ImportError, and calling it without a CUDA device raises
RuntimeError.

Reference-compatible names (bytes are raw UTF-16LE code units):
    fix_utf16le, fix_str, is_well_formed_utf16le, is_well_formed_str,
    unpaired_surrogate_offsets, generate_utf16le, available_kernels,
    default_kernel
Many strings in one GPU call (batched form, no reference counterpart):
    fix_utf16le_batch, fix_str_batch
Device-tensor API (int16/uint16 CUDA tensors, stream-ordered, no copies):
    to_well_formed, to_well_formed_, to_well_formed_halo,
    to_well_formed_batched, count_unpaired, unpaired_offsets_device
"""
from __future__ import annotations

from ._lib import (  # noqa: F401
    U16MError,
    api_version,
    available_kernels,
    backend,
    count_unpaired,
    default_kernel,
    fix_str,
    fix_str_batch,
    fix_utf16_bytes,
    fix_utf16le,
    fix_utf16le_batch,
    generate_utf16le,
    is_well_formed_str,
    is_well_formed_utf16le,
    launch_count,
    lib_path,
    to_well_formed,
    to_well_formed_,
    to_well_formed_batched,
    to_well_formed_bytes,
    to_well_formed_halo,
    to_well_formed_part,
    to_well_formed_sharded,
    unpaired_offsets_device,
    unpaired_surrogate_offsets,
)

__all__ = [
    "available_kernels",
    "backend",
    "default_kernel",
    "fix_str",
    "fix_str_batch",
    "fix_utf16le_batch",
    "fix_utf16le",
    "fix_utf16_bytes",
    "to_well_formed_bytes",
    "generate_utf16le",
    "is_well_formed_str",
    "is_well_formed_utf16le",
    "unpaired_surrogate_offsets",
    "to_well_formed",
    "to_well_formed_",
    "to_well_formed_halo",
    "to_well_formed_part",
    "to_well_formed_batched",
    "to_well_formed_sharded",
    "count_unpaired",
    "unpaired_offsets_device",
]
