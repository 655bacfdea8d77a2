"""What does cuMemGetAddressRange report for a pointer inside a large tensor,
per torch allocator backend? (The length-less batched entry sizes its grid
from it.) Run with PYTORCH_CUDA_ALLOC_CONF unset / expandable_segments:True /
backend:cudaMallocAsync. Then checks the length-less entry on a 600 MiB
string set starting 1 MiB into the tensor."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
from paper_2601_06349_b200 import _lib  # noqa: E402

cuda = ctypes.CDLL("libcuda.so.1")
cuda.cuMemGetAddressRange_v2.argtypes = [ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_size_t), ctypes.c_uint64]
cuda.cuPointerGetAttribute.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_uint64]
conf = os.environ.get("PYTORCH_CUDA_ALLOC_CONF", "default")
n = 300 << 20  # units (600 MiB)
t = torch.empty(n + (1 << 20), dtype=torch.int16, device="cuda")
p = t.data_ptr() + (1 << 20)
base, size = ctypes.c_uint64(0), ctypes.c_size_t(0)
r = cuda.cuMemGetAddressRange_v2(ctypes.byref(base), ctypes.byref(size), p)
after = (base.value + size.value - p) // 2 if r == 0 else 0
cuda.cuMemRetainAllocationHandle.argtypes = [ctypes.POINTER(ctypes.c_uint64), ctypes.c_void_p]
cuda.cuMemRelease.argtypes = [ctypes.c_uint64]
h = ctypes.c_uint64(0)
rr = cuda.cuMemRetainAllocationHandle(ctypes.byref(h), ctypes.c_void_p(p))
if rr == 0:
    cuda.cuMemRelease(h)
print(f"[{conf}] cuMemGetAddressRange rc={r} base_off={p - base.value} size={size.value} units_after={after} "
      f"needed={n} -> {'covers' if after >= n else 'SHORT'}; cuMemRetainAllocationHandle rc={rr}")
# the length-less entry on strings filling [p, p + 2n)
x = O.gen_config(0, n, seed=5)
view = t[(1 << 19):(1 << 19) + n]
view.copy_(torch.from_numpy(x.view(np.int16)))
lens = np.random.default_rng(1).integers(1, 4096, 400_000)
offs = np.concatenate([[0], np.cumsum(lens)])
offs = offs[offs <= n]
offs[-1] = n
d_off = torch.from_numpy(offs.astype(np.int64)).cuda()
L = _lib.raw()
st = L.u16m_to_well_formed_batched(view.data_ptr(), d_off.data_ptr(), d_off.numel() - 1, view.data_ptr(),
                                   torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
got = view.cpu().numpy().view(np.uint16)
exp = O.fix_batched(x, offs)
print(f"[{conf}] length-less batched status={st} exact={np.array_equal(got, exp)} "
      f"mismatches={int((got != exp).sum())}")
