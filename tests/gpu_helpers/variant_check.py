"""Parity of one kernel variant (selected by the U16M_* environment of this
process) against the CPU oracle. Run by tests/test_gpu_variants.py."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
import paper_2601_06349_b200 as P  # noqa: E402

ALPHA = np.array([0x0041, 0xD7FF, 0xD800, 0xDBFF, 0xDC00, 0xDFFF, 0xE000, 0xFFFD], np.uint16)


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.uint16).view(np.int16).copy()).cuda()


def host(t):
    return t.cpu().numpy().view(np.uint16)


def main():
    rng = np.random.default_rng(123)
    small = os.environ.get("U16M_TEST_SMALL") == "1"  # sanitizer runs
    big = torch.zeros(1 << 22, dtype=torch.int16, device="cuda")
    sizes = (1, 7, 9, 8193, 70_001, 300_001) if small else (1, 7, 8, 9, 100, 8191, 8193, 3 * 8192 + 17, 40_000,
                                                              300_001, 2_000_003)
    for n in sizes:
        x = rng.choice(ALPHA, n) if n % 2 else O.gen_config(1, n, seed=n)
        e = O.stencil(x)
        for ph in (0, 3, 8):
            src = big[ph:ph + n]
            src.copy_(dev(x))
            assert (host(P.to_well_formed(src)) == e).all(), ("copy", n, ph)
            P.to_well_formed_(src)
            assert (host(src) == e).all(), ("inplace", n, ph)
            src.copy_(dev(x))
            out = torch.empty(n + 8, dtype=torch.int16, device="cuda")[5:5 + n]
            P.to_well_formed(src, out=out)
            assert (host(out) == e).all(), ("copy-other-phase", n, ph)
    x = O.gen_config(1, 100_000 if small else 1_000_000, seed=5)
    for left in (-1, 0xD800):
        for right in (-1, 0xDC00):
            t = dev(x)
            P.to_well_formed_halo(t, None, left, right)
            assert (host(t) == O.stencil(x, left, right)).all()
    lens = rng.choice([0, 1, 2, 5, 31, 400, 4095, 9000], 300 if small else 5000)
    offs = np.zeros(lens.size + 1, np.int64)
    offs[1:] = np.cumsum(lens) + 3
    offs[0] = 3
    data = O.gen_config(1, int(offs[-1]) + 5, seed=9)
    e = O.fix_batched(data, offs)
    got = host(P.to_well_formed_batched(dev(data), torch.from_numpy(offs).cuda()))
    assert (got == e).all(), "batched"
    t = dev(data)
    P.to_well_formed_batched(t, torch.from_numpy(offs).cuda(), out=t)
    assert (host(t) == e).all(), "batched in place"
    # host-memory path (staged copy-engine pipeline), pinned buffers
    y = O.gen_config(1, 300_001, seed=8)
    pin = torch.from_numpy(y.view(np.int16).copy()).pin_memory()
    outp = torch.empty_like(pin).pin_memory()
    L = P._lib.raw()
    assert L.u16m_to_well_formed_host(pin.data_ptr(), y.size, outp.data_ptr()) == 0
    assert (outp.numpy().view(np.uint16) == O.stencil(y)).all(), "host copy"
    assert L.u16m_to_well_formed_host(pin.data_ptr(), y.size, pin.data_ptr()) == 0
    assert (pin.numpy().view(np.uint16) == O.stencil(y)).all(), "host in place"
    # pageable buffers (the CopyPool bounce-buffer path; with U16M_PIPE_CHUNK_KIB=64
    # this is 10 chunks, more than the 4 pinned bounce buffers)
    pg = y.view(np.int16).copy()
    pgo = np.empty_like(pg)
    assert L.u16m_to_well_formed_host(pg.ctypes.data, y.size, pgo.ctypes.data) == 0
    assert (pgo.view(np.uint16) == O.stencil(y)).all(), "host pageable copy"
    assert L.u16m_to_well_formed_host(pg.ctypes.data, y.size, pg.ctypes.data) == 0
    assert (pg.view(np.uint16) == O.stencil(y)).all(), "host pageable in place"
    be, c = P.fix_utf16_bytes(y.astype(">u2").tobytes(), "be")
    assert np.frombuffer(be, ">u2").astype(np.uint16).tobytes() == O.stencil(y).tobytes(), "host codec"
    torch.cuda.synchronize()
    print("OK", {k: v for k, v in os.environ.items() if k.startswith("U16M_")})


if __name__ == "__main__":
    main()
