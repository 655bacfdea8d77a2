"""GPU: randomised differential fuzz over every entry point against the CPU
oracle (random lengths, 16-byte phases, halos, parts on two streams, batches
with empty / tiny / long strings, byte orders, counts)."""
import numpy as np
import pytest
import torch

import oracle as O
from helpers import ALPHABET

pytestmark = pytest.mark.gpu


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.uint16).view(np.int16).copy()).cuda()


def host(t):
    return t.cpu().numpy().view(np.uint16)


def draw(rng, n):
    kind = rng.integers(0, 3)
    if kind == 0:
        return rng.choice(ALPHABET, n)
    if kind == 1:
        return rng.integers(0, 65536, n).astype(np.uint16)
    return O.gen_config(int(rng.choice([0, 2, 4])), max(n, 1), seed=int(rng.integers(0, 1 << 30)))[:n]


def test_fuzz_all_entry_points(P, cuda):
    import os

    # U16M_FUZZ_ITERS / U16M_FUZZ_SEED: longer or different campaigns on demand
    rng = np.random.default_rng(int(os.environ.get("U16M_FUZZ_SEED", "2026")))
    L = P._lib.raw()
    arena = torch.zeros(1 << 21, dtype=torch.int16, device="cuda")
    arena2 = torch.zeros(1 << 21, dtype=torch.int16, device="cuda")
    for it in range(int(os.environ.get("U16M_FUZZ_ITERS", "300"))):
        n = int(rng.choice([0, 1, 2, 7, 8, 9, 63, 64, 65]) if it % 4 == 0 else rng.integers(1, 900_000))
        x = draw(rng, n)
        left = int(rng.choice([-1, 0x41, 0xD801, 0xDC02]))
        right = int(rng.choice([-1, 0x42, 0xD803, 0xDC04]))
        e = O.stencil(x, left, right)
        pi, po = int(rng.integers(0, 8)), int(rng.integers(0, 8))
        src = arena[pi:pi + n]
        src.copy_(dev(x)) if n else None
        # copy with halos, arbitrary phases
        out = arena2[po:po + n]
        P.to_well_formed_halo(src, out, left, right)
        assert (host(out) == e).all(), ("halo copy", it, n, pi, po)
        # parts on two streams, in place
        if n:
            hal = dev(np.array([left & 0xFFFF, right & 0xFFFF], np.uint16))
            lp = hal.data_ptr() if left >= 0 else 0
            rp = hal.data_ptr() + 2 if right >= 0 else 0
            s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
            s1.wait_stream(torch.cuda.current_stream())
            s2.wait_stream(torch.cuda.current_stream())
            P.to_well_formed_part(src, None, P._lib.PART_INTERIOR, stream=s1)
            P.to_well_formed_part(src, None, P._lib.PART_EDGES, lp, rp, stream=s2)
            torch.cuda.synchronize()
            assert (host(src) == e).all(), ("parts in place", it, n, pi)
        # count + byte-order codec (no halos)
        e0 = O.stencil(x)
        if n:
            assert P.count_unpaired(dev(x)) == int((x != e0).sum())
            bt = dev(x.astype(">u2").view(np.uint16))
            ob, c = P.to_well_formed_bytes(bt, big_endian=True, count=True)
            assert (host(ob).view(">u2").astype(np.uint16) == e0).all() and c == int((x != e0).sum()), it
            # the same between arbitrary 16-byte phases (shifted-store codec kernel), LE and BE
            big = bool(it & 1)
            sb = arena[pi:pi + n]
            sb.copy_(bt if big else dev(x))
            ob2 = arena2[po:po + n]
            r = P.to_well_formed_bytes(sb, out=ob2, big_endian=big, count=bool(it & 2))
            hb = host(ob2)
            hb = hb.view(">u2").astype(np.uint16) if big else hb
            assert (hb == e0).all(), ("codec phases", it, n, pi, po, big)
            if it & 2:
                assert r[1] == int((x != e0).sum()), ("codec phases count", it)
        # batched over a random split of x
        cuts = np.sort(rng.integers(0, n + 1, int(rng.integers(0, 40))))
        offs = np.concatenate([[int(rng.integers(0, min(n, 5) + 1))] if n else [0], cuts, [n]]).astype(np.int64)
        offs = np.maximum.accumulate(offs)
        eb = O.fix_batched(x, offs)
        got = host(P.to_well_formed_batched(dev(x), torch.from_numpy(offs).cuda()))
        assert (got == eb).all(), ("batched", it, n)
        # batched from the phase-pi source into a phase-po output (shifted stores when they differ)
        if n:
            src.copy_(dev(x))
            bo = arena2[po:po + n]
            bo.copy_(src)
            P.to_well_formed_batched(src, torch.from_numpy(offs).cuda(), out=bo)
            assert (host(bo) == eb).all(), ("batched phases", it, n, pi, po)


def test_fuzz_batched_host_pipeline(cuda):
    """Random batches through the pipelined batched host form with 8 KiB
    chunks (4096 units), so strings are cut by many chunk edges."""
    import os
    import subprocess
    import sys

    helper = os.path.join(os.path.dirname(os.path.abspath(__file__)), "gpu_helpers", "batched_host_fuzz.py")
    env = {k: v for k, v in os.environ.items() if not k.startswith("U16M_PIPE")}
    env["U16M_PIPE_CHUNK_KIB"] = "8"
    r = subprocess.run([sys.executable, helper], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout + r.stderr
