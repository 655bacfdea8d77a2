"""GPU: §8(f-3) codec fusion (byte-order-aware repair + replacement count) and
the `u16m` CLI, mirroring the reference CLI tests (proj/tests/test_cli.cpp)
and codec contract (proj/tests/test_codec.cpp)."""
import os
import subprocess

import numpy as np
import pytest
import torch

import oracle as O
import paper_2601_06349_b200 as P

pytestmark = pytest.mark.gpu
CLI = os.path.join(os.path.dirname(P.lib_path()), "u16m")


def run(*args, env=None):
    return subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, env=env)


def test_fix_bytes_le_be_counts(cuda):
    rng = np.random.default_rng(7)
    for n in (1, 2, 31, 8192, 8193, 100_001, 3_000_017):
        x = O.gen_config(1, n, seed=n) if n > 100 else rng.choice(
            np.array([0x41, 0xD800, 0xDBFF, 0xDC00, 0xDFFF, 0xFFFD], np.uint16), n)
        e = O.stencil(x)
        changed = int((x != e).sum())
        le, c = P.fix_utf16_bytes(x.astype("<u2").tobytes(), "le")
        assert le == e.astype("<u2").tobytes() and c == changed, n
        be, c = P.fix_utf16_bytes(x.astype(">u2").tobytes(), "be")
        assert be == e.astype(">u2").tobytes() and c == changed, n
        t = torch.from_numpy(x.astype(">u2").view(np.int16).copy()).cuda()
        out, c = P.to_well_formed_bytes(t, big_endian=True, count=True)
        assert out.cpu().numpy().view(">u2").astype(np.uint16).tolist() == e.tolist() and c == changed
        P.to_well_formed_bytes(t, out=t, big_endian=True)   # in place
        assert (t.cpu().numpy().view(">u2").astype(np.uint16) == e).all()


def test_fix_bytes_chunk_boundaries_be(cuda):
    # host pipeline chunks at 32 Mi units: halos across chunks in BE order
    n = (32 << 20) + 12345
    x = O.gen_config(1, n, seed=3)
    e = O.stencil_mt(x)
    be, c = P.fix_utf16_bytes(x.astype(">u2").tobytes(), "be")
    assert np.frombuffer(be, ">u2").astype(np.uint16).tobytes() == e.tobytes()
    assert c == int((x != e).sum())


def w(path, data):
    with open(path, "wb") as f:
        f.write(bytes(data))


def r(path):
    with open(path, "rb") as f:
        return f.read()


def test_cli_fix_clean_le(tmp_path, cuda):
    inp, out = tmp_path / "in.utf16", tmp_path / "out.utf16"
    w(inp, [0xFF, 0xFE, 0x48, 0x00, 0x69, 0x00])
    p = run("fix", inp, "-o", out)
    assert p.returncode == 0 and p.stdout == "0 replacements\n"
    assert r(out) == r(inp)


def test_cli_fix_lone_high(tmp_path, cuda):
    inp, out = tmp_path / "in", tmp_path / "out"
    w(inp, [0x00, 0xD8, 0x41, 0x00])
    p = run("fix", inp, "-o", out)
    assert p.returncode == 0 and p.stdout == "1 replacement\n"
    assert r(out) == bytes([0xFD, 0xFF, 0x41, 0x00])
    assert "no BOM found" in p.stderr


def test_cli_fix_preserves_be_bom(tmp_path, cuda):
    inp, out = tmp_path / "in", tmp_path / "out"
    w(inp, [0xFE, 0xFF, 0xD8, 0x00, 0x00, 0x41])
    p = run("fix", inp, "-o", out)
    assert p.returncode == 0 and p.stdout == "1 replacement\n"
    assert r(out) == bytes([0xFE, 0xFF, 0xFF, 0xFD, 0x00, 0x41])
    assert run("fix", inp, "-o", out, "--bom", "strip").returncode == 0
    assert r(out) == bytes([0xFF, 0xFD, 0x00, 0x41])


def test_cli_fix_in_place_idempotent(tmp_path, cuda):
    path = tmp_path / "f"
    x = np.frombuffer(P.generate_utf16le(5000, 0.05, 0.02, 11), np.uint16)
    w(path, x.tobytes())
    assert run("fix", "-i", path).returncode == 0
    once = r(path)
    second = run("fix", "-i", path)
    assert second.returncode == 0 and second.stdout == "0 replacements\n"
    assert r(path) == once
    assert once == O.fix_scalar(x).tobytes()


def test_cli_odd_length(tmp_path, cuda):
    inp, out = tmp_path / "in", tmp_path / "out"
    w(inp, [0x41, 0x00, 0x42])
    p = run("fix", inp, "-o", out)
    assert p.returncode == 2 and "truncated" in p.stderr
    p = run("fix", inp, "-o", out, "--pad-final")
    assert p.returncode == 0 and p.stdout == "1 replacement\n"
    assert r(out) == bytes([0x41, 0x00, 0xFD, 0xFF])


def test_cli_kernels_and_env(tmp_path, cuda):
    inp, out = tmp_path / "in", tmp_path / "out"
    w(inp, [0x00, 0xD8])
    for k in ("scalar", "generic16", "bitmask", "bytesplit-emulated"):
        assert run("fix", "-k", k, inp, "-o", out).returncode == 0
        assert r(out) == bytes([0xFD, 0xFF])
    assert run("fix", "-k", "warp9", inp, "-o", out).returncode == 2
    env = dict(os.environ, UTF16MEND_KERNEL="warp9")
    p = run("fix", inp, "-o", out, env=env)
    assert p.returncode == 0 and "UTF16MEND_KERNEL" in p.stderr
    env = dict(os.environ, UTF16MEND_KERNEL="generic8")
    assert "UTF16MEND_KERNEL" not in run("fix", inp, "-o", out, env=env).stderr


def test_cli_check(tmp_path, cuda):
    good, bad = tmp_path / "good", tmp_path / "bad"
    w(good, [0x41, 0x00, 0x3D, 0xD8, 0x0A, 0xDE])
    w(bad, [0x41, 0x00, 0x42, 0x00, 0x43, 0x00, 0x00, 0xDC])
    assert run("check", good).returncode == 0
    p = run("check", bad)
    assert p.returncode == 1 and " 3" in p.stdout
    assert run("check", tmp_path / "missing").returncode == 2
    many = tmp_path / "many"
    w(many, bytes([0x00, 0xDC]) * 40)
    p = run("check", many)
    assert p.returncode == 1
    assert len(p.stdout.split(":")[-1].split()) == 10


def test_cli_generate_and_roundtrip(tmp_path, cuda):
    a, b = tmp_path / "a", tmp_path / "b"
    flags = ["generate", "-n", "10000", "--pair-pct", "0.1", "--mismatch-pct", "0.01", "--seed", "5", "-o"]
    assert run(*flags, a).returncode == 0 and run(*flags, b).returncode == 0
    assert r(a) == r(b) and len(r(a)) == 20000
    assert np.frombuffer(r(a), np.uint16).tolist() == O.ref_generate(10000, 0.1, 0.01, 5).tolist()
    assert run("generate", "-n", "0", "--bom", "-o", tmp_path / "bom").returncode == 0
    assert r(tmp_path / "bom") == bytes([0xFF, 0xFE])
    assert run("check", a).returncode == 1
    fixed = tmp_path / "fixed"
    assert run("fix", a, "-o", fixed).returncode == 0
    assert run("check", fixed).returncode == 0


def test_cli_layout_cases(tmp_path, cuda):
    """The in-place file-buffer path of `fix` / `check`: BOM-only and empty
    files, --bom require, big-endian check, BE + BOM + dangling byte."""
    inp, out = tmp_path / "in", tmp_path / "out"
    w(inp, [0xFF, 0xFE])                               # BOM only
    p = run("fix", inp, "-o", out)
    assert p.returncode == 0 and p.stdout == "0 replacements\n" and r(out) == bytes([0xFF, 0xFE])
    w(inp, [])                                         # empty file
    assert run("fix", inp, "-o", out).returncode == 0 and r(out) == b""
    assert run("check", inp).returncode == 0
    w(inp, [0x41, 0x00])
    p = run("fix", inp, "-o", out, "--bom", "require")
    assert p.returncode != 0 and "BOM required" in p.stderr
    w(inp, [0xFE, 0xFF, 0x00, 0x41, 0xDC, 0x00, 0x00, 0x42])   # BE, lone low at unit 1
    p = run("check", inp)
    assert p.returncode == 1 and p.stdout.split(":")[-1].split() == ["1"]
    w(inp, [0xFE, 0xFF, 0xD8, 0x00, 0x00])             # BE + BOM + lone high + dangling byte
    p = run("fix", inp, "-o", out, "--pad-final")
    assert p.returncode == 0 and p.stdout == "2 replacements\n"
    assert r(out) == bytes([0xFE, 0xFF, 0xFF, 0xFD, 0xFF, 0xFD])
    p = run("fix", inp, "-o", out, "--pad-final", "--bom", "strip")
    assert r(out) == bytes([0xFF, 0xFD, 0xFF, 0xFD])


def test_codec_other_phase_output(cuda):
    """Byte-order-fused repair into an output at another 16-byte phase
    (shifted-store kernel, one pass) — every in/out phase pair, with and
    without the replacement count; nothing outside the output is written."""
    x = np.frombuffer(P.generate_utf16le(100_003, 0.05, 0.02, 3), np.uint16)
    e = O.fix_scalar(x)
    for big in (False, True):
        raw = (x.astype(">u2") if big else x).view(np.uint16)
        src = torch.zeros(x.size + 16, dtype=torch.int16, device="cuda")
        for pi in (0, 3):
            t = src[pi:pi + x.size]
            t.copy_(torch.from_numpy(raw.view(np.int16).copy()))
            for po in range(8):
                if po == pi:
                    continue
                base = torch.full((x.size + 16,), 0x5A5A, dtype=torch.int16, device="cuda")
                out = base[po:po + x.size]
                for count in (True, False):
                    r = P.to_well_formed_bytes(t, out=out, big_endian=big, count=count)
                    got, cnt = r if count else (r, None)
                    h = got.cpu().numpy().view(np.uint16)
                    h = h.view(">u2").astype(np.uint16) if big else h
                    assert (h == e).all(), (big, pi, po, count)
                    if count:
                        assert cnt == int((x != e).sum()), (big, pi, po)
                b = base.cpu().numpy()
                assert (b[:po] == 0x5A5A).all() and (b[po + x.size:] == 0x5A5A).all(), (big, pi, po)
