"""CPU: the C-ABI library loads, exports every symbol include/*.h declares,
validates arguments and fails loudly (no CPU fallback) without a GPU; the
source-compatible C++ header compiles and links; Python-level error
behaviour matches the reference bindings."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import oracle as O
import paper_2601_06349_b200 as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
INC = os.path.join(ROOT, "include")
LIBDIR = os.path.join(ROOT, "paper_2601_06349_b200")


def declared(header):
    text = open(os.path.join(INC, header)).read()
    return sorted(set(re.findall(r"\b(u16m_[a-z0-9_]+)\s*\(", text)))


@pytest.mark.parametrize("header", ["u16m.h", "u16m_datagen.h"])
def test_exports_every_declared_symbol(header):
    lib = ctypes.CDLL(P.lib_path())
    names = declared(header)
    assert len(names) >= 4
    for n in names:
        assert hasattr(lib, n), n
    out = subprocess.run(["nm", "-D", "--defined-only", P.lib_path()], capture_output=True, text=True).stdout
    for n in names:
        assert re.search(rf"\bT {n}\b", out), n


def test_ab_library_same_abi_and_product_library_holds_default_path_only():
    """libu16m_ab.so (-DU16M_AB_VARIANTS) exports the same ABI; the A/B-only
    kernel instantiations (plain streams through the TMA ring, the general
    kernel for plain copy / in place) are absent from the product library."""
    ab = os.path.join(os.path.dirname(P.lib_path()), "libu16m_ab.so")
    assert os.path.exists(ab)
    def dyn(path):
        out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True).stdout
        return sorted(l.split()[-1] for l in out.splitlines() if " T " in l and "launch_repair_tma" not in l)
    assert dyn(ab) == dyn(P.lib_path())
    def kernels(path):
        out = subprocess.run(["cuobjdump", "-elf", path], capture_output=True, text=True).stdout
        return set(re.findall(r"\.text\.(_Z\S+)", out))
    prod, full = kernels(P.lib_path()), kernels(ab)
    assert prod < full
    extra = "\n".join(sorted(full - prod))
    assert "repair_tma_kernel" in extra and "repair_kernel" in extra
    # what the product path launches is all there
    for k in ("stream_kernel", "stream_shift_kernel", "batched_tile_kernel", "tile_first_kernel", "repair_tma_kernel"):
        assert any(k in n for n in prod), k


def test_cpp_api_symbols_exported():
    out = subprocess.run(["nm", "-DC", "--defined-only", P.lib_path()], capture_output=True, text=True).stdout
    for sym in ("utf16mend::to_well_formed(", "utf16mend::to_well_formed_in_place(",
                "utf16mend::to_well_formed_batched(", "utf16mend::parse_kernel_id(",
                "utf16mend::select_kernel(", "utf16mend::available_kernels(",
                "utf16mend::is_well_formed(", "utf16mend::unpaired_surrogate_offsets(",
                "utf16mend::fix_scalar(char16_t*, char16_t const*, unsigned long)",
                "utf16mend::fix_scalar(std::span<char16_t const"):
        assert sym in out, sym


def _has_gpu():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # noqa: BLE001
        return False


def test_c_consumer(tmp_path):
    exe = tmp_path / "c_abi"
    subprocess.run(["gcc", "-std=c11", "-Wall", "-Werror", "-I", INC, os.path.join(ROOT, "tests", "abi", "c_abi.c"),
                    "-L", LIBDIR, "-lu16m", f"-Wl,-rpath,{LIBDIR}", "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == (0 if _has_gpu() else 3), r.stdout + r.stderr


def test_cpp_dropin_compiles_links_runs(tmp_path):
    exe = tmp_path / "cpp_dropin"
    subprocess.run(["g++", "-std=c++20", "-Wall", "-I", INC, os.path.join(ROOT, "tests", "abi", "cpp_dropin.cpp"),
                    "-L", LIBDIR, "-lu16m", f"-Wl,-rpath,{LIBDIR}", "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    if _has_gpu():
        assert r.returncode == 0, r.stdout + r.stderr
    else:
        assert r.returncode == 3 and "no CUDA device" in r.stdout, r.stdout + r.stderr


def _compile(tmp_path, src, name, cuda=False):
    exe = tmp_path / name
    cmd = ["g++", "-std=c++20", "-Wall", "-Wextra", "-Werror", "-I", INC, os.path.join(ROOT, "tests", "abi", src),
           "-L", LIBDIR, "-lu16m", f"-Wl,-rpath,{LIBDIR}", "-o", str(exe)]
    if cuda:
        cmd[1:1] = ["-I", "/usr/local/cuda/include"]
        cmd += ["-L", "/usr/local/cuda/lib64", "-lcudart", "-Wl,-rpath,/usr/local/cuda/lib64"]
    subprocess.run(cmd, check=True)
    return exe


def test_reference_driver_tests_pass_against_dropin_header(tmp_path):
    """proj/tests/test_driver.cpp's selection cases, ported assertion for
    assertion (no GPU needed: selection and argument checks run before any
    device work)."""
    exe = _compile(tmp_path, "driver_compat.cpp", "driver_compat")
    r = subprocess.run([str(exe), "select"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


def test_utf16mend_kernel_env_soft_override(tmp_path):
    """UTF16MEND_KERNEL: a supported name wins, an unknown or unsupported one
    warns exactly as proj/src/driver.cpp:97-104 and falls back."""
    exe = _compile(tmp_path, "driver_compat.cpp", "driver_compat")

    def run(val):
        env = dict(os.environ)
        env.pop("UTF16MEND_KERNEL", None)
        if val is not None:
            env["UTF16MEND_KERNEL"] = val
        return subprocess.run([str(exe), "env"], capture_output=True, text=True, env=env)

    default = run(None)
    assert default.returncode == 0 and default.stderr == ""
    r = run("scalar")
    assert r.stdout.strip() == "scalar" and r.stderr == ""
    r = run("turbo")
    assert r.stdout == default.stdout
    assert r.stderr == "utf16mend: ignoring UTF16MEND_KERNEL=turbo (unknown kernel name); using default\n"
    native = "bytesplit" if default.stdout.strip() != "bytesplit" else "bitmask"
    r = run(native)
    assert r.stdout == default.stdout
    assert r.stderr == f"utf16mend: ignoring UTF16MEND_KERNEL={native} (unsupported on this host); using default\n"
    if O.ref() is not None:
        assert default.stdout.strip() == O.ref_default_kernel()


@pytest.mark.gpu
def test_reference_driver_repair_cases_on_gpu(tmp_path, golden):
    """proj/tests/test_driver.cpp:82-113 on the GPU: every selectable kernel id
    repairs the mixed sample in both modes, and all ids agree with scalar on
    150 generate() inputs."""
    _, arr = golden
    exe = _compile(tmp_path, "driver_compat.cpp", "driver_compat")
    hx = lambda a: ",".join(f"{int(v):x}" for v in a)  # noqa: E731
    r = subprocess.run([str(exe), "repair", hx(arr["mixed_in"]), hx(arr["mixed_expected"])], capture_output=True,
                       text=True)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_dropin_on_gpu(tmp_path, cuda):
    """The C++ drop-in end to end on a GPU: the host-vector program
    (cpp_dropin.cpp) exits 0, and the placement program (cpp_dropin_gpu.cpp:
    device spans, batched with device/host offsets, host spans over more than
    two pipeline chunks, validation on device spans) exits 0 — with the
    default 32 Mi-unit chunks and with 64 KiB chunks."""
    exe = _compile(tmp_path, "cpp_dropin.cpp", "cpp_dropin")
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    exe = _compile(tmp_path, "cpp_dropin_gpu.cpp", "cpp_dropin_gpu", cuda=True)
    for chunk in (None, "64"):
        env = dict(os.environ)
        if chunk:
            env["U16M_PIPE_CHUNK_KIB"] = chunk
        r = subprocess.run([str(exe)], capture_output=True, text=True, env=env, timeout=600)
        assert r.returncode == 0, (chunk, r.stdout + r.stderr)


def test_python_errors_match_reference_bindings():
    with pytest.raises(ValueError, match="even length"):
        P.fix_utf16le(b"\x41")                          # module.cpp:25-26
    with pytest.raises(ValueError, match="unknown kernel"):
        P.fix_utf16le(b"\x41\x00", kernel="nope")       # module.cpp:45
    with pytest.raises(ValueError):
        P.generate_utf16le(4, pair_pct=1.5)             # module.cpp:83-84
    assert P.fix_utf16le(b"") == b""
    native = "bytesplit" if P.default_kernel() != "bytesplit" else "bitmask"
    with pytest.raises(ValueError, match="requires .* which this host does not report"):
        P.fix_utf16le(b"\x41\x00", kernel=native)   # driver.cpp:73-86 via module.cpp (std::invalid_argument)
    if O.ref() is not None:
        # the reference's own lists on this host (module.cpp:95-106)
        assert P.available_kernels() == O.ref_available_kernels()
        assert P.default_kernel() == O.ref_default_kernel()
    assert P.backend() == "cuda-sm100a"


def test_no_cpu_fallback_without_gpu():
    if _has_gpu():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError, match="no CUDA device"):
        P.fix_utf16le(b"\x00\xd8")
    with pytest.raises(RuntimeError, match="no CUDA device"):
        P.fix_str("a\ud800")


def test_generate_utf16le_matches_reference_generator():
    for seed, n, p, m in ((0, 1000, 0.1, 0.3), (3, 50_000, 0.001, 0.0), (9, 17, 0.5, 0.5)):
        a = np.frombuffer(P.generate_utf16le(n, p, m, seed), np.uint16)
        assert (a == O.ref_generate(n, p, m, seed)).all()


def test_header_is_plain_c():
    text = open(os.path.join(INC, "u16m.h")).read()
    assert "torch" not in text and "cuda_runtime" not in text and "extern \"C\"" in text


def test_cli_usage_errors_without_gpu(tmp_path):
    cli = os.path.join(LIBDIR, "u16m")
    assert os.path.exists(cli)
    assert subprocess.run([cli], capture_output=True).returncode == 2
    assert subprocess.run([cli, "bogus"], capture_output=True).returncode == 2
    f = tmp_path / "x"
    f.write_bytes(b"\x41\x00")
    p = subprocess.run([cli, "fix", str(f)], capture_output=True, text=True)
    assert p.returncode == 2 and "--in-place or --output" in p.stderr
    p = subprocess.run([cli, "fix", "-k", "warp9", str(f), "-o", str(f) + ".o"], capture_output=True, text=True)
    assert p.returncode == 2 and "unknown kernel" in p.stderr
