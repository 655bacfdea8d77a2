"""In-tree build of libu16m.so (sm_100a only). Used by __graft_entry__.build().

    python paper_2601_06349_b200/_build.py [--force]

Every .cu in csrc/ is compiled with nvcc for `-gencode arch=compute_100a,
code=sm_100a -lineinfo -O3` and linked (static cudart) into
paper_2601_06349_b200/libu16m.so, next to this file, so the built library
travels to the GPU box with the repo snapshot.

libu16m.so holds the default kernel path only. The kernel families kept for
A/B measurements (U16M_KERNEL=tma|ldg|general) are compiled only with
-DU16M_AB_VARIANTS, into a second library libu16m_ab.so of the same ABI that
tests/test_gpu_variants.py and the A/B scripts load through U16M_LIBRARY.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "build")
LIB = os.path.join(PKG, "libu16m.so")
LIB_AB = os.path.join(PKG, "libu16m_ab.so")   # + the A/B kernel families
AB_SOURCES = ("u16m_kernels.cu", "u16m_tma.cu")  # the files that test U16M_AB_VARIANTS
CLI = os.path.join(PKG, "u16m")
CLI_SRC = os.path.join(PKG, "tools", "u16m_cli.cpp")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ARCH + ["-lineinfo", "-O3", "-std=c++20", "-Xcompiler", "-fPIC,-O3,-Wall",
                "-I", os.path.join(ROOT, "include"), "--expt-relaxed-constexpr"]


def _sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps() -> list[str]:
    return (_sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))
            + glob.glob(os.path.join(ROOT, "include", "*.h"))
            + glob.glob(os.path.join(ROOT, "include", "utf16mend", "*.hpp")) + [__file__])


def needs_build() -> bool:
    if not all(os.path.exists(p) for p in (LIB, LIB_AB, CLI)):
        return True
    t = min(os.path.getmtime(p) for p in (LIB, LIB_AB, CLI))
    return any(os.path.getmtime(p) > t for p in _deps() + [CLI_SRC])


def build_cli() -> str:
    """The `u16m` command-line front end (fix / check / generate) over the C ABI."""
    cmd = ["g++", "-std=c++20", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"), CLI_SRC,
           "-L", PKG, "-lu16m", "-Wl,-rpath,$ORIGIN", "-o", CLI + ".tmp"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"CLI build failed:\n{r.stdout}\n{r.stderr}")
    os.replace(CLI + ".tmp", CLI)
    return CLI


def _compile(job: tuple[str, bool]) -> str:
    src, ab = job
    obj = os.path.join(BUILD, os.path.basename(src) + (".ab.o" if ab else ".o"))
    cmd = [NVCC, *FLAGS, *(["-DU16M_AB_VARIANTS"] if ab else []), "-Xptxas", "-v", "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    with open(obj + ".ptxas.txt", "w") as f:
        f.write(r.stderr)
    return obj


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    os.makedirs(BUILD, exist_ok=True)
    srcs = _sources()
    jobs = [(s, False) for s in srcs] + [(s, True) for s in srcs if os.path.basename(s) in AB_SOURCES]
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = dict(zip(jobs, ex.map(_compile, jobs)))
    for lib, ab in ((LIB, False), (LIB_AB, True)):
        use = [objs[(s, ab and os.path.basename(s) in AB_SOURCES)] for s in srcs]
        tmp = lib + ".tmp"
        cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *use, "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
        os.replace(tmp, lib)
    build_cli()
    if verbose:
        print("built", LIB, "and", CLI)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
