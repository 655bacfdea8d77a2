"""Every kernel variant selectable through U16M_* (the choice is cached per
process, so each runs in its own subprocess) is bit-exact with the oracle.
The U16M_KERNEL families exist only in the A/B build libu16m_ab.so
(-DU16M_AB_VARIANTS, loaded through U16M_LIBRARY); the product library holds
the default path alone and ignores U16M_KERNEL."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
PKG = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2601_06349_b200")
AB_LIB = os.path.join(PKG, "libu16m_ab.so")
HELPER = os.path.join(os.path.dirname(os.path.abspath(__file__)), "gpu_helpers", "variant_check.py")

VARIANTS = [
    {},
    {"U16M_LIBRARY": AB_LIB},
    {"U16M_LIBRARY": AB_LIB, "U16M_KERNEL": "tma"},
    {"U16M_LIBRARY": AB_LIB, "U16M_KERNEL": "general"},
    {"U16M_LIBRARY": AB_LIB, "U16M_KERNEL": "ldg"},
    {"U16M_KERNEL": "general"},  # product library: ignored
    {"U16M_PREFETCH": "0"},
    {"U16M_BATCHED_PDL": "0"},
    {"U16M_PIPE_CHUNK_KIB": "64", "U16M_HOST_THREADS": "3"},
]


@pytest.mark.parametrize("env", VARIANTS, ids=lambda e: ",".join(f"{k}={os.path.basename(v)}" for k, v in e.items()) or "default")
def test_variant(env, cuda):
    full = dict(os.environ)
    for k in list(full):
        if k.startswith("U16M_"):
            del full[k]
    full.update(env)
    r = subprocess.run([sys.executable, HELPER], env=full, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK" in r.stdout
