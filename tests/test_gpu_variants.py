"""Every kernel variant selectable through U16M_* (the choice is cached per
process, so each runs in its own subprocess) is bit-exact with the oracle."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HELPER = os.path.join(os.path.dirname(os.path.abspath(__file__)), "gpu_helpers", "variant_check.py")

VARIANTS = [
    {},
    {"U16M_KERNEL": "tma"},
    {"U16M_KERNEL": "general"},
    {"U16M_KERNEL": "ldg"},
    {"U16M_PREFETCH": "0"},
    {"U16M_BATCHED_PDL": "0"},
    {"U16M_PIPE_CHUNK_KIB": "64", "U16M_HOST_THREADS": "3"},
]


@pytest.mark.parametrize("env", VARIANTS, ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()) or "default")
def test_variant(env, cuda):
    full = dict(os.environ)
    for k in list(full):
        if k.startswith("U16M_"):
            del full[k]
    full.update(env)
    r = subprocess.run([sys.executable, HELPER], env=full, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK" in r.stdout
