"""bench.py prints the one-line JSON contract the driver parses: the CPU
reference arm here, and the GPU arm on a B200 (-m gpu)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config"}


def run_bench(*args, timeout=600):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_contract():
    d = run_bench("--impl", "reference", "--steps", "2", "--warmup", "3", "--config", "c0")
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["unit"] == "GB/s" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["config"]["units_per_gpu"] == 1 << 24 and d["modes"]["copy"]["value"] == d["value"]


@pytest.mark.gpu
def test_gpu_arm_contract(cuda):
    """The default line: config 4 (2^32 units/GPU), copy headline + in place,
    roofline / cpu_baseline / e2e / clocks / gpu_launches present, the same
    `config` dict the reference arm prints."""
    d = run_bench("--steps", "5", "--warmup", "3", timeout=1200)
    assert BASE_KEYS <= set(d)
    assert d["n_gpus"] == 1 and d["higher_is_better"] is True and d["scaling"] == "weak"
    c = d["config"]
    assert c["config_id"] == 4 and c["units_per_gpu"] == 1 << 32 and c["modes"] == ["copy", "inplace"]
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and r["peak"] > 0 and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    assert d["cpu_baseline"]["value"] > 0 and d["cpu_baseline"]["cores"] >= 1
    for m in ("copy", "inplace"):
        md = d["modes"][m]
        assert md["output_check_well_formed"] is True and md["gpu_launches"] == 5
        e = md["e2e"]
        assert e["value"] > 0 and e["h2d_bytes_per_step"] == 2 * c["units_per_gpu"] and e["matches_device_result"]
    assert d["e2e"] == d["modes"]["copy"]["e2e"] and d["value"] == d["modes"]["copy"]["value"]
    assert d["gpu_launches"] == 5
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    ref = run_bench("--impl", "reference", "--steps", "2", "--warmup", "3", timeout=1200)
    assert ref["config"] == c


def test_reference_arm_under_torchrun_env():
    """Under torchrun (N>1) rank 0 alone runs the reference arm and prints the
    same `config` the GPU arm prints at that world size; other ranks print
    nothing and exit 0."""
    sys.path.insert(0, ROOT)
    import bench

    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--steps", "2", "--warmup", "3", "--config", "c0"], capture_output=True, text=True,
                       timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["config"] == bench.config_dict("c0", 1 << 24, 2) and d["config"]["parallelism"] == "shard2"
    env["RANK"] = env["LOCAL_RANK"] = "1"
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--steps", "2", "--warmup", "3", "--config", "c0"], capture_output=True, text=True,
                       timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0 and r.stdout.strip() == ""


@pytest.mark.gpu
def test_gpu_arm_multi_rank_line(cuda):
    """The N>1 line through torchrun (two ranks; on a one-GPU box they share
    it via U16M_BENCH_SHARE_GPU and a gloo group): IPC peer halos, summed
    e2e, max-over-ranks timing, one JSON line from rank 0 — the code path the
    driver's scaling run takes."""
    import torch

    env = dict(os.environ)
    if torch.cuda.device_count() < 2:
        env["U16M_BENCH_SHARE_GPU"] = "1"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", "29531", os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3",
           "--warmup", "3", "--config", "c1"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["parallelism"] == "shard2" and d["value"] > 0
    assert d["run"]["halo"] == "ipc-peer-loads" and d["modes"]["inplace"]["output_check_well_formed"] is True
    assert d["e2e"]["value"] > 0 and d["e2e"]["matches_device_result"] is True
