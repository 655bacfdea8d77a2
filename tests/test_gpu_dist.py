"""GPU + NCCL: the one-process-per-GPU sharded step (dist.repair_shard) under
torchrun, checked against the CPU oracle (world size = every visible GPU, so a
multi-GPU box exercises NVLink peer traffic; one GPU here)."""
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
HELPER = os.path.join(os.path.dirname(os.path.abspath(__file__)), "gpu_helpers", "dist_check.py")


def test_torchrun_sharded_step(cuda):
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    n = torch.cuda.device_count()
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), HELPER],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "ALL OK" in r.stdout


def test_torchrun_peer_halo_ipc(cuda):
    """Zero-collective sharded step (CUDA IPC neighbour loads): one process per
    visible GPU (at least 2; on one GPU both processes share it)."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    helper = os.path.join(os.path.dirname(HELPER), "ipc_check.py")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={max(2, torch.cuda.device_count())}",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), helper],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "ALL OK" in r.stdout
