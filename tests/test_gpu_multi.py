"""Multi-GPU step (SURVEY.md §8e, rows a9 reduce_scatter_v / a17 all_gather_v):
world 2 and 4 over NCCL + NVLink on one node, launched with torchrun.  Each
run checks (scripts/multi_gpu_check.py) that every replica is bit-identical,
that the P-rank step equals the one-rank step over the concatenated batch
(K-invariance, tests/test_dist.cpp:363-387), that the CommLedger rows equal
the oracle restatement, and -- on the ResNet-50 sample with the 4608^2 /
2304^2 / 2048^2 factors -- that the updated weights match the fp64 oracle on
the concatenated batch (<= 1e-4).  Skipped when the box has fewer GPUs."""
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(world, mode, layers):
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "scripts", "multi_gpu_check.py"), "--mode", mode, "--layers", layers]
    p = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    out = p.stdout + p.stderr
    if os.path.isdir(os.path.join(ROOT, "gpurun_out")):  # keep the per-layer report of GPU runs
        with open(os.path.join(ROOT, "gpurun_out", f"multi_{world}_{mode}_{layers}.log"), "w") as f:
            f.write(p.stdout)
    assert p.returncode == 0 and "PASS" in out, out[-4000:]
    return out


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("mode", ["default", "p2p"])
def test_multi_gpu_resnet50_sample(world, mode):
    """NCCL reduce-scatter / all-gather (default) and the fused NVLink
    statistics RS + weight AG (p2p) on the ResNet-50 layer sample."""
    out = _run(world, mode, "r50")
    assert "oracle layer" in out


@pytest.mark.parametrize("mode", ["wgrad", "bn_full", "one_mc", "sgd", "host", "p2p_host"])
def test_multi_gpu_modes(mode):
    """Every optimizer mode of DESIGN.md §3.6 at world 2 on the toy net."""
    _run(2, mode, "toy")
