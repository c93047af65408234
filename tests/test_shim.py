"""INTEGRATION.md's reference-side C++ shim, compiled with g++ against
stand-in reference types and linked to libspngd_b200.so (tests/shim/).
CPU: it builds, links and fails loudly without a GPU (spngd::Error, no
fallback).  GPU: the worked damp_and_invert example and a batch whose block 3
has a non-PD G factor -> NotPositiveDefinite naming request 3 / G factor."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2002_06015_b200")


@pytest.fixture(scope="module")
def shim_bin(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("shim") / "shim_test")
    cmd = ["g++", "-std=c++20", "-O1", "-Wall", "-Wextra", "-o", out, os.path.join(ROOT, "tests", "shim", "shim_test.cpp"),
           "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include", "-L", LIB, "-lspngd_b200",
           "-L", "/usr/local/cuda/lib64", "-lcudart", f"-Wl,-rpath,{LIB}", "-Wl,-rpath,/usr/local/cuda/lib64"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return out


def test_shim_builds_and_fails_loudly_without_gpu(shim_bin):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present: see test_shim_on_gpu")
    p = subprocess.run([shim_bin, "--expect-no-gpu"], capture_output=True, text=True, timeout=60)
    assert p.returncode == 0 and "NO_GPU_OK" in p.stdout, p.stdout + p.stderr


@pytest.mark.gpu
def test_shim_on_gpu(shim_bin, cuda_dev):
    p = subprocess.run([shim_bin], capture_output=True, text=True, timeout=120)
    assert p.returncode == 0 and "SHIM OK" in p.stdout, p.stdout + p.stderr
