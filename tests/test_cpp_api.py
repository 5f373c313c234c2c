"""The C++ noma:: host layer over the C-ABI (paper_2206_05998_b200/host):
builds on CPU; its reference-style test program runs on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HOST = os.path.join(ROOT, "paper_2206_05998_b200", "host")
BIN = os.path.join(HOST, "_build", "test_detector")


@pytest.fixture(scope="module")
def built():
    import __graft_entry__

    __graft_entry__.build()
    assert os.path.exists(BIN)
    return BIN


def test_host_layer_builds_and_links_the_cuda_library(built):
    out = subprocess.run(["ldd", built], capture_output=True, text=True).stdout
    assert "libnoma_host.so" in out and "libnoma_b200.so" in out
    assert "not found" not in out


def test_host_layer_fails_loudly_without_gpu(built):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    r = subprocess.run([built], capture_output=True, text=True)
    assert r.returncode != 0
    assert "no CUDA device" in r.stdout


@pytest.mark.gpu
def test_cpp_api_suite_on_device(built):
    r = subprocess.run([built], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failed" in r.stdout
