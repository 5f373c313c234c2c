"""The reference's own unit tests as checkers of the B200 C++ API.

oracle/reftests.mk compiles proj/tests/test_{iq_transform,lls,hybrid_nn,
fused,eval,channel_sim}.cpp UNMODIFIED (read in place from /root/reference,
never copied) against the reference headers, the doctest / Eigen subsets in
paper_2206_05998_b200/host and libnoma_host.so, whose every compute call runs
on the GPU.  The binaries live in oracle/_ref/reftests/ (built in the
container, shipped to the GPU box with the snapshot).

On CPU: every binary runs, the host-only cases (hand cases of the IQ
transform, hard decisions, BER, RNG draws, config validation, plan packing)
pass and every device case fails loudly with "no CUDA device" -- no
assertion fails and nothing falls back to the CPU.  On the GPU: every test
case of every file passes.
"""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "oracle", "_ref", "reftests")
SUITES = ["iq_transform", "lls", "hybrid_nn", "fused", "eval", "channel_sim"]
REF_TESTS = "/root/reference/proj/tests"


def _binary(name):
    path = os.path.join(OUT, f"test_{name}")
    if not os.path.exists(path) and os.path.isdir(REF_TESTS):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "-f", "reftests.mk"], check=True)
    if not os.path.exists(path):
        pytest.fail(f"{path} missing: build it in a container that has /root/reference (__graft_entry__.build())")
    return path


def _summary(out):
    m = re.search(r"test cases: (\d+) \| (\d+) passed \| (\d+) failed", out)
    a = re.search(r"assertions: (\d+) \| (\d+) passed \| (\d+) failed", out)
    assert m and a, out
    return [int(x) for x in m.groups()], [int(x) for x in a.groups()]


@pytest.mark.parametrize("name", SUITES)
def test_reference_suite_host_cases_without_gpu(name):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present: the device run below covers it")
    r = subprocess.run([_binary(name)], capture_output=True, text=True, timeout=300)
    cases, asserts = _summary(r.stdout)
    assert asserts[2] == 0, r.stderr  # no assertion fails on the host ...
    errs = [ln for ln in r.stderr.splitlines() if "threw" in ln]
    assert len(errs) == cases[2]  # ... every failed case is a device call refusing to run
    assert all("no CUDA device" in ln for ln in errs), errs


@pytest.mark.gpu
@pytest.mark.parametrize("name", SUITES)
def test_reference_suite_on_device(name):
    r = subprocess.run([_binary(name)], capture_output=True, text=True, timeout=1800)
    print(r.stdout)
    print(r.stderr[-4000:])
    cases, asserts = _summary(r.stdout)
    assert r.returncode == 0 and cases[2] == 0 and asserts[2] == 0, r.stderr[-4000:]
