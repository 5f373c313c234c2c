"""The C++ API layer (paper_2206_05998_b200/host -> libnoma_host.so): the
reference's noma:: functions over the C-ABI.  Builds on CPU; its own test
program (host/tests/test_detector.cpp: wide layers, large minibatches, FP64
training == loss_and_grad + adam_step composed, zero hidden layers) runs on
the GPU.  The reference's own unit tests are in test_reference_suite.py."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2206_05998_b200")
LIB = os.path.join(PKG, "libnoma_host.so")
BIN = os.path.join(PKG, "host", "_build", "test_detector")


@pytest.fixture(scope="module")
def built():
    if not os.path.exists(BIN) or not os.path.exists(LIB):
        import __graft_entry__

        __graft_entry__.build()
    assert os.path.exists(BIN) and os.path.exists(LIB)
    return BIN


def test_host_layer_builds_and_links_the_cuda_library(built):
    for f in (LIB, built):
        out = subprocess.run(["ldd", f], capture_output=True, text=True).stdout
        assert "libnoma_b200.so" in out and "not found" not in out, out
    out = subprocess.run(["ldd", built], capture_output=True, text=True).stdout
    assert "libnoma_host.so" in out


def test_host_layer_exports_the_reference_api(built):
    syms = subprocess.run(["nm", "-DC", "--defined-only", LIB], capture_output=True, text=True).stdout
    for name in ["noma::lls::fit(", "noma::lls::predict(", "noma::hybrid_nn::init_params(",
                 "noma::hybrid_nn::forward(", "noma::hybrid_nn::loss_and_grad(", "noma::hybrid_nn::adam_step(",
                 "noma::hybrid_nn::train(", "noma::hybrid_nn::detect(", "noma::fused::build_plan(",
                 "noma::fused::fused_forward(", "noma::fused::fused_forward_into(",
                 "noma::fused::fused_forward_f32(", "noma::fused::bench_compare(", "noma::FusedPlan::unpack()",
                 "noma::BenchReport::to_csv", "noma::AdamState::init(", "noma::HybridNetParams::trainable_count()",
                 "noma::widen_design(", "noma::widen_targets(", "noma::widen_dataset(", "noma::narrow_predictions(",
                 "noma::hard_decision_qpsk(", "noma::map_qpsk_bits(", "noma::bit_error_rate(",
                 "noma::run_noise_sweep(", "noma::BerReport::to_csv", "noma::synthesize(",
                 "noma::gen_symbols(", "noma::gen_channel(", "noma::power_profile(",
                 "noma::ScenarioConfig::validate()", "noma::detector_from_string(", "noma::ablation_from_string("]:
        assert name in syms, name


def test_host_layer_fails_loudly_without_gpu(built):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    r = subprocess.run([built], capture_output=True, text=True)
    assert r.returncode != 0
    assert "no CUDA device" in r.stderr


@pytest.mark.gpu
def test_cpp_api_suite_on_device(built):
    r = subprocess.run([built], capture_output=True, text=True, timeout=900)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "Status: SUCCESS" in r.stdout
