"""Pins the oracle's hybrid network: ports proj/tests/test_hybrid_nn.cpp and
proj/tests/test_fused.cpp against the independent forward / Adam oracles of
tests/refimpl.py (oracles.hpp:75-115)."""
import numpy as np
import pytest

from tests import refimpl as R
from tests.helpers import (make_w0, max_rel_dev, random_mat, random_net_fused,
                           random_net_hybrid, seq_matvec)


def _ref_fwd(net, x):
    layers, final = net.layers()
    return R.reference_forward(net.dims, net.w0, layers, final, x)


# ------------------------------------------------------------ hybrid_nn
def test_init_output_equals_lls_exactly(O):  # test_hybrid_nn.cpp:44-53
    rng = O.Rng(3)
    w0 = make_w0(8, 17)
    net = O.init_params([8, 64, 64, 64], w0, rng)
    x = random_mat(32, 8, 5)
    assert np.max(np.abs(O.forward(net, x) - seq_matvec(x, w0))) == 0.0
    assert np.array_equal(net.w0, w0)


def test_init_determinism_and_count(O):  # :55-64
    w0 = make_w0(8, 17)
    a = O.init_params([8, 64, 64, 64], w0, O.Rng(9))
    b = O.init_params([8, 64, 64, 64], w0, O.Rng(9))
    assert np.array_equal(a.theta, b.theta)
    assert a.trainable_count() == 8 * 64 + 64 + 64 * 64 + 64 + 64 * 64 + 64 + 64


def test_init_draw_order(O):  # hybrid_nn.cpp:43-52: row-major r then c, layer by layer
    dims = [4, 3, 2]
    net = O.init_params(dims, np.zeros(4), O.Rng(21))
    p = R.PyRng(21)
    (W1, b1), (W2, b2) = net.layers()[0]
    for W, fan in ((W1, 4), (W2, 3)):
        for r in range(W.shape[0]):
            for c in range(W.shape[1]):
                assert W[r, c] == p.gaussian() * np.sqrt(2.0 / fan)
    assert not b1.any() and not b2.any() and not net.layers()[1].any()


def test_single_relu_neuron(O):  # :66-79
    net = O.init_params([1, 1], np.zeros(1), O.Rng(1))
    (W, b), final = net.layers()[0][0], net.layers()[1]
    W[0, 0] = 1.0
    final[0] = 1.0
    y = O.forward(net, np.array([[-2.0], [3.0]]))
    assert y[0] == 0.0 and y[1] == 3.0


def test_forward_matches_reference_oracle(O):  # :81-87
    net = random_net_hybrid([8, 16, 16], 21)
    x = random_mat(16, 8, 22)
    assert np.max(np.abs(O.forward(net, x) - _ref_fwd(net, x))) < 1e-12


def test_zero_residual_zero_gradients(O):  # :89-100
    w0 = make_w0(4, 31)
    net = O.init_params([4, 8], w0, O.Rng(4))
    x = random_mat(10, 4, 32)
    y = O.forward(net, x)  # == x w0 exactly for the zero-branch net
    loss, g = O.loss_and_grad(net, x, y)
    assert loss == 0.0 and np.max(np.abs(g)) == 0.0


def test_central_finite_differences(O):  # :102-134
    net = random_net_hybrid([4, 8], 41)
    x = random_mat(12, 4, 42)
    r = O.Rng(43)
    y = np.array([r.gaussian() for _ in range(12)])
    _, g = O.loss_and_grad(net, x, y)
    for i in range(net.theta.size):
        th = net.theta[i]
        h = 1e-6 * max(1.0, abs(th))
        net.theta[i] = th + h
        lp = O.loss_and_grad(net, x, y)[0]
        net.theta[i] = th - h
        lm = O.loss_and_grad(net, x, y)[0]
        net.theta[i] = th
        fd = (lp - lm) / (2 * h)
        denom = max(abs(fd), abs(g[i]), 1e-8)
        assert abs(fd - g[i]) / denom <= 1e-4, i


def test_batch_duplication_invariance(O):  # :136-150
    net = random_net_hybrid([4, 8], 51)
    x = random_mat(6, 4, 52)
    y = random_mat(6, 1, 53)[:, 0]
    l1, g1 = O.loss_and_grad(net, x, y)
    l2, g2 = O.loss_and_grad(net, np.vstack([x, x]), np.concatenate([y, y]))
    assert abs(l1 - l2) <= 1e-14 * max(abs(l1), 1e-300) * 10
    assert np.max(np.abs(g1 - g2)) < 1e-14


def test_adam_zero_grad_and_first_step(O):  # :152-181
    net = random_net_hybrid([4, 8], 61)
    before = net.theta.copy()
    s = O.AdamState(net.theta.size, 0.01)
    O.adam_step(net, np.zeros_like(net.theta), s)
    assert s.step.value == 1 and np.array_equal(net.theta, before)

    net = O.init_params([1, 1], np.zeros(1), O.Rng(1))
    s = O.AdamState(net.theta.size, 0.005)
    g = np.zeros_like(net.theta)
    g[-1] = 1.0
    b0 = net.theta[-1]
    O.adam_step(net, g, s)
    assert abs((b0 - net.theta[-1]) - 0.005) < 1e-6


def test_adam_trajectory_matches_flat_oracle(O):  # :183-227
    net = random_net_hybrid([2, 3], 71)
    x = random_mat(8, 2, 72)
    y = random_mat(8, 1, 73)[:, 0]
    s = O.AdamState(net.theta.size, 0.01)
    theta = net.theta.copy()
    ref = R.ReferenceAdam(theta.size, 0.01)
    for _ in range(10):
        _, g = O.loss_and_grad(net, x, y)
        O.adam_step(net, g, s)
        ref.step(theta, g)
        assert np.max(np.abs(net.theta - theta)) < 1e-12


def _scenario_ds(O, **kw):
    rec = O.synthesize(O.Scenario(**kw))
    return rec


def test_train_zero_epochs_and_trace_length(O):  # :229-251
    rec = O.synthesize(O.Scenario(num_users=2, num_antennas=4, train_symbols=64,
                                  data_symbols=8, seed=81))
    x = O.widen_design(rec.train_rx)
    y = O.widen_targets(rec.train_symbols[:, 0])
    w0 = O.lls_fit(x, y, 1).w
    net = O.init_params([8, 16], w0, O.Rng(82))
    before = net.theta.copy()
    assert O.train(net, x, y, epochs=0).size == 0
    assert np.array_equal(net.theta, before)
    assert O.train(net, x, y, epochs=5).size == 5


def test_train_noiseless_stays_at_lls_optimum(O):  # :253-271
    rec = O.synthesize(O.Scenario(num_users=2, num_antennas=4, train_symbols=685,
                                  data_symbols=8, seed=91))
    x = O.widen_design(rec.train_rx)
    y = O.widen_targets(rec.train_symbols[:, 1])
    w0 = O.lls_fit(x, y, 2).w
    net = O.init_params([8, 64, 64, 64], w0, O.Rng(92))
    trace = O.train(net, x, y, shuffle_seed=93)
    assert trace.size == 50
    assert trace[-1] <= trace[0] + 1e-12
    assert trace[-1] <= 1e-6


def test_w0_frozen_and_determinism(O):  # :273-311
    rec = O.synthesize(O.Scenario(train_symbols=128, data_symbols=8, snr_db=20.0, seed=101))
    x = O.widen_design(rec.train_rx)
    y = O.widen_targets(rec.train_symbols[:, 3])
    w0 = O.lls_fit(x, y, 4).w
    net = O.init_params([8, 32, 32], w0, O.Rng(102))
    O.train(net, x, y, epochs=8)
    assert np.array_equal(net.w0, w0)
    a = O.init_params([8, 16, 16], w0, O.Rng(112))
    b = O.init_params([8, 16, 16], w0, O.Rng(112))
    O.train(a, x, y, epochs=6, shuffle_seed=7)
    O.train(b, x, y, epochs=6, shuffle_seed=7)
    assert np.array_equal(a.theta, b.theta)


def test_detect_zero_branch_and_recovery(O):  # :313-340
    rec = O.synthesize(O.Scenario(num_users=2, num_antennas=4, train_symbols=64,
                                  data_symbols=32, seed=121))
    x = O.widen_design(rec.train_rx)
    y = O.widen_targets(rec.train_symbols[:, 0])
    w0 = O.lls_fit(x, y, 1).w
    net = O.init_params([8, 16], w0, O.Rng(122))
    xd = O.widen_design(rec.data_rx)
    assert np.max(np.abs(O.detect(net, xd) - O.narrow_predictions(seq_matvec(xd, w0)))) == 0.0
    O.train(net, x, y, epochs=10)
    t = O.detect(net, xd)
    truth = rec.data_symbols[:, 0]
    assert np.array_equal(t.real < 0, truth.real < 0)
    assert np.array_equal(t.imag < 0, truth.imag < 0)


def test_error_paths(O):  # :342-352
    with pytest.raises(O.DimensionError):
        O.init_params([8, 16], make_w0(4, 1), O.Rng(2))
    net = O.init_params([4, 8], make_w0(4, 1), O.Rng(2))
    with pytest.raises(O.DimensionError):
        O.forward(net, np.zeros((2, 5)))
    with pytest.raises(O.DimensionError):
        O.train(net, np.zeros((0, 4)), np.zeros(0))
    with pytest.raises(O.ConfigError):
        O.train(net, np.ones((4, 4)), np.ones(4), batch_size=0)


def test_shuffle_matches_independent_fisher_yates(O):  # hybrid_nn.cpp:148-154
    for epoch in (0, 1, 49):
        idx = O.shuffled_indices(1370, 12345, epoch)
        p = R.PyRng(R.substream_seed(12345, epoch))
        ref = list(range(1370))
        for i in range(1369, 0, -1):
            j = p.below(i + 1)
            ref[i], ref[j] = ref[j], ref[i]
        assert idx.tolist() == ref


# ---------------------------------------------------------------- fused
def test_plan_pack_unpack_bit_identical(O):  # test_fused.cpp:64-74
    net = random_net_fused([8, 64, 48, 64], 5)
    u = O.unpack_plan(net.dims, O.build_plan(net))
    assert np.array_equal(u.w0, net.w0) and np.array_equal(u.theta, net.theta)


def test_plan_layout_sizes(O):  # fused_inference.cpp:19-42
    assert O.plan_size([32, 64]) == 2208
    assert O.plan_size([32, 64, 64]) == 6368
    assert O.plan_size([128, 64]) == 8448
    assert O.plan_size([64, 64]) == 4288


def test_zero_final_layer_reduces_to_linear(O):  # :76-85
    rng = O.Rng(6)
    w0 = np.array([rng.gaussian() for _ in range(8)])
    net = O.init_params([8, 64], w0, rng)
    x = random_mat(37, 8, 7)
    assert max_rel_dev(O.fused_forward(net.dims, O.build_plan(net), x), x @ w0) < 1e-15


def test_fused_matches_reference_b3840(O):  # :87-95
    for seed in range(3):
        net = random_net_fused([8, 64, 64, 64], 100 + seed)
        x = random_mat(3840, 8, 200 + seed)
        assert max_rel_dev(O.fused_forward(net.dims, O.build_plan(net), x), _ref_fwd(net, x)) < 1e-12


def test_fused_single_neuron(O):  # :97-110
    net = O.init_params([1, 1], np.zeros(1), O.Rng(8))
    (W, _), final = net.layers()[0][0], net.layers()[1]
    W[0, 0] = 1.0
    final[0] = 1.0
    buf = O.build_plan(net)
    assert O.fused_forward(net.dims, buf, np.array([[3.0]]))[0] == 3.0
    assert O.fused_forward(net.dims, buf, np.array([[-2.0]]))[0] == 0.0


def test_fallback_wide_layer(O):  # :112-119
    net = random_net_fused([8, 256], 9)
    x = random_mat(513, 8, 10)
    assert max_rel_dev(O.fused_forward(net.dims, O.build_plan(net), x), _ref_fwd(net, x)) < 1e-12


def test_f32_path_within_tolerance(O):  # :121-131
    net = random_net_fused([8, 64, 64, 64], 11)
    x = random_mat(512, 8, 12)
    ref = _ref_fwd(net, x)
    got = O.fused_forward_f32(net.dims, O.build_plan(net), x)
    scale = max(1.0, np.max(np.abs(ref)))
    assert np.max(np.abs(got.astype(np.float64) - ref)) / scale < 1e-5


def test_repeat_bit_identical(O):  # :146-153
    net = random_net_fused([8, 64, 64], 15)
    x = random_mat(333, 8, 16)
    buf = O.build_plan(net)
    assert np.array_equal(O.fused_forward(net.dims, buf, x), O.fused_forward(net.dims, buf, x))
