"""GPU parity: init / fused FP32 training / detection kernels against the FP64
oracle and the reference suites test_hybrid_nn.cpp and test_fused.cpp, all
through the C-ABI.

Tolerances (stated):
  * inference with identical weights: |soft - ref| <= 1e-5 * max(1, max|ref|)
    (test_fused.cpp:128-130, the reference's own FP32 tolerance);
  * FP32-trained vs FP64-trained (oracle) networks: short trainings (<= 5
    epochs) soft outputs within SOFT_TOL_SHORT * max(1, max|ref|); full
    trainings within SOFT_TOL_LONG -- FP32 Adam (lr/eps = 5e5 gain) through
    ReLU kinks bifurcates from the FP64 trajectory: an independent numpy FP32
    restatement of the same algorithm deviates from FP64 by up to 1.2e-2 on the
    C1 weakest user, so SOFT_TOL_LONG = 1e-1; hard
    decisions identical on >= 99.99 % of symbols, |delta BER| <= flips / (2 N_D),
    loss trace within TRACE_TOL relative.  Measured on B200 (profiles/parity_r01.md):
    <= 5e-7 soft deviation up to 20 epochs, 4e-3..4e-2 after 50 epochs, 0 flips at 25 dB;
  * init weights equal to the FP64 draws rounded to FP32 within 1 ulp.
"""
import numpy as np
import pytest

from tests import refimpl as R
from tests.helpers import make_w0, random_mat, random_net_fused, record

pytestmark = pytest.mark.gpu
SOFT_TOL_SHORT = 1e-4
SOFT_TOL_LONG = 1e-1
TRACE_TOL = 1e-1
INFER_TOL = 1e-5


@pytest.fixture(scope="module")
def A():
    from paper_2206_05998_b200 import api

    api.context()
    return api


def _ref_fwd(net, x):
    layers, final = net.layers()
    return R.reference_forward(net.dims, net.w0, layers, final, x)


def _dev_net(A, onet):
    layers, final = onet.layers()
    return A.net_from_params(onet.dims, onet.w0, layers, final)


# ----------------------------------------------------------------- init
@pytest.mark.parametrize("dims,seed", [([8, 64, 64, 64], 3), ([32, 64, 64], 17), ([128, 64], 5),
                                       ([4, 3, 2], 21), ([1, 1], 1)])
def test_init_matches_oracle_draws(A, O, dims, seed):
    w0 = make_w0(dims[0], 11)
    onet = O.init_params(dims, w0, O.Rng(seed))
    dnet = A.init_params(dims, w0, seed)
    layers_d, final_d = dnet.unpack()
    layers_o, final_o = onet.layers()
    for (Wd, bd), (Wo, bo) in zip(layers_d, layers_o):
        want = Wo.astype(np.float32).astype(np.float64)
        ulp = np.abs(np.spacing(Wo.astype(np.float32))).astype(np.float64)
        assert np.all(np.abs(Wd - want) <= ulp)
        assert not bd.any()
    assert not final_d.any()
    assert np.array_equal(dnet.plan[:dims[0]], w0.astype(np.float32))


def test_param_count(A):
    dnet = A.init_params([8, 64, 64, 64], make_w0(8, 17), 9)
    assert dnet.trainable_count() == 8 * 64 + 64 + 64 * 64 + 64 + 64 * 64 + 64 + 64


# ------------------------------------------------------------ inference
def test_init_output_equals_lls_branch(A, O):
    rec = O.synthesize(O.Scenario(num_users=2, num_antennas=4, train_symbols=64,
                                  data_symbols=32, seed=121))
    w0 = O.lls_fit(O.widen_design(rec.train_rx), O.widen_targets(rec.train_symbols[:, 0])).w
    net = A.init_params([8, 16], w0, 122)
    soft, _, _ = A.detect(net, rec.data_rx)
    lin = O.narrow_predictions(O.widen_design(rec.data_rx) @ w0)
    assert np.max(np.abs(soft - lin)) <= INFER_TOL * max(1.0, np.max(np.abs(lin)))


def test_single_neuron_hand_case(A):
    net = A.net_from_params([1, 1], np.zeros(1), [(np.ones((1, 1)), np.zeros(1))], np.ones(1))
    out = A.fused_forward_f32(net, np.array([[3.0], [-2.0]]))
    assert out[0] == 3.0 and out[1] == 0.0


@pytest.mark.parametrize("dims,B", [([8, 64, 64, 64], 3840), ([32, 64, 64], 1000),
                                    ([32, 64], 513), ([128, 64], 300), ([64, 64], 777),
                                    ([8, 64, 48, 64], 333), ([8], 50), ([3, 5, 7], 129)])
def test_fused_f32_matches_reference(A, O, dims, B):
    onet = random_net_fused(dims, 100 + B)
    x = random_mat(B, dims[0], 200 + B)
    ref = _ref_fwd(onet, x)
    got = A.fused_forward_f32(_dev_net(A, onet), x)
    scale = max(1.0, np.max(np.abs(ref)))
    assert np.max(np.abs(got.astype(np.float64) - ref)) / scale < INFER_TOL


def test_detect_widened_matches_reference(A, O):
    onet = random_net_fused([32, 64, 64], 7)
    rows = random_mat(3840, 16, 8) + 1j * random_mat(3840, 16, 9)
    ref = O.narrow_predictions(_ref_fwd(onet, O.widen_design(rows)))
    truth = rows[:, 0]
    soft, bits, errs = A.detect(_dev_net(A, onet), rows, truth_symbols=truth)
    scale = max(1.0, np.max(np.abs(ref)))
    assert np.max(np.abs(soft - ref)) / scale < INFER_TOL
    assert np.array_equal(bits, O.hard_decision_qpsk(soft.astype(np.complex128)))
    assert errs == int(np.count_nonzero(bits != O.hard_decision_qpsk(truth)))


def test_repeat_bit_identical(A):
    onet = random_net_fused([8, 64, 64], 15)
    from oracle import oracle as O  # noqa: F401

    x = random_mat(333, 8, 16)
    net = _dev_net(A, onet)
    assert np.array_equal(A.fused_forward_f32(net, x), A.fused_forward_f32(net, x))


def test_wide_layer_runs_the_shape_general_path(A, O):
    """[8, 256] (test_fused.cpp:112-119): the single-pass kernel with an
    adaptive tile height (detect mode 3) within the FP32 bar of the FP64
    forward."""
    onet = random_net_fused([8, 256], 9)
    x = random_mat(513, 8, 10)
    got = A.fused_forward_f32(_dev_net(A, onet), x)
    assert A.context().detect_mode == 3
    want = O.forward(onet, x)
    assert np.abs(got - want).max() / max(1.0, np.abs(want).max()) < 1e-5


# ------------------------------------------------------------- training
def _train_pair(A, O, sc, k, dims, epochs, seed_init, shuffle_seed):
    rec = O.synthesize(sc)
    x = O.widen_design(rec.train_rx)
    y = O.widen_targets(rec.train_symbols[:, k])
    w0 = O.lls_fit(x, y).w
    onet = O.init_params(dims, w0, O.Rng(seed_init))
    dnet = A.init_params(dims, w0, seed_init)
    otrace = O.train(onet, x, y, epochs=epochs, shuffle_seed=shuffle_seed)
    dtrace = A.train(dnet, rec.train_rx, rec.train_symbols[:, k], epochs=epochs,
                     shuffle_seed=shuffle_seed, widened_complex=True)
    return rec, onet, dnet, otrace, dtrace


def test_train_zero_epochs_and_trace_length(A, O):
    rec = O.synthesize(O.Scenario(num_users=2, num_antennas=4, train_symbols=64, data_symbols=8,
                                  seed=81))
    x = O.widen_design(rec.train_rx)
    y = O.widen_targets(rec.train_symbols[:, 0])
    w0 = O.lls_fit(x, y).w
    net = A.init_params([8, 16], w0, 82)
    before = net.plan.copy()
    assert A.train(net, x, y, epochs=0).size == 0
    assert np.array_equal(net.plan, before)
    assert A.train(net, x, y, epochs=5).size == 5


def test_train_noiseless_stays_at_lls_optimum(A, O):
    rec, onet, dnet, otrace, dtrace = _train_pair(
        A, O, O.Scenario(num_users=2, num_antennas=4, train_symbols=685, data_symbols=8, seed=91),
        1, [8, 64, 64, 64], 50, 92, 93)
    assert dtrace.size == 50
    assert dtrace[-1] <= dtrace[0] + 1e-12
    assert dtrace[-1] <= 1e-6


def test_w0_frozen_and_determinism(A, O):
    rec = O.synthesize(O.Scenario(train_symbols=128, data_symbols=8, snr_db=25.0, seed=111))
    x = O.widen_design(rec.train_rx)
    y = O.widen_targets(rec.train_symbols[:, 0])
    w0 = O.lls_fit(x, y).w
    a = A.init_params([8, 16, 16], w0, 112)
    b = A.init_params([8, 16, 16], w0, 112)
    w0_slot = a.plan[:8].copy()
    A.train(a, x, y, epochs=6, shuffle_seed=7)
    A.train(b, x, y, epochs=6, shuffle_seed=7)
    assert np.array_equal(a.plan, b.plan)
    assert np.array_equal(a.plan[:8], w0_slot)


def test_detect_zero_branch_and_trained_recovery(A, O):
    rec = O.synthesize(O.Scenario(num_users=2, num_antennas=4, train_symbols=64, data_symbols=32,
                                  seed=121))
    x = O.widen_design(rec.train_rx)
    y = O.widen_targets(rec.train_symbols[:, 0])
    w0 = O.lls_fit(x, y).w
    net = A.init_params([8, 16], w0, 122)
    A.train(net, x, y, epochs=10)
    soft, bits, errs = A.detect(net, rec.data_rx, truth_symbols=rec.data_symbols[:, 0])
    assert errs == 0
    assert np.array_equal(bits, O.hard_decision_qpsk(rec.data_symbols[:, 0]))


def test_error_paths(A):
    from paper_2206_05998_b200 import native as N

    with pytest.raises(N.DimensionError):
        A.init_params([8, 16], make_w0(4, 1), 2)
    net = A.init_params([4, 8], make_w0(4, 1), 2)
    with pytest.raises(N.DimensionError):
        A.fused_forward_f32(net, np.zeros((2, 5)))
    with pytest.raises(N.DimensionError):
        A.train(net, np.zeros((0, 4)), np.zeros(0))
    with pytest.raises(N.ConfigError):
        A.train(net, np.ones((4, 4)), np.ones(4), batch_size=0)


@pytest.mark.parametrize("M,K,k,hidden,snr,epochs", [
    (4, 2, 1, [8], 20.0, 5),
    (16, 6, 5, [64], 25.0, 5),         # C1 shape, weakest user, short
    (16, 6, 5, [64, 64], 25.0, 5),     # C2 shape, short
    (16, 6, 5, [64], 25.0, 50),        # C1 shape, full training
    (16, 6, 0, [64], 25.0, 50),        # C1 shape, strongest user
    (16, 6, 5, [64, 64], 25.0, 50),    # C2 shape, weakest user
    (16, 6, 3, [64, 64], 10.0, 20),    # low SNR: decisions stressed
    (16, 6, 5, [64], 8.0, 20),         # very low SNR: BER > 0
    (32, 16, 15, [64, 64], 25.0, 5),   # C5 shape
    (64, 32, 31, [64], 25.0, 2),       # C4 shape (input width 128)
])
def test_fp32_training_tracks_fp64_reference(A, O, M, K, k, hidden, snr, epochs):
    sc = O.Scenario(num_users=K, num_antennas=M, train_symbols=685, data_symbols=3840,
                    power_step_db=3.0 if K <= 6 else 1.0, snr_db=snr, rx_nonlinearity_gain=0.05,
                    seed=1000 + M + k)
    dims = [2 * M] + hidden
    rec, onet, dnet, otrace, dtrace = _train_pair(A, O, sc, k, dims, epochs, 77, 78)
    trace_dev = float(np.max(np.abs(dtrace - otrace) / np.abs(otrace)))
    ref = O.detect(onet, O.widen_design(rec.data_rx))
    soft, bits, errs = A.detect(dnet, rec.data_rx, truth_symbols=rec.data_symbols[:, k])
    scale = max(1.0, np.max(np.abs(ref)))
    dev = np.max(np.abs(soft - ref)) / scale
    rbits = O.hard_decision_qpsk(ref)
    flips = int(np.count_nonzero(np.any(bits != rbits, axis=1)))
    ref_err = int(np.count_nonzero(rbits != O.hard_decision_qpsk(rec.data_symbols[:, k])))
    record("fp32_training", config=str((M, K, k, hidden, snr, epochs)), soft_dev=dev,
           trace_dev=trace_dev, flips=flips, symbols=len(ref), dev_bit_errors=errs,
           ref_bit_errors=ref_err)
    assert trace_dev <= (1e-4 if epochs <= 5 else TRACE_TOL), trace_dev
    assert abs(errs - ref_err) <= 2 * flips
    if epochs <= 5 or snr >= 10.0:
        assert dev < (SOFT_TOL_SHORT if epochs <= 5 else SOFT_TOL_LONG), dev
        assert flips <= 1e-4 * len(ref) + 0.5, flips
    else:
        # below 10 dB a bifurcated FP32 trajectory moves the many near-zero soft
        # outputs: decisions agree statistically, BER within 3 binomial sigma
        p = max(ref_err, 1) / (2 * len(ref))
        assert flips <= 0.02 * len(ref), flips
        assert abs(errs - ref_err) <= 3 * np.sqrt(2 * len(ref) * p * (1 - p)) + 1


def test_init_params_state_advances_the_callers_rng(A, O):
    """init_params(dims, w0, Rng&) (hybrid_nn.hpp:55): FP64 weights equal the
    oracle's draws and the caller's stream is advanced identically."""
    dims = [8, 16, 4]
    w0 = make_w0(8, 3)
    r = O.Rng(44)
    onet = O.init_params(dims, w0, r)
    net, theta, state = A.init_params_state(dims, w0, O.Rng(44).state())
    assert state == r.state()
    assert np.max(np.abs(theta - onet.theta)) <= 4e-16 * np.max(np.abs(onet.theta))


def test_lls_predict_fp64(A, O):
    rec = O.synthesize(O.Scenario(train_symbols=64, data_symbols=300, snr_db=20.0, seed=31))
    xt = O.widen_design(rec.train_rx)
    w = O.lls_fit(xt, O.widen_targets(rec.train_symbols[:, 2])).w
    xd = O.widen_design(rec.data_rx)
    got = A.lls_predict(w, xd)
    ref = O.narrow_predictions(xd @ w)
    assert np.max(np.abs(got - ref)) <= 1e-13 * np.max(np.abs(ref))
    # coordinate selector / zero weights (test_lls.cpp:58-73)
    x = np.array([[1 + 2j, 3 + 4j], [-1 + 0.5j, 0 + 1j], [2 - 2j, 1 + 1j]])
    sel = np.array([1.0, 0, 0, 0])
    assert np.array_equal(A.lls_predict(sel, O.widen_design(x)), x[:, 0])
    assert np.array_equal(A.lls_predict(np.zeros(4), O.widen_design(x)), np.zeros(3, complex))
