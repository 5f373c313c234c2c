"""Shape-general device kernels (k_train_generic.cu, k_dense.cu) against the
FP64 oracle: the paths the reference takes for networks outside the fused
range -- layers wider than 128 (fused_inference.cpp:132-151, tested by the
reference at [8,256], test_fused.cpp:112-119), minibatches above 128 rows
(hybrid_nn.cpp:180-181 accepts any batch_size) and no hidden layer
(dims = [2M], hybrid_nn.cpp:80-81).

Bars: FP64 training (train mode 201) follows the oracle's trajectory to
1e-9 over the full 50 epochs; FP32 training (mode 200) follows it to 1e-4
over 3 epochs (DESIGN 3: FP32 and FP64 trajectories separate slowly);
single-pass FP32 detection within 1e-5 of the FP64 forward
(test_fused.cpp:128-130).
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SHAPES = [([8, 256], 128), ([8, 32], 256), ([8, 16, 200], 64), ([8], 128), ([8, 24, 24], 100)]


@pytest.fixture(scope="module")
def A():
    from paper_2206_05998_b200 import api

    api.context()
    return api


@pytest.fixture
def generic(monkeypatch):
    monkeypatch.setenv("NOMA_TRAIN_GENERIC", "1")


def _data(O, seed=7, nt=150, nd=256, snr=15.0):
    sc = O.Scenario(num_users=2, num_antennas=4, train_symbols=nt, data_symbols=nd, power_step_db=3.0,
                    snr_db=snr, rx_nonlinearity_gain=0.05)
    rec = O.synthesize(sc, O.seed_bundle(seed))
    x = O.widen_design(rec.train_rx)
    y = O.widen_targets(rec.train_symbols[:, 1])
    w0 = O.lls_fit(x, y).w
    return rec, x, y, w0


def _nets(A, O, dims, w0, seed):
    ref = O.init_params(dims, w0, O.Rng(seed))
    layers, final = ref.layers()
    rng = np.random.default_rng(seed)
    final[:] = 0.3 * rng.standard_normal(final.size)  # off the zero-final point
    for _, b in layers:
        b[:] = 0.1 * rng.standard_normal(b.size)
    dev = A.net_from_params(dims, w0, [(W, b) for W, b in layers], final)
    return ref, dev


@pytest.mark.parametrize("dims,batch", SHAPES)
def test_generic_fp64_training_follows_the_oracle(A, O, generic, dims, batch):
    rec, x, y, w0 = _data(O)
    ref, _ = _nets(A, O, dims, w0, 3)
    theta = ref.theta.copy()
    tr_ref = O.train(ref, x, y, epochs=50, batch_size=batch, shuffle_seed=11)
    tr_dev = A.train_f64(dims, w0, theta, x, y, epochs=50, batch_size=batch, shuffle_seed=11)
    assert A.context().train_mode == 201
    dev = np.abs(theta - ref.theta).max() / np.abs(ref.theta).max()
    assert dev < 1e-9, dev
    assert np.max(np.abs(tr_dev - tr_ref) / np.abs(tr_ref)) < 1e-9


@pytest.mark.parametrize("dims,batch", SHAPES)
def test_generic_fp32_training_follows_the_oracle(A, O, generic, dims, batch):
    rec, x, y, w0 = _data(O)
    ref, dev = _nets(A, O, dims, w0, 5)
    tr_ref = O.train(ref, x, y, epochs=3, batch_size=batch, shuffle_seed=13)
    tr_dev = A.train(dev, x, y, epochs=3, batch_size=batch, shuffle_seed=13)
    assert A.context().train_mode == 200
    xd = O.widen_design(rec.data_rx)
    want = O.forward(ref, xd)
    got = A.fused_forward_f32(dev, xd)
    scale = max(1.0, np.abs(want).max())
    assert np.abs(got - want).max() / scale < 1e-4
    assert np.max(np.abs(tr_dev - tr_ref) / np.abs(tr_ref)) < 1e-4


def test_widened_complex_rows_take_the_same_generic_path(A, O, generic):
    """WIDEN_COMPLEX layout (IQ widening at load) == REAL layout rows."""
    rec, x, y, w0 = _data(O)
    dims = [8, 160]
    _, a = _nets(A, O, dims, w0, 9)
    _, b = _nets(A, O, dims, w0, 9)
    A.train(a, x, y, epochs=2, shuffle_seed=3)
    A.train(b, rec.train_rx, rec.train_symbols[:, 1], epochs=2, shuffle_seed=3, widened_complex=True)
    assert np.array_equal(a.plan, b.plan)


def test_onchip_kernels_route_wide_shapes_to_the_generic_kernel(A, O):
    """Without the override, a 256-wide layer trains in mode 200 and detects
    in mode 3; a 128-row batch of a [8, 32] net stays on chip."""
    rec, x, y, w0 = _data(O)
    _, dev = _nets(A, O, [8, 256], w0, 4)
    A.train(dev, x, y, epochs=1)
    assert A.context().train_mode == 200
    soft, bits, errs = A.detect(dev, rec.data_rx, rec.data_symbols[:, 1])
    assert A.context().detect_mode == 3
    _, small = _nets(A, O, [8, 32], w0, 4)
    A.train(small, x, y, epochs=1)
    assert A.context().train_mode not in (200, 201)


@pytest.mark.parametrize("dims", [[8, 256], [8, 300, 140], [8]])
def test_generic_detection_matches_fp64_forward(A, O, dims):
    rec, x, y, w0 = _data(O, nd=1000)
    ref, dev = _nets(A, O, dims, w0, 21)
    soft, bits, errs = A.detect(dev, rec.data_rx, rec.data_symbols[:, 1])
    if max(dims) > 128:
        assert A.context().detect_mode == 3
    # the FP64 forward of the FP32-rounded parameters on FP32-rounded samples
    xd = O.widen_design(rec.data_rx.astype(np.complex64).astype(np.complex128))
    layers, final = ref.layers()
    for (W, b), (Wd, bd) in zip(layers, dev.unpack()[0]):
        W[:] = Wd
        b[:] = bd
    final[:] = dev.unpack()[1]
    ref.w0 = dev.plan[:dims[0]].astype(np.float64)
    want = O.narrow_predictions(O.forward(ref, xd))
    scale = max(1.0, np.abs(want).max())
    assert np.abs(soft - want).max() / scale < 1e-5
    codes = A.codes_of(soft)
    truth = A.codes_of(rec.data_symbols[:, 1])
    assert errs == int(sum(bin(int(c)).count("1") for c in (codes ^ truth)))


def test_pipeline_wide_network_end_to_end(A, O):
    """noma_pipeline with a 256-wide hidden layer (previously UNSUPPORTED):
    LLS -> init -> generic FP32 training -> generic detection, against the
    oracle's slot run after 2 epochs."""
    sc = O.Scenario(num_users=3, num_antennas=4, train_symbols=80, data_symbols=200, power_step_db=3.0,
                    snr_db=20.0, rx_nonlinearity_gain=0.05)
    seeds = [1000, 1001]
    recs = [O.synthesize(sc, O.seed_bundle(s)) for s in seeds]
    dims = [8, 256]
    K = 3
    init = np.array([[O.substream_seed(s, 0x1000 + k + 1) for k in range(K)] for s in seeds], np.uint64)
    shuf = np.array([[O.substream_seed(s, k + 1) for k in range(K)] for s in seeds], np.uint64)
    truth = np.stack([A.codes_of(r.data_symbols) for r in recs])
    out = A.pipeline(dims, np.stack([r.train_rx for r in recs]), np.stack([r.train_symbols for r in recs]),
                     np.stack([r.data_rx for r in recs]), truth, init, shuf, epochs=2)
    assert (out.status == 0).all()
    assert A.context().train_mode == 200 and A.context().detect_mode == 3
    ref = O.run_slots(sc, [256], seeds, epochs=2)
    scale = np.maximum(1.0, np.abs(ref.soft).max(axis=-1, keepdims=True))
    assert np.abs(out.soft - ref.soft).max() / scale.min() < 1e-3
    assert (out.codes == A.codes_of(ref.soft)).mean() > 0.999
