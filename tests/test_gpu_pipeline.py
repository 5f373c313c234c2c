"""GPU parity of the whole slot pipeline (noma_pipeline: LLS -> init -> fused
training -> streaming detection) and of the device channel synthesiser,
against the FP64 oracle's slot run (noma_cli.cpp:86-160 composition)."""
import numpy as np
import pytest

from tests.helpers import record

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def A():
    from paper_2206_05998_b200 import api

    api.context()
    return api


def _seeds(O, seeds, K):
    init = np.array([[O.substream_seed(s, 0x1000 + k + 1) for k in range(K)] for s in seeds],
                    np.uint64)
    shuf = np.array([[O.substream_seed(s, k + 1) for k in range(K)] for s in seeds], np.uint64)
    return init, shuf


@pytest.mark.parametrize("M,K,hidden,snr,epochs,S", [
    (4, 3, [16], 20.0, 3, 2),
    (16, 6, [64], 25.0, 50, 2),      # C1
    (16, 6, [64, 64], 25.0, 10, 1),  # C2 shape (fewer epochs to bound oracle time)
    (16, 6, [64], 8.0, 20, 2),       # low SNR: non-zero BER
])
def test_pipeline_matches_oracle(A, O, M, K, hidden, snr, epochs, S):
    sc = O.Scenario(num_users=K, num_antennas=M, train_symbols=685 if M > 4 else 64,
                    data_symbols=3840 if M > 4 else 256, power_step_db=3.0, snr_db=snr,
                    rx_nonlinearity_gain=0.05)
    seeds = [1000 + s for s in range(S)]
    recs = [O.synthesize(sc, O.seed_bundle(s)) for s in seeds]
    ref = O.run_slots(sc, hidden, seeds, epochs=epochs, threads=8)
    dims = [2 * M] + hidden
    init, shuf = _seeds(O, seeds, K)
    truth = np.stack([A.codes_of(r.data_symbols) for r in recs])
    out = A.pipeline(dims, np.stack([r.train_rx for r in recs]),
                     np.stack([r.train_symbols for r in recs]),
                     np.stack([r.data_rx for r in recs]), truth, init, shuf, epochs=epochs)
    assert (out.status == 0).all()
    werr = np.max(np.abs(out.w0 - ref.w0)) / np.max(np.abs(ref.w0))
    assert werr < 1e-10
    assert np.all(np.abs(out.gram_condition - ref.gram_condition) <= 1e-6 * ref.gram_condition)
    scale = max(1.0, np.max(np.abs(ref.soft)))
    soft_dev = np.max(np.abs(out.soft - ref.soft)) / scale
    rcodes = A.codes_of(ref.soft)
    flips = int(np.count_nonzero(out.codes != rcodes))
    trace_dev = float(np.max(np.abs(out.trace - ref.trace) / np.abs(ref.trace)))
    record("pipeline", config=str((M, K, hidden, snr, epochs, S)), w0_dev=werr, soft_dev=soft_dev,
           trace_dev=trace_dev, flips=flips, symbols=out.codes.size,
           dev_bit_errors=int(out.bit_errors.sum()), ref_bit_errors=int(ref.bit_errors.sum()))
    assert soft_dev < (1e-4 if epochs <= 5 else 1e-1), soft_dev
    assert flips <= 1e-4 * out.codes.size + 0.5, flips
    assert np.all(np.abs(out.bit_errors.astype(np.int64) - ref.bit_errors) <= 2 * flips)
    assert trace_dev <= (1e-4 if epochs <= 5 else 1e-1), trace_dev


def test_pipeline_lls_paths_match_lls_fit(A, O):
    # The pipeline's LLS solves by Cholesky (Jacobi fallback for slots whose
    # pivots approach the rank threshold) and takes the condition numbers
    # from a Jacobi-only launch overlapping training; noma_lls_fit runs the
    # Jacobi path throughout.  Same slots -> same status, bitwise-equal
    # condition numbers, w0 within 1e-10 relative (test_lls.cpp:40).
    rng = np.random.default_rng(11)
    S, NT, M, K, ND = 4, 96, 4, 3, 32
    x = rng.normal(size=(S, NT, M)) + 1j * rng.normal(size=(S, NT, M))
    x[1] *= np.array([1.0, 0.1, 0.03, 1.0])           # near-far columns: larger condition
    x[2, :, 3] = x[2, :, 0]                            # exactly rank deficient (Jacobi fallback) ...
    c = rng.normal(size=(S, M, K)) + 1j * rng.normal(size=(S, M, K))
    y = np.einsum("stm,smk->stk", x, c)                # ... but consistent: min-norm, status OK
    y[[0, 1, 3]] += 0.01 * (rng.normal(size=(3, NT, K)) + 1j * rng.normal(size=(3, NT, K)))
    init, shuf = _seeds(O, [1, 2, 3, 4], K)
    out = A.pipeline([2 * M, 8], x, y, np.zeros((S, ND, M), np.complex64),
                     np.zeros((S, ND, K), np.uint8), init, shuf, epochs=0)
    w0, cond, status = A.lls_fit_slots(x, y)
    assert np.array_equal(out.status, status) and (status == 0).all()
    assert np.array_equal(out.gram_condition, cond)
    assert cond[1].min() > 10 * cond[0].max()          # the near-far slot is the worse conditioned
    werr = np.abs(out.w0 - w0).max(axis=-1) / np.abs(w0).max(axis=-1)
    assert werr.max() <= 1e-10, werr


def test_jacobi_path_slot_trains_like_the_oracle(A, O):
    # A consistent rank-deficient slot takes the LLS's Jacobi path (min-norm
    # w0, status OK) next to a full-rank Cholesky-path slot: its residuals
    # come from the in-kernel pass, the other's from the r0 kernel, and both
    # w0 go straight into the plans.  Three epochs of training and detection
    # against the FP64 oracle's lls_fit -> init_params -> train -> detect:
    # the full-rank slot to 1e-4; the consistent slot's residual targets are
    # rounding noise (~1e-15), which Adam turns into full-size steps, so its
    # network part is chaotic in FP32 and only the LLS-dominated output is
    # compared (w0 to 1e-10, soft to 2e-2).
    rng = np.random.default_rng(21)
    S, NT, M, K, ND, dims = 2, 96, 4, 2, 64, [8, 16]
    x = rng.normal(size=(S, NT, M)) + 1j * rng.normal(size=(S, NT, M))
    x[1, :, 3] = x[1, :, 0]                            # rank 3 of 4: Jacobi path
    c = rng.normal(size=(S, M, K)) + 1j * rng.normal(size=(S, M, K))
    y = np.einsum("stm,smk->stk", x, c)                # slot 1 consistent: min-norm, OK
    y[0] += 0.05 * (rng.normal(size=(NT, K)) + 1j * rng.normal(size=(NT, K)))
    xd = (rng.normal(size=(S, ND, M)) + 1j * rng.normal(size=(S, ND, M))).astype(np.complex64)
    init, shuf = _seeds(O, [41, 42], K)
    out = A.pipeline(dims, x, y, xd, np.zeros((S, ND, K), np.uint8), init, shuf, epochs=3)
    assert (out.status == 0).all()
    for s in range(S):
        wx = O.widen_design(x[s])
        for k in range(K):
            wy = O.widen_targets(y[s][:, k])
            lls = O.lls_fit(wx, wy)
            net = O.init_params(dims, lls.w, O.Rng(int(init[s, k])))
            O.train(net, wx, wy, epochs=3, batch_size=128, lr=0.005, shuffle_seed=int(shuf[s, k]))
            ref = O.detect(net, O.widen_design(xd[s].astype(np.complex128)))
            wdev = np.max(np.abs(out.w0[s, k] - lls.w)) / np.max(np.abs(lls.w))
            dev = np.max(np.abs(out.soft[s, k] - ref)) / max(1.0, np.max(np.abs(ref)))
            record("jacobi_path_training", config=f"slot={s} user={k}", soft_dev=dev, w0_dev=wdev)
            assert wdev < 1e-10, (s, k, wdev)
            assert dev < (1e-4 if s == 0 else 2e-2), (s, k, dev)


def test_ill_conditioned_slot_is_flagged(A, O):
    # duplicate antennas -> rank-deficient complex design; random targets are
    # inconsistent -> status ILL for every user, no training for them.
    rng = np.random.default_rng(0)
    NT, M, K, ND = 64, 4, 2, 32
    x = rng.normal(size=(NT, M)) + 1j * rng.normal(size=(NT, M))
    x[:, 1] = x[:, 0]
    y = rng.normal(size=(NT, K)) + 1j * rng.normal(size=(NT, K))
    init, shuf = _seeds(O, [5], K)
    out = A.pipeline([8, 8], x[None], y[None], np.zeros((1, ND, M), np.complex64),
                     np.zeros((1, ND, K), np.uint8), init, shuf, epochs=2)
    assert (out.status == 3).all()
    assert (out.gram_condition > 1e12).all()
    assert (out.bit_errors == 0xFFFFFFFF).all()


@pytest.mark.parametrize("K,M,NT,ND,snr,gain", [(6, 16, 685, 3840, 25.0, 0.05),
                                               (3, 2, 16, 64, float("inf"), 0.0),
                                               (8, 4, 32, 100, 10.0, 0.0)])
def test_device_synthesis_matches_oracle(A, O, K, M, NT, ND, snr, gain):
    seeds = [7, 1000, 2**40 + 3]
    sy = A.synthesize(K, M, NT, ND, seeds, power_step_db=3.0, snr_db=snr, rx_nonlinearity_gain=gain)
    sc = O.Scenario(num_users=K, num_antennas=M, train_symbols=NT, data_symbols=ND,
                    power_step_db=3.0, snr_db=snr, rx_nonlinearity_gain=gain)
    for i, s in enumerate(seeds):
        rec = O.synthesize(sc, O.seed_bundle(s))
        assert np.array_equal(sy.pilot_sym[i], rec.train_symbols)          # integer stream: exact
        assert np.array_equal(sy.data_codes[i], A.codes_of(rec.data_symbols))
        assert np.max(np.abs(sy.channel[i] - rec.channel)) <= 4e-16 * np.max(np.abs(rec.channel))
        assert np.max(np.abs(sy.pilot_rx[i] - rec.train_rx)) <= 1e-14 * np.max(np.abs(rec.train_rx))
        assert np.max(np.abs(sy.data_rx[i] - rec.data_rx.astype(np.complex64))) <= \
            1e-6 * np.max(np.abs(rec.data_rx))
        assert abs(sy.noise_power[i] - rec.noise_power) <= 1e-14 * max(rec.noise_power, 1e-300)


def test_large_detect_self_consistent(A, O):
    """C3-sized data phase (2^20 symbols): codes are the sign pattern of the
    soft outputs and the error count equals the code mismatches vs truth."""
    from tests.helpers import random_net_fused

    onet = random_net_fused([32, 64, 64], 3)
    layers, final = onet.layers()
    net = A.net_from_params(onet.dims, onet.w0, layers, final)
    sy = A.synthesize(6, 16, 32, 1 << 20, [11], snr_db=25.0, rx_nonlinearity_gain=0.05)
    truth = sy.data_rx[0][:, 0].astype(np.complex128)
    soft, bits, errs = A.detect(net, sy.data_rx[0], truth_symbols=truth)
    assert np.array_equal(bits, O.hard_decision_qpsk(soft.astype(np.complex128)))
    assert errs == int(np.count_nonzero(bits != O.hard_decision_qpsk(truth)))
    # spot-check a slice against the FP64 reference forward
    sl = slice(123456, 123456 + 2048)
    from tests import refimpl as R
    ref = O.narrow_predictions(R.reference_forward(onet.dims, onet.w0, layers, final,
                                                   O.widen_design(sy.data_rx[0][sl])))
    assert np.max(np.abs(soft[sl] - ref)) / max(1.0, np.max(np.abs(ref))) < 1e-5


@pytest.mark.parametrize("NT,l2", [(64, "1"), (100, "1"), (64, "0"), (100, "0")])
def test_throughput_kernel_c2_shape(A, O, NT, l2, monkeypatch):
    """The C2 network shape ([32, 64, 64], 78 nets) on the two-hidden-layer
    8-warp kernel (k_train_l2.cu, mode 5) and, with NOMA_TRAIN_L2=0, on the
    general one-CTA-per-net kernel (mode 1: idle warps summing the first
    layer's bias gradient, next minibatch staged into a dead activation
    region).  NT = 64: one minibatch per epoch, staging across epoch
    boundaries; NT = 100: a partial second minibatch.  Short trainings against
    the FP64 oracle."""
    monkeypatch.setenv("NOMA_TRAIN_L2", l2)
    sc = O.Scenario(num_users=6, num_antennas=16, train_symbols=NT, data_symbols=128,
                    power_step_db=3.0, snr_db=20.0, rx_nonlinearity_gain=0.05)
    S = 13  # 78 nets: the throughput kernel
    seeds = [3000 + s for s in range(S)]
    recs = [O.synthesize(sc, O.seed_bundle(s)) for s in seeds]
    ref = O.run_slots(sc, [64, 64], seeds, epochs=3, threads=8)
    init, shuf = _seeds(O, seeds, 6)
    out = A.pipeline([32, 64, 64], np.stack([r.train_rx for r in recs]),
                     np.stack([r.train_symbols for r in recs]), np.stack([r.data_rx for r in recs]),
                     np.stack([A.codes_of(r.data_symbols) for r in recs]), init, shuf, epochs=3)
    assert A.context().train_mode == (5 if l2 == "1" else 1)
    assert (out.status == 0).all()
    soft_dev = np.max(np.abs(out.soft - ref.soft)) / max(1.0, np.max(np.abs(ref.soft)))
    trace_dev = float(np.max(np.abs(out.trace - ref.trace) / np.abs(ref.trace)))
    record("throughput_c2_shape", config=f"NT={NT} l2={l2}", soft_dev=soft_dev, trace_dev=trace_dev)
    assert soft_dev < 1e-4 and trace_dev < 1e-4


@pytest.mark.parametrize("NT", [128, 75])
def test_throughput_kernel_l2_wide_input(A, O, NT):
    """The two-hidden-layer kernel at a 64-wide input ([64, 64, 64]: 32
    antennas, 8 users x 10 slots); NT = 75 (150 widened rows) leaves a
    22-row ragged minibatch at every epoch end."""
    sc = O.Scenario(num_users=8, num_antennas=32, train_symbols=NT, data_symbols=128,
                    power_step_db=2.0, snr_db=20.0, rx_nonlinearity_gain=0.05)
    S = 10
    seeds = [3500 + s for s in range(S)]
    recs = [O.synthesize(sc, O.seed_bundle(s)) for s in seeds]
    ref = O.run_slots(sc, [64, 64], seeds, epochs=3, threads=8)
    init, shuf = _seeds(O, seeds, 8)
    out = A.pipeline([64, 64, 64], np.stack([r.train_rx for r in recs]),
                     np.stack([r.train_symbols for r in recs]), np.stack([r.data_rx for r in recs]),
                     np.stack([A.codes_of(r.data_symbols) for r in recs]), init, shuf, epochs=3)
    assert A.context().train_mode == 5
    assert (out.status == 0).all()
    soft_dev = np.max(np.abs(out.soft - ref.soft)) / max(1.0, np.max(np.abs(ref.soft)))
    trace_dev = float(np.max(np.abs(out.trace - ref.trace) / np.abs(ref.trace)))
    record("throughput_l2_wide", config=f"NT={NT}", soft_dev=soft_dev, trace_dev=trace_dev)
    assert soft_dev < 1e-4 and trace_dev < 1e-4


@pytest.mark.parametrize("NT", [128, 150])
def test_throughput_kernel_c4_shape(A, O, NT):
    """The 8-warp kernel (k_train_w8.cu) at the C4 network shape ([128, 64],
    3 slots x 32 users): K split across the warp halves, gradient tiles over
    all 128 columns; NT = 150 (300 widened rows) ends every epoch on a ragged
    44-row minibatch.  Short trainings against the FP64 oracle."""
    sc = O.Scenario(num_users=32, num_antennas=64, train_symbols=NT, data_symbols=128,
                    power_step_db=1.0, snr_db=20.0, rx_nonlinearity_gain=0.05)
    S = 3
    seeds = [4000 + s for s in range(S)]
    recs = [O.synthesize(sc, O.seed_bundle(s)) for s in seeds]
    ref = O.run_slots(sc, [64], seeds, epochs=3, threads=8)
    init, shuf = _seeds(O, seeds, 32)
    out = A.pipeline([128, 64], np.stack([r.train_rx for r in recs]),
                     np.stack([r.train_symbols for r in recs]), np.stack([r.data_rx for r in recs]),
                     np.stack([A.codes_of(r.data_symbols) for r in recs]), init, shuf, epochs=3)
    assert A.context().train_mode == 4
    assert (out.status == 0).all()
    soft_dev = np.max(np.abs(out.soft - ref.soft)) / max(1.0, np.max(np.abs(ref.soft)))
    trace_dev = float(np.max(np.abs(out.trace - ref.trace) / np.abs(ref.trace)))
    record("throughput_c4_shape", config=f"NT={sc.train_symbols}", soft_dev=soft_dev, trace_dev=trace_dev)
    assert soft_dev < 1e-4 and trace_dev < 1e-4


@pytest.mark.parametrize("mode", ["1", "2", "4"])
def test_train_modes_agree(A, O, mode, monkeypatch):
    """The one-CTA-per-net kernel (throughput mode) and the cluster kernels
    (latency mode: 2 or 4 CTAs per net, gradients reduced over DSMEM) follow
    the FP64 oracle for short trainings; >74 nets also exercise the
    many-nets launch path."""
    monkeypatch.setenv("NOMA_TRAIN_CLUSTER", mode)
    sc = O.Scenario(num_users=6, num_antennas=4, train_symbols=64, data_symbols=128,
                    power_step_db=3.0, snr_db=20.0, rx_nonlinearity_gain=0.05)
    S = 13  # 78 nets
    seeds = [2000 + s for s in range(S)]
    recs = [O.synthesize(sc, O.seed_bundle(s)) for s in seeds]
    ref = O.run_slots(sc, [16, 16], seeds, epochs=3, threads=8)
    init, shuf = _seeds(O, seeds, 6)
    out = A.pipeline([8, 16, 16], np.stack([r.train_rx for r in recs]),
                     np.stack([r.train_symbols for r in recs]), np.stack([r.data_rx for r in recs]),
                     np.stack([A.codes_of(r.data_symbols) for r in recs]), init, shuf, epochs=3)
    assert (out.status == 0).all()
    soft_dev = np.max(np.abs(out.soft - ref.soft)) / max(1.0, np.max(np.abs(ref.soft)))
    trace_dev = float(np.max(np.abs(out.trace - ref.trace) / np.abs(ref.trace)))
    record("train_modes", config=f"cluster={mode}", soft_dev=soft_dev, trace_dev=trace_dev)
    assert soft_dev < 1e-4 and trace_dev < 1e-4


@pytest.mark.parametrize("where", ["host", "device"])
def test_pipeline_chunks_bit_identical(A, O, where, monkeypatch):
    """Slots run in chunks of bounded scratch (NOMA_CHUNK_MB); host buffers are
    uploaded per chunk on the copy stream and results downloaded per chunk.
    One slot per chunk must reproduce the one-chunk call bit for bit (slots
    are independent, kernels deterministic), including the SER counters."""
    import torch

    from paper_2206_05998_b200 import native as N

    K, M, NT, ND, S, dims, epochs = 3, 4, 64, 256, 7, [8, 16], 3
    sy = A.synthesize(K, M, NT, ND, [50 + s for s in range(S)], snr_db=12.0, rx_nonlinearity_gain=0.05)
    init, shuf = _seeds(O, [50 + s for s in range(S)], K)
    cfg = N.TrainCfg.of(epochs, 128, 0.005)
    ps = N.plan_size(dims)

    def run():
        if where == "host":
            out = A.pipeline(dims, sy.pilot_rx, sy.pilot_sym, sy.data_rx, sy.data_codes, init, shuf,
                             epochs=epochs)
            return [out.w0, out.gram_condition, out.plans, out.trace, out.soft, out.codes,
                    out.bit_errors, out.symbol_errors, out.status]
        dev = torch.device("cuda", 0)
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
        o = [torch.zeros((S, K, 2 * M), dtype=torch.float64, device=dev),
             torch.zeros((S, K), dtype=torch.float64, device=dev),
             torch.zeros((S, K, ps), dtype=torch.float32, device=dev),
             torch.zeros((S, K, epochs), dtype=torch.float64, device=dev),
             torch.zeros((S, K, ND, 2), dtype=torch.float32, device=dev),
             torch.zeros((S, K, ND), dtype=torch.uint8, device=dev),
             torch.zeros((S, K), dtype=torch.int32, device=dev),
             torch.zeros((S, K), dtype=torch.int32, device=dev),
             torch.zeros((S, K), dtype=torch.int32, device=dev)]
        A.context().pipeline(dims, cfg, S, K, M, NT, ND, t(sy.pilot_rx.view(np.float64)),
                             t(sy.pilot_sym.view(np.float64)), t(sy.data_rx.view(np.float32)),
                             t(sy.data_codes), t(init.view(np.int64)), t(shuf.view(np.int64)), o[8],
                             w0=o[0], cond=o[1], plans=o[2], trace=o[3], soft=o[4], codes=o[5],
                             bit_errors=o[6], symbol_errors=o[7])
        torch.cuda.synchronize()
        return [x.cpu().numpy() for x in o]

    one = run()
    monkeypatch.setenv("NOMA_CHUNK_MB", "0")  # budget 0 -> one slot per chunk
    many = run()
    for a, b in zip(one, many):
        assert np.array_equal(a, b)
    assert int(np.asarray(one[7]).sum()) > 0  # the low-SNR slots do make symbol errors
    # chunk ch+1's prologue issued beside chunk ch's training (double-buffered
    # scratch, NOMA_OVERLAP=1): the same bits
    monkeypatch.setenv("NOMA_OVERLAP", "1")
    over = run()
    for a, b in zip(one, over):
        assert np.array_equal(a, b)
    if where == "device":  # no w0 / plans requested: per-chunk scratch, double-buffered
        dev = torch.device("cuda", 0)
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
        soft = torch.zeros((S, K, ND, 2), dtype=torch.float32, device=dev)
        codes = torch.zeros((S, K, ND), dtype=torch.uint8, device=dev)
        errs = torch.zeros((S, K), dtype=torch.int32, device=dev)
        st = torch.zeros((S, K), dtype=torch.int32, device=dev)
        A.context().pipeline(dims, cfg, S, K, M, NT, ND, t(sy.pilot_rx.view(np.float64)),
                             t(sy.pilot_sym.view(np.float64)), t(sy.data_rx.view(np.float32)),
                             t(sy.data_codes), t(init.view(np.int64)), t(shuf.view(np.int64)), st,
                             soft=soft, codes=codes, bit_errors=errs)
        torch.cuda.synchronize()
        assert np.array_equal(soft.cpu().numpy(), one[4])
        assert np.array_equal(codes.cpu().numpy(), one[5])
        assert np.array_equal(errs.cpu().numpy(), one[6])
