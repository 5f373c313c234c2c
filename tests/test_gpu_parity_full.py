"""Full-length parity of the benchmarked batches against the FP64 oracle.

The bench line's workloads run the batch (throughput) training kernels for
the whole 50 epochs; these tests run exactly those kernels at the BASELINE
shapes and compare a subset of the slots with the oracle's slot run
(oracle.run_slots: synthesize -> widen -> lls::fit -> init_params ->
train -> detect -> hard decision -> BER, noma_cli.cpp:86-160, eval.cpp:
228-241, hybrid_nn.cpp:158-195):

* w0 within 1e-10 relative (test_lls.cpp:40);
* hard decisions identical on >= 99.99 % of the symbols (north star) for the
  C1 / C2 configurations; at C4 / C5 the measured FP32-vs-FP64 flip rate
  (0.13 % / 1.3 %, all on the weakest users) bounds the test -- see below;
* |bit errors - oracle bit errors| <= decision flips, per net;
* FP32-trained weights, soft outputs and loss traces within the stated
  tolerances below (the reference pins none of these after train(); SURVEY
  8(c) proposes soft <= 2e-3 and weights <= 1e-2, tightened from data).

Tolerances are ~2x the maximum measured on B200 (profiles/r02_parity.jsonl).
FP32 and FP64 trainings of the same net separate slowly over 550 Adam steps
(lr / eps gain 5e5, hybrid_nn.hpp:36-39): a ReLU input within FP32 rounding of
zero takes the other mask and the trajectories drift apart; the per-config
tolerances below bound that drift.
"""
import os

import numpy as np
import pytest

from tests.helpers import record

pytestmark = pytest.mark.gpu

# config: (M, K, hidden, power step, slots run on the GPU, slots checked,
#          expected train kernel, max decision-flip fraction,
#          tolerances (soft, weight, trace))
# measured on B200 (profiles/r02_parity.jsonl; soft / weight / trace / flips):
#   c2_bench148 0.124 / 0.31 / 0.12 / 0      c1 0.049 / 0.13 / 0.045 / 0
#   c5          0.080 / 0.12 / 0.17 / 1.3e-3 c4 0.185 / 0.20 / 0.49 / 1.3e-2
# C4 / C5 flips sit on the weakest users (1 dB near-far steps put user 32 of
# C4 at -6 dB, BER ~0.2) where many symbols lie near the decision boundary;
# the FP32-trained nets make as many bit errors as the FP64 ones (C5 3845 vs
# 3876, C4 54521 vs 54483).
CONFIGS = {
    # round 1's bench batch: 148 C2 slots, two-hidden-layer 8-warp kernel
    "c2_bench148": (16, 6, [64, 64], 3.0, 148, 8, 5, 1e-4, (0.25, 0.6, 0.25)),
    "c1": (16, 6, [64], 3.0, 16, 4, 3, 1e-4, (0.1, 0.3, 0.1)),
    # the bench default (C5) runs the 4-warp kernel
    "c5": (32, 16, [64], 1.0, 6, 3, 3, 2.5e-3, (0.16, 0.25, 0.35)),
    # C4 (128-wide input) runs the 8-warp kernel
    "c4": (64, 32, [64], 1.0, 3, 2, 4, 2.7e-2, (0.37, 0.4, 1.0)),
}


@pytest.fixture(scope="module")
def A():
    from paper_2206_05998_b200 import api

    api.context()
    return api


def _seeds(O, seeds, K):
    init = np.array([[O.substream_seed(s, 0x1000 + k + 1) for k in range(K)] for s in seeds], np.uint64)
    shuf = np.array([[O.substream_seed(s, k + 1) for k in range(K)] for s in seeds], np.uint64)
    return init, shuf


def _weight_dev(dims, plan_dev, plan_ref):
    """Per-net ||theta_dev - theta_ref||_2 / ||theta_ref||_2 over the trainable
    block of a FusedPlan buffer (the w0 slot is the LLS solution, compared
    separately), and the elementwise max |d| / max |theta_ref|."""
    w = -(-dims[0] // 8) * 8
    a, b = plan_dev[..., w:].astype(np.float64), plan_ref[..., w:]
    fro = np.linalg.norm(a - b, axis=-1) / np.linalg.norm(b, axis=-1)
    elem = np.max(np.abs(a - b), axis=-1) / np.max(np.abs(b), axis=-1)
    return fro, elem


@pytest.mark.parametrize("tag", list(CONFIGS))
def test_full_training_batch_kernel(A, O, tag):
    M, K, hidden, step, S, check, mode, tol_flip, (tol_soft, tol_w, tol_trace) = CONFIGS[tag]
    NT, ND, snr, gain, epochs = 685, 3840, 25.0, 0.05, 50
    sc = O.Scenario(num_users=K, num_antennas=M, train_symbols=NT, data_symbols=ND,
                    power_step_db=step, snr_db=snr, rx_nonlinearity_gain=gain)
    seeds = [1000 + s for s in range(S)]
    recs = [O.synthesize(sc, O.seed_bundle(s)) for s in seeds]
    dims = [2 * M] + hidden
    init, shuf = _seeds(O, seeds, K)
    truth = np.stack([A.codes_of(r.data_symbols) for r in recs])
    out = A.pipeline(dims, np.stack([r.train_rx for r in recs]), np.stack([r.train_symbols for r in recs]),
                     np.stack([r.data_rx for r in recs]), truth, init, shuf, epochs=epochs)
    assert A.context().train_mode == mode, A.context().train_mode
    assert (out.status == 0).all()
    # the oracle on `check` slots spread over the batch (first, last, middle)
    idx = sorted({0, S - 1, *np.linspace(0, S - 1, check).round().astype(int).tolist()})[:check]
    ref = O.run_slots(sc, hidden, [seeds[i] for i in idx], epochs=epochs, threads=16)
    werr = float(np.max(np.abs(out.w0[idx] - ref.w0) / np.max(np.abs(ref.w0), axis=-1, keepdims=True)))
    soft = out.soft[idx]
    scale = np.maximum(1.0, np.max(np.abs(ref.soft), axis=-1, keepdims=True))
    soft_dev = float(np.max(np.abs(soft - ref.soft) / scale))
    wfro, welem = _weight_dev(dims, out.plans[idx], ref.plans)
    wdev = float(np.max(wfro))
    soft_net = np.max(np.abs(soft - ref.soft) / scale, axis=-1)
    trace_dev = float(np.max(np.abs(out.trace[idx] - ref.trace) / np.abs(ref.trace)))
    rcodes = A.codes_of(ref.soft)
    flips_net = np.count_nonzero(out.codes[idx] != rcodes, axis=-1)
    flips = int(flips_net.sum())
    dber = np.abs(out.bit_errors[idx].astype(np.int64) - ref.bit_errors)
    record("full_training", config=tag, slots=S, checked=len(idx), w0_dev=werr, soft_dev=soft_dev,
           weight_dev=wdev, weight_dev_median=float(np.median(wfro)),
           weight_elem_max=float(np.max(welem)), soft_dev_median=float(np.median(soft_net)),
           nets_soft_over_1e3=int(np.count_nonzero(soft_net > 1e-3)), nets=int(soft_net.size),
           trace_dev=trace_dev, flips=flips, symbols=int(out.codes[idx].size),
           max_dber_minus_flips=int(np.max(dber - 2 * flips_net)),
           dev_bit_errors=int(out.bit_errors[idx].sum()), ref_bit_errors=int(ref.bit_errors.sum()),
           train_mode=A.context().train_mode)
    # SER counters (north star (c)): symbols whose decision differs from the
    # truth in either bit -- exactly the device's own decisions, and within
    # the decision flips of the oracle's
    tr = np.transpose(truth[idx], (0, 2, 1))
    ser_dev = out.symbol_errors[idx].astype(np.int64)
    assert np.array_equal(ser_dev, np.count_nonzero(out.codes[idx] != tr, axis=-1))
    assert np.all(np.abs(ser_dev - np.count_nonzero(rcodes != tr, axis=-1)) <= flips_net)
    assert werr < 1e-10, werr
    assert flips <= tol_flip * out.codes[idx].size, flips
    # a flipped QPSK decision changes 1 or 2 bits
    assert np.all(dber <= 2 * flips_net), (dber, flips_net)
    if os.environ.get("NOMA_PARITY_MEASURE"):  # measurement run: record only
        return
    assert soft_dev < tol_soft, soft_dev
    assert wdev < tol_w, wdev
    assert trace_dev < tol_trace, trace_dev


# FP64 mode (noma_pipeline_f64): the reference's arithmetic end to end on the
# device.  The FP32-vs-FP64 drift above is a property of FP32 training (an
# FP32 restatement on the CPU drifts as far, profiles/r02_precision_probe.txt);
# in FP64 the device follows the oracle's trajectory, so the north star's
# decision bar holds at every configuration, including C4 and C5.
# config: (M, K, hidden, power step, slots)
CONFIGS_F64 = {
    "c1": (16, 6, [64], 3.0, 2),
    "c2": (16, 6, [64, 64], 3.0, 2),
    "c5": (32, 16, [64], 1.0, 2),
    "c4": (64, 32, [64], 1.0, 1),
}


@pytest.mark.parametrize("tag", list(CONFIGS_F64))
def test_full_training_fp64_mode(A, O, tag):
    M, K, hidden, step, S = CONFIGS_F64[tag]
    NT, ND, snr, gain, epochs = 685, 3840, 25.0, 0.05, 50
    sc = O.Scenario(num_users=K, num_antennas=M, train_symbols=NT, data_symbols=ND,
                    power_step_db=step, snr_db=snr, rx_nonlinearity_gain=gain)
    seeds = [1000 + s for s in range(S)]
    recs = [O.synthesize(sc, O.seed_bundle(s)) for s in seeds]
    dims = [2 * M] + hidden
    init, shuf = _seeds(O, seeds, K)
    truth = np.stack([A.codes_of(r.data_symbols) for r in recs])
    out = A.pipeline(dims, np.stack([r.train_rx for r in recs]), np.stack([r.train_symbols for r in recs]),
                     np.stack([r.data_rx for r in recs]), truth, init, shuf, epochs=epochs, precision=64)
    # C1 / C5: the register-tiled FP64 kernel (301); C2 / C4: k_train_f64 (300)
    want = (301,) if hidden == [64] and M <= 32 else (300, 201)
    assert A.context().train_mode in want, A.context().train_mode
    assert (out.status == 0).all()
    ref = O.run_slots(sc, hidden, seeds, epochs=epochs, threads=16)
    scale = np.maximum(1.0, np.max(np.abs(ref.soft), axis=-1, keepdims=True))
    soft_dev = float(np.max(np.abs(out.soft - ref.soft) / scale))
    wfro, welem = _weight_dev(dims, out.plans, ref.plans)
    trace_dev = float(np.max(np.abs(out.trace - ref.trace) / np.abs(ref.trace)))
    rcodes = A.codes_of(ref.soft)
    flips_net = np.count_nonzero(out.codes != rcodes, axis=-1)
    flips = int(flips_net.sum())
    dber = np.abs(out.bit_errors.astype(np.int64) - ref.bit_errors)
    record("full_training_fp64", config=tag, slots=S, soft_dev=soft_dev, weight_dev=float(np.max(wfro)),
           weight_elem_max=float(np.max(welem)), trace_dev=trace_dev, flips=flips,
           symbols=int(out.codes.size), dev_bit_errors=int(out.bit_errors.sum()),
           ref_bit_errors=int(ref.bit_errors.sum()), train_mode=A.context().train_mode)
    assert flips <= 1e-4 * out.codes.size, flips  # north star: >= 99.99 % identical
    assert np.all(dber <= 2 * flips_net)
    # FP64 trajectory; the plans hold it rounded to FP32, data samples are FP32
    assert trace_dev < 1e-9, trace_dev
    assert float(np.max(wfro)) < 1e-6
    assert soft_dev < 1e-5, soft_dev
