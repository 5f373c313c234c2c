"""GPU parity of the latency-mode training kernel (k_train_lat.cu: one
neuron-split thread-block cluster per user network, partial outputs and
activations exchanged through st.async + mbarrier) against the FP64 oracle,
for every cluster size and hidden-layer count it supports, plus the ragged
minibatch edge cases of hybrid_nn.cpp:180-181 and bitwise determinism
(test_hybrid_nn.cpp:290-311)."""
import numpy as np
import pytest

from tests.helpers import record

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def A():
    from paper_2206_05998_b200 import api

    api.context()
    return api


def _run(A, O, *, M, K, hidden, NT, ND, epochs, S=1, snr=20.0, seed0=3000):
    sc = O.Scenario(num_users=K, num_antennas=M, train_symbols=NT, data_symbols=ND,
                    power_step_db=3.0, snr_db=snr, rx_nonlinearity_gain=0.05)
    seeds = [seed0 + s for s in range(S)]
    recs = [O.synthesize(sc, O.seed_bundle(s)) for s in seeds]
    ref = O.run_slots(sc, hidden, seeds, epochs=epochs, threads=8)
    init = np.array([[O.substream_seed(s, 0x1000 + k + 1) for k in range(K)] for s in seeds],
                    np.uint64)
    shuf = np.array([[O.substream_seed(s, k + 1) for k in range(K)] for s in seeds], np.uint64)
    out = A.pipeline([2 * M] + hidden, np.stack([r.train_rx for r in recs]),
                     np.stack([r.train_symbols for r in recs]), np.stack([r.data_rx for r in recs]),
                     np.stack([A.codes_of(r.data_symbols) for r in recs]), init, shuf,
                     epochs=epochs)
    return out, ref


def _devs(out, ref):
    soft = np.max(np.abs(out.soft - ref.soft)) / max(1.0, np.max(np.abs(ref.soft)))
    trace = float(np.max(np.abs(out.trace - ref.trace) / np.abs(ref.trace)))
    return soft, trace


@pytest.mark.parametrize("cs,M,hidden", [
    (16, 16, [32]), (16, 16, [64]), (16, 16, [128]), (8, 16, [32]), (8, 16, [64]), (4, 16, [32]),
    (16, 16, [64, 64]), (8, 16, [32, 32]), (8, 16, [64, 64]), (4, 16, [32, 32]),
    (16, 32, [64]), (16, 32, [64, 64]),
])
def test_latency_cluster_matches_oracle(A, O, cs, M, hidden, monkeypatch):
    """Every (cluster size, own neurons per CTA, layers, input width) instance
    of the latency kernel against the FP64 oracle (short training)."""
    monkeypatch.setenv("NOMA_LAT_CLUSTER", str(cs))
    out, ref = _run(A, O, M=M, K=3, hidden=hidden, NT=100, ND=256, epochs=3)
    assert A.context().train_mode == 100 + cs
    assert (out.status == 0).all()
    soft, trace = _devs(out, ref)
    record("latency_cluster", config=f"cs={cs} M={M} hidden={hidden}", soft_dev=soft, trace_dev=trace)
    assert soft < 1e-4 and trace < 1e-4, (soft, trace)


@pytest.mark.parametrize("NT", [64, 100, 129])
def test_latency_ragged_minibatches(A, O, NT, monkeypatch):
    """2 N_T = 128 (one full batch per epoch), 200 (128 + 72), 258 (128+128+2)."""
    monkeypatch.setenv("NOMA_LAT_CLUSTER", "16")
    out, ref = _run(A, O, M=16, K=2, hidden=[64], NT=NT, ND=64, epochs=4)
    assert A.context().train_mode == 116
    soft, trace = _devs(out, ref)
    assert soft < 1e-4 and trace < 1e-4, (NT, soft, trace)


def test_latency_unsupported_shape_falls_back(A, O, monkeypatch):
    """Unequal hidden widths are outside the latency kernel: the pipeline
    runs the one-CTA-per-net kernel instead, with the same results."""
    monkeypatch.setenv("NOMA_LAT_CLUSTER", "16")
    out, ref = _run(A, O, M=16, K=2, hidden=[64, 32], NT=100, ND=64, epochs=3)
    assert A.context().train_mode < 100
    soft, trace = _devs(out, ref)
    assert soft < 1e-4 and trace < 1e-4


def test_latency_c1_single_slot(A, O):
    """C1 (M=16, K=6, [32, 64], 50 epochs) as one slot: default cluster choice
    (16 CTAs per net), full training; decisions vs the FP64 oracle."""
    out, ref = _run(A, O, M=16, K=6, hidden=[64], NT=685, ND=3840, epochs=50, snr=25.0,
                    seed0=1000)
    assert A.context().train_mode == 116
    soft, trace = _devs(out, ref)
    flips = int(np.count_nonzero(out.codes != A.codes_of(ref.soft)))
    record("latency_c1", soft_dev=soft, trace_dev=trace, flips=flips, symbols=out.codes.size,
           dev_bit_errors=int(out.bit_errors.sum()), ref_bit_errors=int(ref.bit_errors.sum()))
    assert soft < 1e-1 and trace < 1e-1
    assert flips <= 1e-4 * out.codes.size + 0.5
    assert np.all(np.abs(out.bit_errors.astype(np.int64) - ref.bit_errors) <= 2 * flips)


def test_latency_deterministic(A, O, monkeypatch):
    monkeypatch.setenv("NOMA_LAT_CLUSTER", "16")
    a, _ = _run(A, O, M=16, K=3, hidden=[64, 64], NT=100, ND=64, epochs=5)
    b, _ = _run(A, O, M=16, K=3, hidden=[64, 64], NT=100, ND=64, epochs=5)
    assert np.array_equal(a.plans, b.plans)
    assert np.array_equal(a.trace, b.trace)
