"""GPU parity of the tcgen05 (3xTF32) detection kernel, k_detect_tc.cu, for
every shape it covers: soft outputs against the FP64 reference forward at the
reference's FP32 inference tolerance (test_fused.cpp:128-130), hard decisions
against the reference's sign pattern, and bit-for-bit agreement of decisions
and error counters with the FFMA kernel (the north star's gate for putting
the data phase on tensor cores)."""
import numpy as np
import pytest

from tests.helpers import random_net_fused, record

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def A():
    from paper_2206_05998_b200 import api

    api.context()
    return api


@pytest.mark.parametrize("dims", [[32, 64], [32, 64, 64], [64, 64], [64, 64, 64]])
@pytest.mark.parametrize("nsym", [4096, 1000])  # 1000: ragged last tile
def test_detect_tc_matches_reference(A, O, dims, nsym, monkeypatch):
    from tests import refimpl as R

    M = dims[0] // 2
    onet = random_net_fused(dims, 7 + len(dims))
    layers, final = onet.layers()
    net = A.net_from_params(onet.dims, onet.w0, layers, final)
    sy = A.synthesize(6, M, 2 * M, nsym, [23], snr_db=8.0, rx_nonlinearity_gain=0.05)
    x = sy.data_rx[0]
    truth = sy.data_rx[0][:, 0].astype(np.complex128)  # any symbols: only the count is compared
    soft, bits, errs = A.detect(net, x, truth_symbols=truth)
    assert A.context().detect_mode == 2
    ref = O.narrow_predictions(R.reference_forward(onet.dims, onet.w0, layers, final,
                                                   O.widen_design(x.astype(np.complex128))))
    scale = max(1.0, float(np.max(np.abs(ref))))
    dev = float(np.max(np.abs(soft - ref))) / scale
    ref_bits = O.hard_decision_qpsk(ref)
    margin = np.minimum(np.abs(ref.real), np.abs(ref.imag)) > 1e-5 * scale
    flips = int(np.count_nonzero((bits != ref_bits).any(axis=-1) & margin))
    record("detect_tc", config=str(dims), symbols=nsym, soft_dev=dev, flips=flips)
    assert dev < 1e-5, dev
    assert flips == 0
    # identical decisions and counters to the FFMA kernel
    monkeypatch.setenv("NOMA_DETECT_TC", "0")
    soft_f, bits_f, errs_f = A.detect(net, x, truth_symbols=truth)
    assert A.context().detect_mode == 1
    assert np.max(np.abs(soft_f - soft)) / scale < 2e-6
    assert np.array_equal(bits, bits_f)
    assert errs == errs_f


def test_bench_rows(A, O):
    """`noma bench` GPU rows (fused_inference.cpp:325-338 schema), gated
    against the FP64 forward; the CPU naive row comes from the oracle here."""
    import time

    onet = random_net_fused([32, 64, 64], 5)
    layers, final = onet.layers()
    net = A.net_from_params(onet.dims, onet.w0, layers, final)
    x = np.random.default_rng(1).normal(size=(4096, 32))
    t0 = time.perf_counter()
    O.fused_forward(onet.dims, O.build_plan(onet), x)
    naive = (time.perf_counter() - t0) * 1e9 / 4096
    rows = A.bench_rows(net, 1 << 16, repeats=5, naive_ns_per_sample=naive).splitlines()
    assert [r.split(",")[0] for r in rows] == ["gpu_tcgen05", "gpu_ffma"]
    for r in rows:
        path, dims, batch, ns, sp = r.split(",")
        assert dims == "32x64x64" and batch == str(1 << 16)
        assert float(ns) > 0 and float(sp) > 1


@pytest.mark.parametrize("dims", [[32, 64, 64], [64, 64]])
@pytest.mark.parametrize("rows", [1000, 9000])  # ragged tiles; CTAs whose share spans several nets
def test_detect_tc_many_nets(A, dims, rows, monkeypatch):
    """A batch of designs x users through noma_detect: the persistent
    detection grid splits all nets' tiles evenly over the SMs, so a CTA runs
    several nets back to back (weights reloaded, barrier phases carried on).
    Every net must give what it gives alone, and the same decisions, soft
    outputs and bit-error counters as the FFMA kernel."""
    from paper_2206_05998_b200 import native as N

    M, n_designs, K = dims[0] // 2, 5, 6
    nets = [A.net_from_params(o.dims, o.w0, *o.layers())
            for o in (random_net_fused(dims, 100 + i) for i in range(n_designs * K))]
    plans = np.ascontiguousarray(np.stack([n.plan.reshape(-1) for n in nets]))
    rng = np.random.default_rng(5)
    x = (rng.normal(size=(n_designs, rows, M)) + 1j * rng.normal(size=(n_designs, rows, M))).astype(np.complex64)
    truth = rng.integers(0, 4, size=(n_designs, rows, K), dtype=np.uint8)

    def run():
        soft = np.zeros((n_designs * K, rows), np.complex64)
        codes = np.zeros((n_designs * K, rows), np.uint8)
        errs = np.zeros(n_designs * K, np.uint32)
        A.context().detect(nets[0].dims, N.LAYOUT_WIDEN, n_designs, K, rows, x.view(np.float32), plans,
                           truth=truth, soft=soft.view(np.float32), codes=codes, bit_errors=errs)
        return soft, codes, errs, A.context().detect_mode

    soft, codes, errs, mode = run()
    assert mode == 2
    for net in (0, K + 1, n_designs * K - 1):  # alone: the same kernel on one net
        d, k = divmod(net, K)
        s1, b1, e1 = A.detect(nets[net], x[d])
        assert np.array_equal(s1, soft[net])
        assert np.array_equal(b1[:, 0] | (b1[:, 1] << 1), codes[net])
    want = np.array([np.count_nonzero((codes[n] ^ truth[n // K, :, n % K]) & 1)
                     + np.count_nonzero((codes[n] ^ truth[n // K, :, n % K]) & 2) for n in range(n_designs * K)])
    assert np.array_equal(errs, want)
    monkeypatch.setenv("NOMA_DETECT_TC", "0")
    soft_f, codes_f, errs_f, mode_f = run()
    assert mode_f == 1
    scale = max(1.0, float(np.max(np.abs(soft_f))))
    assert np.max(np.abs(soft_f - soft)) / scale < 2e-6
    # random data puts a few of the 2 x nets x rows soft values within
    # rounding of zero, where the two kernels' FP32 sums may take either sign
    # (the synthetic channels of the shape tests above have none)
    near = (np.abs(soft.real) < 1e-5 * scale) | (np.abs(soft.imag) < 1e-5 * scale)
    assert np.array_equal(codes[~near], codes_f[~near])
    assert np.all(np.abs(errs.astype(np.int64) - errs_f.astype(np.int64)) <= 2 * near.sum(axis=1))


@pytest.mark.parametrize("n_designs", [2, 1])  # 1: a plain copy per design
@pytest.mark.parametrize("tc", ["1", "0"])
def test_detect_host_chunked_upload(A, tc, n_designs, monkeypatch):
    """Host buffers of >= 32 MB are uploaded in row chunks on the copy stream,
    each chunk detected as it lands (strided 2-D copies across designs, ragged
    last chunk).  Outputs must be bit-identical to the same call on device
    buffers, which runs one launch."""
    import torch

    from paper_2206_05998_b200 import native as N

    monkeypatch.setenv("NOMA_DETECT_TC", tc)
    dims, K = [32, 64, 64], 3
    rows = 300001 // n_designs
    M = dims[0] // 2
    nets = [A.net_from_params(o.dims, o.w0, *o.layers())
            for o in (random_net_fused(dims, 200 + i) for i in range(n_designs * K))]
    plans = np.ascontiguousarray(np.stack([n.plan.reshape(-1) for n in nets]))
    rng = np.random.default_rng(9)
    x = (rng.normal(size=(n_designs, rows, M)) + 1j * rng.normal(size=(n_designs, rows, M))).astype(np.complex64)
    assert x.nbytes >= 32 << 20
    truth = rng.integers(0, 4, size=(n_designs, rows, K), dtype=np.uint8)
    ctx = A.context()
    soft = np.zeros((n_designs * K, rows), np.complex64)
    codes = np.zeros((n_designs * K, rows), np.uint8)
    errs = np.zeros(n_designs * K, np.uint32)
    sers = np.zeros(n_designs * K, np.uint32)
    ctx.detect(dims, N.LAYOUT_WIDEN, n_designs, K, rows, x.view(np.float32), plans, truth=truth,
               soft=soft.view(np.float32), codes=codes, bit_errors=errs, symbol_errors=sers)
    # fused counters = the decisions' mismatches (eval.cpp:56-65; SER: either bit)
    tr = np.transpose(truth, (0, 2, 1)).reshape(n_designs * K, rows)
    assert np.array_equal(sers.astype(np.int64), np.count_nonzero(codes != tr, axis=-1))
    xor = codes ^ tr
    assert np.array_equal(errs.astype(np.int64),
                          np.count_nonzero(xor & 1, axis=-1) + np.count_nonzero(xor & 2, axis=-1))
    dev = torch.device("cuda", 0)
    xd = torch.from_numpy(x.view(np.float32)).to(dev)
    pd = torch.from_numpy(plans).to(dev)
    td = torch.from_numpy(truth).to(dev)
    sd = torch.zeros((n_designs * K, rows, 2), dtype=torch.float32, device=dev)
    cd = torch.zeros((n_designs * K, rows), dtype=torch.uint8, device=dev)
    ed = torch.zeros(n_designs * K, dtype=torch.int32, device=dev)
    ctx.detect(dims, N.LAYOUT_WIDEN, n_designs, K, rows, xd, pd, truth=td, soft=sd, codes=cd, bit_errors=ed)
    torch.cuda.synchronize()
    assert ctx.detect_mode == (2 if tc == "1" else 1)
    assert np.array_equal(soft.view(np.float32).reshape(n_designs * K, rows, 2), sd.cpu().numpy())
    assert np.array_equal(codes, cd.cpu().numpy())
    assert np.array_equal(errs.astype(np.int64), ed.cpu().numpy().astype(np.int64))
