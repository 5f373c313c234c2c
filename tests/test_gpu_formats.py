"""Device ingest of the reference's on-disk formats: a NOMA1 dataset read
back from disk drives noma_pipeline to bit-identical results, and trained
parameters written as noma-net JSON and read back detect identically."""
import numpy as np
import pytest

from paper_2206_05998_b200 import formats as F

pytestmark = pytest.mark.gpu


def test_noma1_ingest_and_params_round_trip(O, tmp_path):
    from paper_2206_05998_b200 import api

    sc = O.Scenario(num_users=3, num_antennas=4, train_symbols=64, data_symbols=300,
                    power_step_db=3.0, snr_db=15.0, rx_nonlinearity_gain=0.05)
    r = O.synthesize(sc, O.seed_bundle(77))
    rec = F.TransmissionRecord(r.channel, r.powers, r.train_rx, r.train_symbols, r.data_rx,
                               r.data_symbols, r.noise_power)
    path = str(tmp_path / "slot.noma")
    F.write_dataset(rec, path)
    px, py, dx, tr = F.to_device_slot(F.read_dataset(path))
    init = np.array([[O.substream_seed(77, 0x1000 + k) for k in range(1, 4)]], np.uint64)
    shuf = np.array([[O.substream_seed(77, k) for k in range(1, 4)]], np.uint64)
    a = api.pipeline([8, 16], px, py, dx, tr, init, shuf, epochs=4)
    b = api.pipeline([8, 16], r.train_rx[None], r.train_symbols[None],
                     r.data_rx.astype(np.complex64)[None], api.codes_of(r.data_symbols)[None],
                     init, shuf, epochs=4)
    for f in ("w0", "plans", "codes", "bit_errors", "trace"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    # noma-net round trip of user 2's trained detector
    dims = [8, 16]
    net = O.unpack_plan(dims, a.plans[0, 1].astype(np.float64))
    layers, final = net.layers()
    p = str(tmp_path / "u2.json")
    F.write_params(dims, net.w0, layers, final, 2, "", p)
    lp = F.read_params(p)
    n2 = api.net_from_params(lp.dims, lp.w0, lp.layers, lp.final_weights)
    assert np.array_equal(n2.plan.astype(np.float32), a.plans[0, 1])
    s1, bits1, _ = api.detect(n2, dx[0])
    assert np.array_equal(api.codes_of(s1), a.codes[0, 1])
