"""Pins the oracle's channel synthesiser: ports proj/tests/test_channel_sim.cpp."""
import math

import numpy as np
import pytest

from tests import refimpl as R


def test_symbols_unit_energy_qpsk(O):  # test_channel_sim.cpp:11-20
    rec = O.synthesize(O.Scenario(num_users=1, num_antennas=1, train_symbols=4,
                                  data_symbols=4, seed=7))
    a = 1 / math.sqrt(2)
    assert np.all(np.abs(np.abs(rec.train_symbols.real) - a) < 1e-15)
    assert np.all(np.abs(np.abs(rec.train_symbols.imag) - a) < 1e-15)


def test_symbol_stream_matches_independent_restatement(O):
    sc = O.Scenario(num_users=3, num_antennas=2, train_symbols=20, data_symbols=7, seed=11)
    rec = O.synthesize(sc)
    seeds = O.seed_bundle(11)
    p = R.PyRng(seeds[0])
    a = 1 / math.sqrt(2)
    want = []
    for _ in range(20 + 7):
        row = []
        for _ in range(3):  # row-major t then k (channel_sim.cpp:36-45)
            bits = p.below(4)
            row.append(complex(-a if bits & 1 else a, -a if bits & 2 else a))
        want.append(row)
    want = np.array(want)
    assert np.array_equal(rec.train_symbols, want[:20])
    assert np.array_equal(rec.data_symbols, want[20:])


def test_channel_draw_order_matches_gxx(O):
    """channel k then m; imaginary drawn first (g++ argument order)."""
    sc = O.Scenario(num_users=2, num_antennas=3, train_symbols=6, data_symbols=2, seed=3)
    rec = O.synthesize(sc)
    p = R.PyRng(O.seed_bundle(3)[1])
    s = 1 / math.sqrt(2)
    for k in range(2):
        for m in range(3):
            im = p.gaussian() * s
            re = p.gaussian() * s
            assert rec.channel[m, k] == complex(re, im)


def test_record_determinism(O):  # :94-106
    sc = O.Scenario(train_symbols=32, data_symbols=16, snr_db=20.0, seed=77)
    a, b = O.synthesize(sc), O.synthesize(sc)
    for f in ("train_rx", "data_rx", "channel", "train_symbols"):
        assert np.array_equal(getattr(a, f), getattr(b, f))


def test_symbol_counts_within_4sd(O):  # :29-44
    n = 100000
    rec = O.synthesize(O.Scenario(num_users=1, num_antennas=1, train_symbols=n,
                                  data_symbols=1, seed=123))
    s = rec.train_symbols[:, 0]
    idx = (s.real < 0).astype(int) + 2 * (s.imag < 0).astype(int)
    counts = np.bincount(idx, minlength=4)
    sd = math.sqrt(n * 0.25 * 0.75)
    assert np.all(np.abs(counts - n / 4) < 4 * sd)


def test_channel_cn01_statistics(O):  # :52-69
    acc = []
    for seed in range(400):
        rec = O.synthesize(O.Scenario(num_users=5, num_antennas=5, train_symbols=10,
                                      data_symbols=1, seed=seed))
        acc.append(np.mean(np.abs(rec.channel) ** 2))
    assert abs(np.mean(acc) - 1.0) < 0.05


def test_linearity_noiseless(O):  # :71-85
    sc = O.Scenario(num_users=3, num_antennas=4, train_symbols=16, data_symbols=8, seed=11)
    rec = O.synthesize(sc)
    expect = rec.train_symbols @ (rec.channel * np.sqrt(rec.powers)[None, :]).T
    assert np.max(np.abs(rec.train_rx - expect)) < 1e-15
    assert rec.noise_power == 0.0


def test_power_profile(O):  # :87-92
    p = O.power_profile(6, 3.0)
    assert p[0] == 1.0
    assert abs(p[3] - 10 ** -0.9) < 1e-12 * 10 ** -0.9
    assert np.all(np.diff(p) < 0)


def test_measured_snr(O):  # :108-125
    sc = O.Scenario(num_users=6, num_antennas=4, train_symbols=8, data_symbols=100000,
                    snr_db=10.0, seed=3)
    noisy = O.synthesize(sc)
    clean = O.synthesize(O.Scenario(num_users=6, num_antennas=4, train_symbols=8,
                                    data_symbols=100000, seed=3))
    sig = np.sum(np.abs(clean.data_rx) ** 2) / clean.data_rx.shape[0]
    noise = np.sum(np.abs(noisy.data_rx - clean.data_rx) ** 2) / noisy.data_rx.shape[0]
    assert abs(10 * math.log10(sig / noise) - 10.0) < 0.1


def test_soi_power_share(O):  # :127-142
    p = O.power_profile(6, 3.0)
    soi = tot = 0.0
    for seed in range(2000):
        rec = O.synthesize(O.Scenario(num_users=6, num_antennas=4, train_symbols=8,
                                      data_symbols=1, seed=seed))
        pk = p * np.sum(np.abs(rec.channel) ** 2, axis=0)
        soi += pk[3]
        tot += pk.sum()
    assert abs(10 * math.log10(soi / tot) + 12.0) < 1.0


def test_validation(O):  # :144-154
    with pytest.raises(O.ConfigError):
        O.synthesize(O.Scenario(num_users=0))
    with pytest.raises(O.ConfigError):
        O.synthesize(O.Scenario(train_symbols=5))
    with pytest.raises(O.ConfigError):
        O.synthesize(O.Scenario(power_step_db=-1.0))


def test_cubic_distortion_before_noise(O):  # :156-171
    base = dict(num_users=1, num_antennas=2, train_symbols=8, data_symbols=4, seed=9)
    lin = O.synthesize(O.Scenario(**base))
    nl = O.synthesize(O.Scenario(rx_nonlinearity_gain=0.05, **base))
    u = lin.data_rx
    assert np.max(np.abs(nl.data_rx - (u + 0.05 * u * np.abs(u) ** 2))) < 1e-15
