"""NOMA1 dataset and noma-net params formats (formats.py; io.cpp:80-211),
ported from test_io.cpp:37-97: bit-exact round trips, the byte layout
restated independently with struct, and the fault cases (corrupted magic,
truncation, missing file, bad version, zero dimension, malformed params)."""
import json
import os
import struct

import numpy as np
import pytest

from paper_2206_05998_b200 import formats as F


def _record(O):
    sc = O.Scenario(num_users=3, num_antennas=4, train_symbols=16, data_symbols=24,
                    power_step_db=3.0, snr_db=12.0, rx_nonlinearity_gain=0.05)
    r = O.synthesize(sc, O.seed_bundle(4242))
    return F.TransmissionRecord(r.channel, r.powers, r.train_rx, r.train_symbols, r.data_rx,
                                r.data_symbols, r.noise_power)


def test_dataset_round_trip_bit_exact(O, tmp_path):
    rec = _record(O)
    p = str(tmp_path / "d.noma")
    F.write_dataset(rec, p)
    back = F.read_dataset(p)
    for f in ("channel", "powers", "train_rx", "train_symbols", "data_rx", "data_symbols"):
        assert np.array_equal(getattr(back, f), getattr(rec, f)), f
    assert back.noise_power == rec.noise_power


def test_dataset_byte_layout(O, tmp_path):
    """io.hpp:10-15 restated with struct: packed little-endian, 23-byte header."""
    rec = _record(O)
    p = str(tmp_path / "d.noma")
    F.write_dataset(rec, p)
    raw = open(p, "rb").read()
    K, M, NT, ND = 3, 4, 16, 24
    exp = b"NOMA1" + struct.pack("<HIIII", 1, K, M, NT, ND)
    exp += struct.pack(f"<{K}d", *rec.powers)
    for a in (rec.channel, rec.train_rx, rec.train_symbols, rec.data_rx, rec.data_symbols):
        for z in a.reshape(-1):
            exp += struct.pack("<dd", z.real, z.imag)
    exp += struct.pack("<d", rec.noise_power)
    assert raw == exp


def test_dataset_faults(O, tmp_path):
    rec = _record(O)
    p = str(tmp_path / "d.noma")
    F.write_dataset(rec, p)
    raw = open(p, "rb").read()
    bad = tmp_path / "bad"
    bad.write_bytes(b"NOMA2" + raw[5:])
    with pytest.raises(F.FormatError):
        F.read_dataset(str(bad))
    bad.write_bytes(raw[:-1])
    with pytest.raises(F.TruncationError):
        F.read_dataset(str(bad))
    bad.write_bytes(raw[:3])
    with pytest.raises(F.TruncationError):
        F.read_dataset(str(bad))
    bad.write_bytes(raw[:5] + struct.pack("<H", 2) + raw[7:])
    with pytest.raises(F.FormatError):
        F.read_dataset(str(bad))
    bad.write_bytes(raw[:7] + struct.pack("<I", 0) + raw[11:])
    with pytest.raises(F.FormatError):
        F.read_dataset(str(bad))
    with pytest.raises(F.IoError):
        F.read_dataset(str(tmp_path / "missing.noma"))
    assert issubclass(F.TruncationError, F.IoError) and issubclass(F.FormatError, F.IoError)


def _net(O):
    from tests.helpers import random_net_hybrid

    net = random_net_hybrid([8, 6, 5], 11)
    return net, net.layers()


def test_params_round_trip(O, tmp_path):
    net, (layers, final) = _net(O)
    p = str(tmp_path / "n.json")
    F.write_params(net.dims, net.w0, layers, final, 2, "abc123", p)
    lp = F.read_params(p)
    assert lp.dims == list(net.dims) and lp.user_index == 2 and lp.config_digest == "abc123"
    assert np.array_equal(lp.w0, net.w0) and np.array_equal(lp.final_weights, final)
    for (W, b), (W2, b2) in zip(layers, lp.layers):
        assert np.array_equal(W, W2) and np.array_equal(b, b2)
    text = open(p).read()
    doc = json.loads(text)
    assert doc["format"] == "noma-net" and doc["version"] == 1
    # nlohmann dump(): sorted keys, compact separators
    assert text == json.dumps(doc, sort_keys=True, separators=(",", ":"))
    assert list(doc) == sorted(doc)


def test_params_faults(tmp_path):
    p = tmp_path / "p.json"
    p.write_text("{not json")
    with pytest.raises(F.FormatError):
        F.read_params(str(p))
    p.write_text(json.dumps({"format": "other"}))
    with pytest.raises(F.FormatError):
        F.read_params(str(p))
    p.write_text(json.dumps({"format": "noma-net", "user_index": 1, "dims": [2, 2], "w0": [0, 0],
                             "layers": [{"weights": [[1, 2], [3]], "bias": [0, 0]}],
                             "final_weights": [0, 0]}))
    with pytest.raises(F.FormatError):
        F.read_params(str(p))
    with pytest.raises(F.IoError):
        F.read_params(str(tmp_path / "none.json"))
