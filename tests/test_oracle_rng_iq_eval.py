"""Pins the oracle's RNG, IQ transform and evaluation helpers.

Ports the known-answer tests of proj/tests/test_iq_transform.cpp and
proj/tests/test_eval.cpp:10-37, and cross-checks the C RNG against the
independent pure-Python restatement in tests/refimpl.py.
"""
import os
import shutil
import subprocess

import numpy as np
import pytest

from tests import refimpl as R
from tests.helpers import random_mat

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ----------------------------------------------------------------- rng.hpp
def test_splitmix64_published_vector(O):
    # splitmix64 reference stream for seed 1234567 (Vigna's splitmix64.c).
    want = [6457827717110365317, 3203168211198807973, 9817491932198370423,
            4593380528125082431, 16408922859458223821]
    s = 1234567
    got = []
    for _ in range(5):
        out, s = O.splitmix64(s)
        got.append(out)
    assert got == want
    ps = 1234567
    pgot = []
    for _ in range(5):
        out, ps = R.splitmix64(ps)
        pgot.append(out)
    assert pgot == want


def test_xoshiro_stream_matches_independent_restatement(O):
    for seed in (0, 1, 42, 0xDEADBEEF, 2**64 - 1):
        c = O.rng_u64(seed, 64)
        p = R.PyRng(seed)
        assert [int(v) for v in c] == [p.next_u64() for _ in range(64)]


def test_uniform_below_gaussian_match_independent_restatement(O):
    r, p = O.Rng(77), R.PyRng(77)
    for _ in range(200):
        assert r.uniform() == p.uniform()
        assert r.below(1370) == p.below(1370)
        assert r.below(4) == p.below(4)
    g = O.rng_gaussian(5, 500)
    p = R.PyRng(5)
    pg = np.array([p.gaussian() for _ in range(500)])
    assert np.array_equal(g, pg)  # same libm on one host


def test_substream_and_mix_tag(O):
    for m in (0, 1, 1000, 2**63 + 5):
        for t in (0, 1, 2, 3, 0x1001, 2**40):
            assert O.substream_seed(m, t) == R.substream_seed(m, t)
    # golden values from the reference's mix_tag (eval.cpp:77-84) compiled with
    # g++ 13 -std=c++20 at -O0 and -O3 (sequencing of `s ^= splitmix64(s) + b`).
    assert O.mix_tag(1, 2, 3, 4) == 12041511949808429858
    assert O.mix_tag(0, 11) == 1028850491766231610
    assert O.mix_tag(7, 12, 1) == 5950532866604775551
    for args in ((1, 2, 3, 4), (0, 11), (7, 12, 1), (5, 9, 2, 3)):
        assert O.mix_tag(*args) == R.mix_tag(*args)


def test_seed_bundle(O):
    assert O.seed_bundle(9) == tuple(R.substream_seed(9, t) for t in (1, 2, 3))


@pytest.mark.skipif(shutil.which("g++") is None, reason="g++ absent")
def test_gxx_evaluates_constructor_arguments_right_to_left(tmp_path):
    """The reference draws complex noise as cplx(g()*s, g()*s)
    (channel_sim.cpp:56, :71); g++ evaluates the arguments right to left, so the
    first draw is the imaginary part.  The oracle (and the device synthesiser)
    follow the g++ order; this probe pins it."""
    exe = tmp_path / "probe"
    subprocess.run(["g++", "-std=c++20", "-O3", os.path.join(GOLDEN, "probe_eval_order.cpp"),
                    "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split()
    assert out == ["second_draw_is_real"]


# ---------------------------------------------------------- iq_transform
def test_widen_design_hand_rows(O):  # test_iq_transform.cpp:10-20
    x = np.array([[1 + 2j, 3 - 1j]])
    w = O.widen_design(x)
    assert w.shape == (2, 4)
    assert np.array_equal(w, np.array([[1, 3, 2, -1], [2, -1, -1, -3]], dtype=float))


def test_widen_with_targets_1x1(O):  # :22-35
    w = O.widen_design(np.array([[1 + 1j]]))
    assert np.array_equal(w, np.array([[1, 1], [1, -1]], dtype=float))
    t = O.widen_targets(np.array([0.5 - 0.5j]))
    assert t[0] == 0.5 and t[1] == -0.5


def test_widened_shape(O):  # :37-43
    r = O.Rng(1)
    x = np.array([[complex(0, 0)] * 4] * 685)
    assert O.widen_design(x + 1).shape == (1370, 8)


def test_narrow_and_round_trip(O):  # :45-72
    z = O.narrow_predictions(np.array([0.5, -0.5]))
    assert z[0] == 0.5 - 0.5j
    z2 = O.narrow_predictions(np.array([1.0, 0, 0, 1]))
    assert z2[0] == 1 and z2[1] == 1j
    with pytest.raises(O.DimensionError):
        O.narrow_predictions(np.zeros(3))
    rec = O.synthesize(O.Scenario(train_symbols=33, data_symbols=8, seed=4))
    for k in range(6):
        y = rec.train_symbols[:, k]
        assert np.array_equal(O.narrow_predictions(O.widen_targets(y)), y)


def test_norm_preservation(O):  # :74-83
    x = random_mat(50, 6, 8)
    xc = x[:, :3] + 1j * x[:, 3:]
    w = O.widen_design(xc)
    rn = np.linalg.norm(xc, axis=1)
    assert np.allclose(np.linalg.norm(w[0::2], axis=1), rn, rtol=1e-14)
    assert np.allclose(np.linalg.norm(w[1::2], axis=1), rn, rtol=1e-14)


def test_widen_errors(O):  # :85-92
    with pytest.raises(O.DimensionError):
        O.widen_design(np.zeros((0, 0), dtype=complex))


# ------------------------------------------------------------------- eval
def test_hard_decision_quadrants_ties_round_trip(O):  # test_eval.cpp:10-25
    s = np.array([0.9 + 0.8j, -0.1 - 2.0j, 0.0 + 0.0j, complex(-0.0, -0.0)])
    bits = O.hard_decision_qpsk(s)
    assert bits.tolist() == [[0, 0], [1, 1], [0, 0], [0, 0]]
    allb = np.array([[0, 0], [0, 1], [1, 0], [1, 1]], dtype=np.uint8)
    assert np.array_equal(O.hard_decision_qpsk(O.map_qpsk_bits(allb)), allb)


def test_bit_error_rate_basics(O):  # :27-37
    a = np.zeros((50, 2), np.uint8)
    b = np.ones((50, 2), np.uint8)
    assert O.bit_error_rate(a, a) == 0.0
    assert O.bit_error_rate(a, b) == 1.0
    c = a.copy()
    c[7, 1] = 1
    assert abs(O.bit_error_rate(c, a) - 0.01) < 1e-15
    with pytest.raises(O.DimensionError):
        O.bit_error_rate(a, np.zeros((10, 2), np.uint8))
