"""Pins the oracle's LLS solver: ports proj/tests/test_lls.cpp and acceptance
criterion 2 (acceptance.cpp:73-86) against the independent pseudo-inverse
restated in tests/refimpl.py (oracles.hpp:19-72)."""
import numpy as np
import pytest

from tests import refimpl as R
from tests.helpers import random_mat


def test_identity_design(O):  # test_lls.cpp:23-30
    w = O.lls_fit(np.eye(2), np.array([0.3, 0.7]))
    assert abs(w.w[0] - 0.3) < 1e-14 and abs(w.w[1] - 0.7) < 1e-14


def test_matches_pinv_oracle_1370x8(O):  # :32-42
    for seed in range(20):
        x = random_mat(1370, 8, 1000 + seed)
        r = O.Rng(2000 + seed)
        y = np.array([r.gaussian() for _ in range(1370)])
        w = O.lls_fit(x, y).w
        wr = R.pinv_solve(x, y)
        assert np.linalg.norm(w - wr) / np.linalg.norm(wr) < 1e-10


def test_noiseless_k2_m4_solved_exactly(O):  # :44-56 (rank-deficient, min-norm path)
    rec = O.synthesize(O.Scenario(num_users=2, num_antennas=4, train_symbols=64,
                                  data_symbols=32, seed=5))
    x = O.widen_design(rec.train_rx)
    y = O.widen_targets(rec.train_symbols[:, 0])
    w = O.lls_fit(x, y, 1)
    assert np.max(np.abs(x @ w.w - y)) < 1e-10
    sv = O.singular_values(x)
    assert sv[3] > 1e-3 * sv[0] and sv[4] < 1e-12 * sv[0]  # rank 4 of 8


def test_predict_selector_and_zero(O):  # :58-73
    x = np.array([[1 + 2j, 3 + 4j], [-1 + 0.5j, 0 + 1j], [2 - 2j, 1 + 1j]])
    wid = O.widen_design(x)
    sel = np.zeros(4)
    sel[0] = 1.0
    pred = O.narrow_predictions(wid @ sel)
    assert np.array_equal(pred, x[:, 0])
    assert np.array_equal(O.narrow_predictions(wid @ np.zeros(4)), np.zeros(3, complex))


def test_single_user_recovery(O):  # :75-87
    rec = O.synthesize(O.Scenario(num_users=1, num_antennas=2, train_symbols=16,
                                  data_symbols=64, seed=12))
    w = O.lls_fit(O.widen_design(rec.train_rx), O.widen_targets(rec.train_symbols[:, 0]))
    pred = O.narrow_predictions(O.widen_design(rec.data_rx) @ w.w)
    assert np.max(np.abs(pred - rec.data_symbols[:, 0])) < 1e-10


def test_residual_orthogonality(O):  # :89-100
    for seed in range(5):
        x = random_mat(200, 8, 10 + seed)
        r = O.Rng(20 + seed)
        y = np.array([r.gaussian() for _ in range(200)])
        w = O.lls_fit(x, y).w
        lhs = np.max(np.abs(x.T @ (x @ w - y)))
        assert lhs <= 1e-8 * np.max(np.abs(x)) * np.max(np.abs(y))


def test_rotation_equivariance(O):  # :102-118
    rec = O.synthesize(O.Scenario(train_symbols=64, data_symbols=16, snr_db=20.0, seed=31))
    w = O.lls_fit(O.widen_design(rec.train_rx), O.widen_targets(rec.train_symbols[:, 3]), 4)
    r = O.Rng(77)
    s = 1 / np.sqrt(2)
    rows = np.empty((1000, 4), complex)  # gen_channel(1000, 4)^T, g++ draw order
    for k in range(1000):
        for m in range(4):
            im = r.gaussian() * s
            re = r.gaussian() * s
            rows[k, m] = complex(re, im)
    g = O.narrow_predictions(O.widen_design(rows) @ w.w)
    gi = O.narrow_predictions(O.widen_design(1j * rows) @ w.w)
    assert np.max(np.abs(gi - 1j * g)) / np.max(np.abs(g)) < 1e-10


def test_batched_equals_independent(O):  # :120-134
    rec = O.synthesize(O.Scenario(train_symbols=64, data_symbols=8, snr_db=15.0, seed=9))
    design = O.widen_design(rec.train_rx)
    for k in range(6):
        wa = O.lls_fit(design, O.widen_targets(rec.train_symbols[:, k]), k + 1).w
        wb = O.lls_fit(O.widen_design(rec.train_rx), O.widen_targets(rec.train_symbols[:, k])).w
        assert np.array_equal(wa, wb)


def _dup_design():
    x = np.zeros((6, 4))
    x[:, 0] = 1
    x[:, 1] = 1
    x[:, 2] = np.linspace(0, 5, 6)
    x[:, 3] = 2 * x[:, 2]
    return x


def test_min_norm_rank_deficient(O):  # :136-149
    x = _dup_design()
    y = np.ones(6) + 3 * x[:, 2]
    w = O.lls_fit(x, y).w
    assert np.linalg.norm(x @ w - y) < 1e-10
    assert abs(w[0] - w[1]) < 1e-12 * max(1, abs(w[0]))
    assert abs(w[3] - 2 * w[2]) < 1e-12 * max(1, abs(w[3]))
    assert np.allclose(w, np.linalg.pinv(x) @ y, rtol=1e-10, atol=1e-12)


def test_inconsistent_rank_deficient_raises(O):  # :151-166
    x = _dup_design()
    y = np.zeros(6)
    y[0] = 1.0
    with pytest.raises(O.IllConditionedError) as e:
        O.lls_fit(x, y)
    assert e.value.gram_condition > 1e12


def test_dimension_errors(O):  # :168-176
    with pytest.raises(O.DimensionError):
        O.lls_fit(np.ones((4, 8)), np.ones(4))
    with pytest.raises(O.DimensionError):
        O.lls_fit(np.ones((8, 4)), np.ones(7))


def test_gram_condition_is_singular_value_ratio(O):
    x = random_mat(300, 6, 3)
    y = random_mat(300, 1, 4)[:, 0]
    sv = np.linalg.svd(x, compute_uv=False)
    w = O.lls_fit(x, y)
    assert abs(w.gram_condition - (sv[0] / sv[-1]) ** 2) < 1e-10 * w.gram_condition
    assert np.allclose(w.w, np.linalg.lstsq(x, y, rcond=None)[0], rtol=1e-11, atol=1e-13)
