"""GPU parity: the sm_100a LLS kernel (noma_lls_fit) against the FP64 oracle and
the reference's lls test suite (proj/tests/test_lls.cpp) -- through the C-ABI.

Tolerance: w0 <= 1e-10 relative (test_lls.cpp:40); the Gram
condition <= 1e-6 relative (a diagnostic, lls.hpp:12)."""
import numpy as np
import pytest

from tests import refimpl as R
from tests.helpers import random_mat

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def A():
    from paper_2206_05998_b200 import api

    api.context()
    return api


def test_identity_design(A):
    w = A.lls_fit(np.eye(2), np.array([0.3, 0.7]))
    assert abs(w.w[0] - 0.3) < 1e-14 and abs(w.w[1] - 0.7) < 1e-14


def test_matches_pinv_oracle_1370x8(A, O):
    for seed in range(20):
        x = random_mat(1370, 8, 1000 + seed)
        r = O.Rng(2000 + seed)
        y = np.array([r.gaussian() for _ in range(1370)])
        w = A.lls_fit(x, y).w
        wr = R.pinv_solve(x, y)
        assert np.linalg.norm(w - wr) / np.linalg.norm(wr) < 1e-10


def test_noiseless_k2_m4_min_norm(A, O):
    rec = O.synthesize(O.Scenario(num_users=2, num_antennas=4, train_symbols=64,
                                  data_symbols=32, seed=5))
    w = A.lls_fit_widened(rec.train_rx, rec.train_symbols[:, 0], 1)
    x = O.widen_design(rec.train_rx)
    y = O.widen_targets(rec.train_symbols[:, 0])
    assert np.max(np.abs(x @ w.w - y)) < 1e-10
    ref = O.lls_fit(x, y)
    assert np.linalg.norm(w.w - ref.w) / np.linalg.norm(ref.w) < 1e-9


def test_single_user_recovery(A, O):
    rec = O.synthesize(O.Scenario(num_users=1, num_antennas=2, train_symbols=16,
                                  data_symbols=64, seed=12))
    w = A.lls_fit_widened(rec.train_rx, rec.train_symbols[:, 0])
    pred = O.narrow_predictions(O.widen_design(rec.data_rx) @ w.w)
    assert np.max(np.abs(pred - rec.data_symbols[:, 0])) < 1e-10


def test_residual_orthogonality(A, O):
    for seed in range(5):
        x = random_mat(200, 8, 10 + seed)
        r = O.Rng(20 + seed)
        y = np.array([r.gaussian() for _ in range(200)])
        w = A.lls_fit(x, y).w
        assert np.max(np.abs(x.T @ (x @ w - y))) <= 1e-8 * np.max(np.abs(x)) * np.max(np.abs(y))


def test_rotation_equivariance(A, O):
    rec = O.synthesize(O.Scenario(train_symbols=64, data_symbols=16, snr_db=20.0, seed=31))
    w = A.lls_fit_widened(rec.train_rx, rec.train_symbols[:, 3], 4)
    rows = random_mat(1000, 4, 77) + 1j * random_mat(1000, 4, 78)
    g = O.narrow_predictions(O.widen_design(rows) @ w.w)
    gi = O.narrow_predictions(O.widen_design(1j * rows) @ w.w)
    assert np.max(np.abs(gi - 1j * g)) / np.max(np.abs(g)) < 1e-10


def test_batched_equals_independent_bitwise(A, O):
    rec = O.synthesize(O.Scenario(train_symbols=64, data_symbols=8, snr_db=15.0, seed=9))
    w0, cond, status = A.lls_fit_slots(rec.train_rx[None], rec.train_symbols[None])
    assert (status == 0).all()
    for k in range(6):
        wk, ck, sk = A.lls_fit_slots(rec.train_rx[None], rec.train_symbols[None, :, k:k + 1])
        assert np.array_equal(wk[0, 0], w0[0, k])


def _dup_design():
    x = np.zeros((6, 4))
    x[:, 0] = 1
    x[:, 1] = 1
    x[:, 2] = np.linspace(0, 5, 6)
    x[:, 3] = 2 * x[:, 2]
    return x


def test_min_norm_rank_deficient(A):
    x = _dup_design()
    y = np.ones(6) + 3 * x[:, 2]
    w = A.lls_fit(x, y).w
    assert np.linalg.norm(x @ w - y) < 1e-10
    assert np.allclose(w, np.linalg.pinv(x) @ y, rtol=1e-9, atol=1e-11)


def test_inconsistent_rank_deficient_raises(A):
    from paper_2206_05998_b200 import native as N

    x = _dup_design()
    y = np.zeros(6)
    y[0] = 1.0
    with pytest.raises(N.IllConditionedError) as e:
        A.lls_fit(x, y)
    assert e.value.gram_condition > 1e12


def test_dimension_errors(A):
    from paper_2206_05998_b200 import native as N

    with pytest.raises(N.DimensionError):
        A.lls_fit(np.ones((4, 8)), np.ones(4))
    with pytest.raises(N.DimensionError):
        A.lls_fit(np.ones((8, 4)), np.ones(7))


@pytest.mark.parametrize("M,K,step,snr,gain", [(16, 6, 3.0, 25.0, 0.05), (4, 6, 3.0, 10.0, 0.0),
                                               (64, 32, 1.0, 25.0, 0.05), (32, 16, 1.0, 25.0, 0.05),
                                               (16, 6, 3.0, float("inf"), 0.0)])
def test_slots_match_oracle(A, O, M, K, step, snr, gain):
    sc = O.Scenario(num_users=K, num_antennas=M, train_symbols=685, data_symbols=8,
                    power_step_db=step, snr_db=snr, rx_nonlinearity_gain=gain)
    S = 3
    recs = [O.synthesize(sc, O.seed_bundle(1000 + s)) for s in range(S)]
    px = np.stack([r.train_rx for r in recs])
    py = np.stack([r.train_symbols for r in recs])
    w0, cond, status = A.lls_fit_slots(px, py)
    assert (status == 0).all()
    for s, r in enumerate(recs):
        x = O.widen_design(r.train_rx)
        for k in range(K):
            ref = O.lls_fit(x, O.widen_targets(r.train_symbols[:, k]))
            err = np.linalg.norm(w0[s, k] - ref.w) / np.linalg.norm(ref.w)
            assert err < 1e-10, (s, k, err)
            assert abs(cond[s, k] - ref.gram_condition) < 1e-6 * ref.gram_condition
