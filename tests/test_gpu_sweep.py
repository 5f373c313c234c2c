"""GPU noise sweep / symmetry ablation harness (sweep.py, eval.cpp:100-254)
against the FP64 oracle restatement: identical cell order, seeds and
per-trial BER (LLS exactly up to FP32 data rounding; the trained detectors
within the decision-flip allowance of FP32 vs FP64 training)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    from paper_2206_05998_b200 import api, sweep

    api.context()
    return sweep


def _opts(S, **kw):
    base = dict(scenario=S.SweepScenario(num_users=3, num_antennas=4, train_symbols=48,
                                         data_symbols=400, power_step_db=3.0,
                                         rx_nonlinearity_gain=0.05),
                snr_list=[4.0, 12.0], trials=2, detectors=[S.LLS, S.HYBRID],
                ablations=[S.SYM_ON, S.SYM_OFF, S.SYM_HALF], users=[], hidden_dims=[16],
                epochs=6, batch_size=32, lr=0.005, master_seed=17)
    base.update(kw)
    return S.SweepOptions(**base)


def test_sweep_matches_oracle(S, O):
    opts = _opts(S)
    rep = S.run_noise_sweep(opts)
    ref = O.run_noise_sweep_ref(opts)
    assert [(c.snr_db, c.detector, c.ablation, c.user) for c in rep.cells] == \
        [(s, d, a, u) for s in opts.snr_list for d in opts.detectors for a in opts.ablations
         for u in (1, 2, 3)]
    nbits = 2 * opts.scenario.data_symbols
    for c in rep.cells:
        r = ref[(opts.snr_list.index(c.snr_db), c.detector, c.ablation, c.user)]
        diff = np.abs(np.array(c.per_trial_ber) - np.array(r)) * nbits  # bit counts
        allow = 1 if c.detector == S.LLS else max(2, int(0.01 * nbits))
        assert diff.max() <= allow, (c, r)
        assert c.mean_ber == pytest.approx(np.mean(c.per_trial_ber))
        assert c.total_bits == nbits * opts.trials
    csv = rep.to_csv().splitlines()
    assert csv[0] == "snr_db,user,detector,ablation,trials,mean_ber,sd_ber,total_bits"
    assert len(csv) == len(rep.cells) + 1


def test_sweep_deterministic_and_noiseless_lls(S):
    """test_eval.cpp:57-100: noiseless LLS sweep has zero BER; reruns agree."""
    opts = _opts(S, snr_list=[float("inf")], detectors=[S.LLS], ablations=[S.SYM_ON],
                 scenario=S.SweepScenario(num_users=2, num_antennas=4, train_symbols=32,
                                          data_symbols=200))
    a = S.run_noise_sweep(opts)
    b = S.run_noise_sweep(opts)
    assert all(c.mean_ber == 0.0 for c in a.cells)
    assert a.to_csv() == b.to_csv()


def test_sweep_argument_errors(S):
    for kw in (dict(snr_list=[]), dict(trials=0), dict(detectors=[]), dict(users=[5])):
        with pytest.raises(S.ConfigError):
            S.run_noise_sweep(_opts(S, **kw))
