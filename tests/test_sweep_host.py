"""Host-side logic of the GPU sweep harness (no GPU): seed conventions of
run_noise_sweep (eval.cpp:77-84, :212-219, :231-234) against the oracle's
compiled restatement, argument validation (eval.cpp:171-182) and the CSV
schema (eval.cpp:256-266)."""
import math
import random

import numpy as np
import pytest

from paper_2206_05998_b200 import sweep as S
from paper_2206_05998_b200.seeds import mix_tag, substream_seed


def test_mix_tag_matches_reference_function(O):
    rng = random.Random(3)
    for _ in range(300):
        a, b, c, d = (rng.getrandbits(rng.choice((2, 8, 32, 64))) for _ in range(4))
        assert mix_tag(a, b, c, d) == O.mix_tag(a, b, c, d)


@pytest.mark.parametrize("fresh", [True, False])
def test_trial_bundles(O, fresh):
    b = S.trial_bundles(99, 2, 4, fresh)
    for t in range(4):
        assert int(b[t, 0]) == O.substream_seed(99, 1)
        assert int(b[t, 1]) == O.substream_seed(99, O.mix_tag(2, t) if fresh else 2)
        assert int(b[t, 2]) == O.substream_seed(99, O.mix_tag(3, 2, t))
    assert substream_seed(99, 1) == O.substream_seed(99, 1)


@pytest.mark.parametrize("kw", [dict(snr_list=[]), dict(trials=0), dict(detectors=[]),
                                dict(users=[0]), dict(users=[7]), dict(detectors=["x"]),
                                dict(ablations=["y"])])
def test_argument_errors(kw):
    opts = S.SweepOptions(scenario=S.SweepScenario(num_users=3), snr_list=[10.0], trials=1)
    for k, v in kw.items():
        setattr(opts, k, v)
    with pytest.raises(S.ConfigError):
        S.run_noise_sweep(opts)


def test_csv_schema():
    c = S.BerCell(float("inf"), 2, S.LLS, S.SYM_OFF, 3, 600, [0.0, 0.25, 0.5])
    c.mean_ber = 0.25
    c.sd_ber = math.sqrt(1 / 24)
    rep = S.BerReport([c], 5, 3)
    lines = rep.to_csv().splitlines()
    assert lines[0] == "snr_db,user,detector,ablation,trials,mean_ber,sd_ber,total_bits"
    assert lines[1].split(",")[:6] == ["inf", "2", "LLS", "symmetry_off", "3", "0.25"]
    assert float(lines[1].split(",")[6]) == c.sd_ber
    assert lines[1].endswith(",600")
    np.testing.assert_allclose(float(lines[1].split(",")[6]), 0.2041241452319315)
