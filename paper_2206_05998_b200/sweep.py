"""Batched noise sweep / symmetry ablation harness on the GPU: run_noise_sweep
(eval.cpp:170-254) and detect_user (eval.cpp:100-166), SURVEY §8(f) next #2.

Same API and semantics as the reference (eval.hpp:35-73): cells in the order
snr -> detector -> ablation -> user; per trial the symbol stream is fixed by
the master seed, the channel optionally and the noise always get fresh
substreams (eval.cpp:212-219); every (trial, user, detector, ablation) draws
its init / shuffle seeds from mix_tag(si, trial, user, di << 8 | ai)
(eval.cpp:231-234, :125-129, :150-154).  What changes is the execution: for
one SNR point all trials are synthesised in one device call (explicit
SeedBundles), and every (detector, ablation) group trains and detects all
trials x users in one batched call -- widened ablations through
noma_pipeline, SymmetryOff (two independently trained real-valued target
slots per user, eval.cpp:135-165) through noma_lls_fit / noma_init_params /
noma_train / noma_detect on the REAL layout.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import api
from . import native as N
from .seeds import mix_tag, substream_seed

LLS, HYBRID = "LLS", "HybridNN"  # to_string(DetectorId), eval.cpp:12-14
SYM_ON, SYM_OFF, SYM_HALF = "symmetry_on", "symmetry_off", "symmetry_on_half_data"  # eval.cpp:16-23


class ConfigError(ValueError):
    """noma::config_error"""


@dataclass
class SweepScenario:
    """ScenarioConfig (channel_sim.hpp:14-28); snr_db is set per sweep point."""
    num_users: int = 6
    num_antennas: int = 4
    train_symbols: int = 685
    data_symbols: int = 3840
    power_step_db: float = 3.0
    rx_nonlinearity_gain: float = 0.0


@dataclass
class SweepOptions:
    """SweepOptions (eval.hpp:35-46)."""
    scenario: SweepScenario = field(default_factory=SweepScenario)
    snr_list: List[float] = field(default_factory=list)
    trials: int = 20
    detectors: List[str] = field(default_factory=lambda: [LLS, HYBRID])
    ablations: List[str] = field(default_factory=lambda: [SYM_ON])
    users: List[int] = field(default_factory=list)  # 1-based; empty = all
    hidden_dims: List[int] = field(default_factory=lambda: [64, 64, 64])
    epochs: int = 50
    batch_size: int = 128
    lr: float = 0.005
    fresh_channel_per_trial: bool = True
    master_seed: int = 0


@dataclass
class BerCell:
    """BerCell (eval.hpp:48-58)."""
    snr_db: float
    user: int
    detector: str
    ablation: str
    trials: int
    total_bits: int
    per_trial_ber: List[float] = field(default_factory=list)
    mean_ber: float = 0.0
    sd_ber: float = 0.0


@dataclass
class BerReport:
    cells: List[BerCell]
    master_seed: int
    trials: int

    def to_csv(self) -> str:
        """BerReport::to_csv (eval.cpp:256-266); repr() of a float is the
        shortest round-trip form, like format_double (format.hpp:9-13)."""
        out = ["snr_db,user,detector,ablation,trials,mean_ber,sd_ber,total_bits"]
        for c in self.cells:
            out.append(f"{_fmt(c.snr_db)},{c.user},{c.detector},{c.ablation},{c.trials},"
                       f"{_fmt(c.mean_ber)},{_fmt(c.sd_ber)},{c.total_bits}")
        return "\n".join(out) + "\n"


def _fmt(x: float) -> str:
    if math.isinf(x):
        return "inf" if x > 0 else "-inf"
    r = repr(float(x))
    return r[:-2] if r.endswith(".0") else r


def trial_bundles(master: int, si: int, trials: int, fresh_channel: bool) -> np.ndarray:
    """SeedBundle per trial (eval.cpp:212-219)."""
    out = np.empty((trials, 3), dtype=np.uint64)
    for t in range(trials):
        out[t, 0] = substream_seed(master, 1)
        out[t, 1] = (substream_seed(master, mix_tag(2, t)) if fresh_channel
                     else substream_seed(master, 2))
        out[t, 2] = substream_seed(master, mix_tag(3, si, t))
    return out


def _validate(opts: SweepOptions):
    # run_noise_sweep argument checks (eval.cpp:171-182) + ScenarioConfig::validate
    if not opts.snr_list:
        raise ConfigError("run_noise_sweep: empty SNR list")
    if opts.trials < 1:
        raise ConfigError("run_noise_sweep: trials must be >= 1")
    if not opts.detectors:
        raise ConfigError("run_noise_sweep: no detectors")
    sc = opts.scenario
    if (sc.num_users < 1 or sc.num_antennas < 1 or sc.data_symbols < 1
            or sc.train_symbols < 2 * sc.num_antennas or sc.power_step_db < 0
            or sc.rx_nonlinearity_gain < 0):
        raise ConfigError("invalid scenario")
    users = list(opts.users) or list(range(1, sc.num_users + 1))
    for u in users:
        if u < 1 or u > sc.num_users:
            raise ConfigError("run_noise_sweep: user index out of range")
    for d in opts.detectors:
        if d not in (LLS, HYBRID):
            raise ConfigError(f"unknown detector id: {d}")
    for a in opts.ablations:
        if a not in (SYM_ON, SYM_OFF, SYM_HALF):
            raise ConfigError(f"unknown ablation: {a}")
    return users


def run_noise_sweep(opts: SweepOptions) -> BerReport:
    users = _validate(opts)
    sc = opts.scenario
    K, M, NT, ND = sc.num_users, sc.num_antennas, sc.train_symbols, sc.data_symbols
    T = opts.trials
    bits_per_trial = 2 * ND
    cells = []
    index = {}
    for si, snr in enumerate(opts.snr_list):
        for di, det in enumerate(opts.detectors):
            for ai, abl in enumerate(opts.ablations):
                for u in users:
                    index[(si, di, ai, u)] = len(cells)
                    cells.append(BerCell(snr, u, det, abl, T, bits_per_trial * T))
    ctx = api.context()
    for si, snr in enumerate(opts.snr_list):
        scn = N.Scenario(K, M, NT, ND, sc.power_step_db, snr, sc.rx_nonlinearity_gain)
        bundles = trial_bundles(opts.master_seed, si, T, opts.fresh_channel_per_trial)
        px = np.zeros((T, NT, M), np.complex128)
        py = np.zeros((T, NT, K), np.complex128)
        dx = np.zeros((T, ND, M), np.complex64)
        codes = np.zeros((T, ND, K), np.uint8)
        ctx.synthesize_bundles(scn, bundles, px.view(np.float64), py.view(np.float64),
                               dx.view(np.float32), codes)
        for di, det in enumerate(opts.detectors):
            for ai, abl in enumerate(opts.ablations):
                tags = {(t, u): mix_tag(si, t, u, (di << 8) | ai) for t in range(T) for u in users}
                if abl == SYM_OFF:
                    ber = _symmetry_off(opts, det, tags, users, px, py, dx, codes)
                else:
                    ber = _widened(opts, det, abl, tags, users, px, py, dx, codes)
                for t in range(T):
                    for u in users:
                        cells[index[(si, di, ai, u)]].per_trial_ber.append(ber[t, u - 1])
    for c in cells:  # population mean / SD (eval.cpp:244-252)
        b = np.asarray(c.per_trial_ber)
        c.mean_ber = float(b.sum() / b.size)
        c.sd_ber = float(math.sqrt(((b - c.mean_ber) ** 2).sum() / b.size))
    return BerReport(cells, opts.master_seed, T)


def _widened(opts, det, abl, tags, users, px, py, dx, codes):
    """SymmetryOn / SymmetryOnHalfData (eval.cpp:108-131): widened design of
    all (or the first half of the) pilot symbols; LLS = the net at init
    (zero final layer: detect == lls::predict, test_hybrid_nn.cpp:313-340)."""
    T, NT, M = px.shape
    K = py.shape[2]
    if abl == SYM_HALF:
        half = NT // 2
        px, py = np.ascontiguousarray(px[:, :half]), np.ascontiguousarray(py[:, :half])
    ms = opts.master_seed
    init = np.zeros((T, K), np.uint64)
    shuf = np.zeros((T, K), np.uint64)
    for (t, u), tag in tags.items():
        init[t, u - 1] = substream_seed(ms, mix_tag(tag, 11))
        shuf[t, u - 1] = substream_seed(ms, mix_tag(tag, 12))
    epochs = 0 if det == LLS else opts.epochs
    dims = [2 * M] + list(opts.hidden_dims)
    out = api.pipeline(dims, px, py, dx, codes, init, shuf, epochs=epochs,
                       batch_size=opts.batch_size, lr=opts.lr)
    if (out.status != 0).any():
        raise N.IllConditionedError(3, "lls::fit: design matrix rank deficient and system inconsistent",
                                    float(out.gram_condition[out.status != 0][0]))
    return out.bit_errors.astype(np.float64) / (2 * dx.shape[1])


def _symmetry_off(opts, det, tags, users, px, py, dx, codes):
    """SymmetryOff (eval.cpp:135-165): non-widened real design [Re r; Im r]
    (N_T x 2M), one independently fitted / trained slot per real target
    (Re, Im), predictions recombined into complex symbols."""
    ctx = api.context()
    T, NT, M = px.shape
    ND = dx.shape[1]
    U = len(users)
    ms = opts.master_seed
    design = np.ascontiguousarray(np.concatenate([px.real, px.imag], axis=2))      # [T][NT][2M]
    ddata = np.ascontiguousarray(np.concatenate([dx.real, dx.imag], axis=2), np.float32)
    targets = np.zeros((T, 2 * U, NT))
    init = np.zeros((T, 2 * U), np.uint64)
    shuf = np.zeros((T, 2 * U), np.uint64)
    for t in range(T):
        for i, u in enumerate(users):
            y = py[t, :, u - 1]
            targets[t, 2 * i] = y.real
            targets[t, 2 * i + 1] = y.imag
            for slot in (1, 2):
                init[t, 2 * i + slot - 1] = substream_seed(ms, mix_tag(tags[(t, u)], 11, slot))
                shuf[t, 2 * i + slot - 1] = substream_seed(ms, mix_tag(tags[(t, u)], 12, slot))
    nets = T * 2 * U
    w0 = np.zeros((nets, 2 * M))
    cond = np.zeros(nets)
    status = np.zeros(nets, np.int32)
    ctx.lls_fit(N.LAYOUT_REAL, T, 2 * U, NT, 2 * M, design, targets, w0, cond, status)
    dims = [2 * M] + list(opts.hidden_dims)
    plans = np.zeros((nets, N.plan_size(dims)), np.float32)
    ctx.init_params(dims, init.reshape(-1), w0, plans)
    if det == HYBRID:
        ctx.train(N.LAYOUT_REAL, T, 2 * U, NT, 2 * M, design, targets, dims,
                  N.TrainCfg.of(opts.epochs, opts.batch_size, opts.lr), w0, plans, shuf.reshape(-1))
    soft = np.zeros((nets, ND), np.float32)
    ctx.detect(dims, N.LAYOUT_REAL, T, 2 * U, ND, ddata, plans, soft=soft)
    soft = soft.reshape(T, U, 2, ND)
    K = codes.shape[2]
    ber = np.zeros((T, K))
    for i, u in enumerate(users):
        pred = (soft[:, i, 0] < 0).astype(np.uint8) | ((soft[:, i, 1] < 0).astype(np.uint8) << 1)
        truth = codes[:, :, u - 1]
        ber[:, u - 1] = np.array([np.unpackbits((pred[t] ^ truth[t]).astype(np.uint8)).sum()
                                  for t in range(T)]) / (2 * ND)
    return ber
