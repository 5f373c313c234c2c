"""TEST INFRASTRUCTURE ONLY -- numpy/ctypes front end of the FP64 CPU oracle.

The oracle (oracle/*.c, built by oracle/Makefile into oracle/_build/liboracle.so)
restates the reference detector path (arxiv 2206.05998 "noma-detect",
proj/src/*.cpp) in plain C.  Only tests/, __graft_entry__.smoke() and the
CPU-baseline legs of bench.py may import this module, and only as the checker
or as the timed CPU baseline; the product (paper_2206_05998_b200) never does.

Array conventions: complex arrays are numpy complex128; real matrices are
row-major float64.  Functions mirror the reference API names.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None

OK, ERR_DIMENSION, ERR_CONFIG, ERR_ILL = 0, 1, 2, 3

_dp = C.POINTER(C.c_double)
_fp = C.POINTER(C.c_float)
_ip = C.POINTER(C.c_int)
_u64p = C.POINTER(C.c_uint64)
_lp = C.POINTER(C.c_long)
_u8p = C.POINTER(C.c_uint8)
MAX_DIMS = 9


class OracleError(Exception):
    def __init__(self, code, msg=""):
        super().__init__(f"oracle status {code} {msg}")
        self.code = code


class DimensionError(OracleError):
    pass


class ConfigError(OracleError):
    pass


class IllConditionedError(OracleError):
    def __init__(self, code, cond):
        super().__init__(code, f"gram_condition={cond}")
        self.gram_condition = cond


def _raise(code, cond=None):
    if code == OK:
        return
    if code == ERR_DIMENSION:
        raise DimensionError(code)
    if code == ERR_CONFIG:
        raise ConfigError(code)
    if code == ERR_ILL:
        raise IllConditionedError(code, cond)
    raise OracleError(code)


def build():
    """Compile the oracle with its Makefile (idempotent)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        L.orc_splitmix64.restype = C.c_uint64
        L.orc_splitmix64.argtypes = [_u64p]
        L.orc_substream_seed.restype = C.c_uint64
        L.orc_substream_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_mix_tag.restype = C.c_uint64
        L.orc_mix_tag.argtypes = [C.c_uint64] * 4
        L.orc_rng_fill_u64.argtypes = [C.c_uint64, C.c_int, _u64p]
        L.orc_rng_fill_gaussian.argtypes = [C.c_uint64, C.c_int, _dp]
        L.orc_power_profile.argtypes = [C.c_int, C.c_double, _dp]
        L.orc_synthesize.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64] + [_dp] * 7
        L.orc_seed_bundle.argtypes = [C.c_uint64, _u64p]
        L.orc_widen_design.argtypes = [C.c_int, C.c_int, _dp, _dp]
        L.orc_lls_fit.argtypes = [C.c_int, C.c_int, _dp, _dp, _dp, _dp]
        L.orc_singular_values.argtypes = [C.c_int, C.c_int, _dp, _dp]
        L.orc_param_count.argtypes = [C.c_int, _ip]
        L.orc_init_params.argtypes = [C.c_int, _ip, C.c_void_p, _dp]
        L.orc_rng_seed.argtypes = [C.c_void_p, C.c_uint64]
        L.orc_rng_next.restype = C.c_uint64
        L.orc_rng_next.argtypes = [C.c_void_p]
        L.orc_rng_uniform.restype = C.c_double
        L.orc_rng_uniform.argtypes = [C.c_void_p]
        L.orc_rng_below.restype = C.c_uint64
        L.orc_rng_below.argtypes = [C.c_void_p, C.c_uint64]
        L.orc_rng_gaussian.restype = C.c_double
        L.orc_rng_gaussian.argtypes = [C.c_void_p]
        L.orc_forward.argtypes = [C.c_int, _ip, _dp, _dp, C.c_int, _dp, _dp]
        L.orc_loss_and_grad.argtypes = [C.c_int, _ip, _dp, _dp, C.c_int, _dp, _dp, _dp, _dp]
        L.orc_adam_step.argtypes = [C.c_int, _dp, _dp, _dp, _dp, _lp] + [C.c_double] * 4
        L.orc_train.argtypes = [C.c_int, _ip, _dp, _dp, C.c_int, _dp, _dp, C.c_int, C.c_int,
                                C.c_double, C.c_uint64, _dp]
        L.orc_shuffled_indices.argtypes = [C.c_int, C.c_uint64, C.c_int, _ip]
        L.orc_plan_size.argtypes = [C.c_int, _ip]
        L.orc_build_plan.argtypes = [C.c_int, _ip, _dp, _dp, _dp]
        L.orc_unpack_plan.argtypes = [C.c_int, _ip, _dp, _dp, _dp]
        L.orc_fused_forward_f64.argtypes = [C.c_int, _ip, _dp, C.c_int, _dp, _dp]
        L.orc_fused_forward_f32.argtypes = [C.c_int, _ip, _fp, C.c_int, _fp, _fp]
        L.orc_bench_fused_ns.restype = C.c_double
        L.orc_bench_fused_ns.argtypes = [C.c_int, _ip, _dp, C.c_int, _dp, C.c_int, _dp]
        L.orc_slot_run.argtypes = [C.c_void_p, C.c_uint64, _dp, _dp, _ip, _dp, _dp, _dp, _lp]
        L.orc_slots_run_threaded.argtypes = [C.c_void_p, C.c_int, _u64p, C.c_int, _dp, _dp,
                                             _ip, _dp, _dp, _dp, _lp]
        _lib = L
    return _lib


def _d(a):
    return a.ctypes.data_as(_dp)


def _c64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _dims(dims):
    return (C.c_int * len(dims))(*dims)


class _Rng(C.Structure):
    _fields_ = [("s", C.c_uint64 * 4)]


class _Scenario(C.Structure):
    _fields_ = [("num_users", C.c_int), ("num_antennas", C.c_int),
                ("train_symbols", C.c_int), ("data_symbols", C.c_int),
                ("power_step_db", C.c_double), ("snr_db", C.c_double),
                ("rx_nonlinearity_gain", C.c_double)]


class _SlotCfg(C.Structure):
    _fields_ = [("sc", _Scenario), ("ndims", C.c_int), ("dims", C.c_int * MAX_DIMS),
                ("epochs", C.c_int), ("batch", C.c_int), ("lr", C.c_double)]


# ------------------------------------------------------------------ rng.hpp
def splitmix64(state: int):
    s = C.c_uint64(state)
    out = lib().orc_splitmix64(C.byref(s))
    return out, s.value


def substream_seed(master: int, tag: int) -> int:
    return lib().orc_substream_seed(master, tag)


def mix_tag(a, b, c=0, d=0) -> int:
    return lib().orc_mix_tag(a, b, c, d)


def rng_u64(seed: int, n: int) -> np.ndarray:
    out = np.empty(n, dtype=np.uint64)
    lib().orc_rng_fill_u64(seed, n, out.ctypes.data_as(_u64p))
    return out


def rng_gaussian(seed: int, n: int) -> np.ndarray:
    out = np.empty(n, dtype=np.float64)
    lib().orc_rng_fill_gaussian(seed, n, _d(out))
    return out


class Rng:
    """Stateful xoshiro256++ handle (rng.hpp:28-67)."""

    def __init__(self, seed: int):
        self._r = _Rng()
        lib().orc_rng_seed(C.byref(self._r), seed)

    def next_u64(self) -> int:
        return lib().orc_rng_next(C.byref(self._r))

    def uniform(self) -> float:
        return lib().orc_rng_uniform(C.byref(self._r))

    def below(self, bound: int) -> int:
        return lib().orc_rng_below(C.byref(self._r), bound)

    def gaussian(self) -> float:
        return lib().orc_rng_gaussian(C.byref(self._r))

    def state(self):
        return tuple(self._r.s)


# ---------------------------------------------------------- channel_sim
@dataclass
class Scenario:
    num_users: int = 6
    num_antennas: int = 4
    train_symbols: int = 685
    data_symbols: int = 3840
    power_step_db: float = 3.0
    snr_db: float = float("inf")
    rx_nonlinearity_gain: float = 0.0
    seed: int = 0

    def _c(self):
        return _Scenario(self.num_users, self.num_antennas, self.train_symbols,
                         self.data_symbols, self.power_step_db, self.snr_db,
                         self.rx_nonlinearity_gain)


@dataclass
class Record:
    channel: np.ndarray      # M x K complex
    powers: np.ndarray       # K
    train_rx: np.ndarray     # NT x M complex
    train_symbols: np.ndarray
    data_rx: np.ndarray
    data_symbols: np.ndarray
    noise_power: float


def seed_bundle(master: int):
    out = np.empty(3, dtype=np.uint64)
    lib().orc_seed_bundle(master, out.ctypes.data_as(_u64p))
    return tuple(int(v) for v in out)


def power_profile(k: int, step_db: float) -> np.ndarray:
    out = np.empty(k)
    lib().orc_power_profile(k, step_db, _d(out))
    return out


def synthesize(sc: Scenario, seeds=None) -> Record:
    K, M, NT, ND = sc.num_users, sc.num_antennas, sc.train_symbols, sc.data_symbols
    if seeds is None:
        seeds = seed_bundle(sc.seed)
    ch = np.empty((M, K), np.complex128)
    pw = np.empty(K)
    trx = np.empty((NT, M), np.complex128)
    tsy = np.empty((NT, K), np.complex128)
    drx = np.empty((ND, M), np.complex128)
    dsy = np.empty((ND, K), np.complex128)
    npw = C.c_double(0)
    cs = sc._c()
    st = lib().orc_synthesize(C.byref(cs), seeds[0], seeds[1], seeds[2],
                              *(a.ctypes.data_as(_dp) for a in (ch, pw, trx, tsy, drx, dsy)),
                              C.byref(npw))
    _raise(st)
    return Record(ch, pw, trx, tsy, drx, dsy, npw.value)


# --------------------------------------------------------- iq_transform
def widen_design(x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.complex128)
    n, m = x.shape
    out = np.empty((2 * n, 2 * m))
    _raise(lib().orc_widen_design(n, m, x.ctypes.data_as(_dp), _d(out)))
    return out


def widen_targets(y: np.ndarray) -> np.ndarray:
    y = np.asarray(y, dtype=np.complex128)
    out = np.empty(2 * y.size)
    out[0::2] = y.real
    out[1::2] = y.imag
    return out


def narrow_predictions(yhat: np.ndarray) -> np.ndarray:
    if yhat.size % 2:
        raise DimensionError(ERR_DIMENSION)
    return yhat[0::2] + 1j * yhat[1::2]


# ------------------------------------------------------------------ lls
@dataclass
class LlsWeights:
    w: np.ndarray
    user_index: int = 0
    gram_condition: float = 0.0


def lls_fit(design: np.ndarray, targets: np.ndarray, user_index: int = 0) -> LlsWeights:
    x = _c64(design)
    y = _c64(targets)
    rows, cols = x.shape
    if rows != y.size:
        raise DimensionError(ERR_DIMENSION)
    w = np.zeros(cols)
    cond = C.c_double(0)
    st = lib().orc_lls_fit(rows, cols, _d(x), _d(y), _d(w), C.byref(cond))
    _raise(st, cond.value)
    return LlsWeights(w, user_index, cond.value)


def singular_values(x: np.ndarray) -> np.ndarray:
    x = _c64(x)
    sv = np.empty(x.shape[1])
    _raise(lib().orc_singular_values(x.shape[0], x.shape[1], _d(x), _d(sv)))
    return sv


# ------------------------------------------------------------ hybrid_nn
@dataclass
class HybridNet:
    """HybridNetParams (hybrid_nn.hpp:15-23) with a flat trainable vector."""
    dims: list
    w0: np.ndarray
    theta: np.ndarray = field(repr=False)

    def layers(self):
        """[(W_l, b_l)], final -- views into theta."""
        out, off = [], 0
        d = self.dims
        for l in range(1, len(d)):
            W = self.theta[off:off + d[l] * d[l - 1]].reshape(d[l], d[l - 1])
            off += d[l] * d[l - 1]
            b = self.theta[off:off + d[l]]
            off += d[l]
            out.append((W, b))
        return out, self.theta[off:off + d[-1]]

    def trainable_count(self):
        return self.theta.size


def param_count(dims) -> int:
    return lib().orc_param_count(len(dims), _dims(dims))


def init_params(dims, w0: np.ndarray, rng: Rng) -> HybridNet:
    if len(dims) == 0 or dims[0] != len(w0):
        raise DimensionError(ERR_DIMENSION)
    theta = np.empty(param_count(dims)) if min(dims) >= 1 else None
    if theta is None:
        raise DimensionError(ERR_DIMENSION)
    _raise(lib().orc_init_params(len(dims), _dims(dims), C.byref(rng._r), _d(theta)))
    return HybridNet(list(dims), np.array(w0, dtype=np.float64), theta)


def forward(net: HybridNet, x: np.ndarray) -> np.ndarray:
    x = _c64(x)
    if x.shape[1] != net.dims[0]:
        raise DimensionError(ERR_DIMENSION)
    out = np.empty(x.shape[0])
    _raise(lib().orc_forward(len(net.dims), _dims(net.dims), _d(_c64(net.w0)),
                             _d(net.theta), x.shape[0], _d(x), _d(out)))
    return out


def loss_and_grad(net: HybridNet, x: np.ndarray, y: np.ndarray):
    x = _c64(x)
    y = _c64(y)
    if x.shape[0] == 0:
        raise DimensionError(ERR_DIMENSION)
    if x.shape[1] != net.dims[0] or y.size != x.shape[0]:
        raise DimensionError(ERR_DIMENSION)
    g = np.empty_like(net.theta)
    loss = C.c_double(0)
    _raise(lib().orc_loss_and_grad(len(net.dims), _dims(net.dims), _d(_c64(net.w0)),
                                   _d(net.theta), x.shape[0], _d(x), _d(y), C.byref(loss),
                                   _d(g)))
    return loss.value, g


class AdamState:
    def __init__(self, p: int, lr: float):
        self.m = np.zeros(p)
        self.v = np.zeros(p)
        self.step = C.c_long(0)
        self.lr, self.beta1, self.beta2, self.eps = lr, 0.9, 0.999, 1e-8


def adam_step(net: HybridNet, grad: np.ndarray, s: AdamState):
    g = _c64(grad)
    lib().orc_adam_step(net.theta.size, _d(net.theta), _d(g), _d(s.m), _d(s.v),
                        C.byref(s.step), s.lr, s.beta1, s.beta2, s.eps)


def shuffled_indices(n: int, shuffle_seed: int, epoch: int) -> np.ndarray:
    idx = np.empty(n, dtype=np.int32)
    lib().orc_shuffled_indices(n, shuffle_seed, epoch, idx.ctypes.data_as(_ip))
    return idx


def train(net: HybridNet, x: np.ndarray, y: np.ndarray, epochs=50, batch_size=128, lr=0.005,
          shuffle_seed=0) -> np.ndarray:
    x = _c64(x)
    y = _c64(y)
    trace = np.empty(max(epochs, 0))
    st = lib().orc_train(len(net.dims), _dims(net.dims), _d(_c64(net.w0)), _d(net.theta),
                         x.shape[0], _d(x), _d(y), epochs, batch_size, lr, shuffle_seed,
                         _d(trace))
    _raise(st)
    return trace


def detect(net: HybridNet, widened: np.ndarray) -> np.ndarray:
    return narrow_predictions(forward(net, widened))


# ---------------------------------------------------------------- fused
def plan_size(dims) -> int:
    return lib().orc_plan_size(len(dims), _dims(dims))


def build_plan(net: HybridNet) -> np.ndarray:
    buf = np.empty(plan_size(net.dims))
    lib().orc_build_plan(len(net.dims), _dims(net.dims), _d(_c64(net.w0)), _d(net.theta),
                         _d(buf))
    return buf


def unpack_plan(dims, buf: np.ndarray) -> HybridNet:
    w0 = np.empty(dims[0])
    theta = np.empty(param_count(dims))
    lib().orc_unpack_plan(len(dims), _dims(dims), _d(_c64(buf)), _d(w0), _d(theta))
    return HybridNet(list(dims), w0, theta)


def fused_forward(dims, buf: np.ndarray, x: np.ndarray) -> np.ndarray:
    x = _c64(x)
    out = np.empty(x.shape[0])
    lib().orc_fused_forward_f64(len(dims), _dims(dims), _d(_c64(buf)), x.shape[0], _d(x),
                                _d(out))
    return out


def fused_forward_f32(dims, buf: np.ndarray, x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float32)
    b32 = np.ascontiguousarray(buf, dtype=np.float32)
    out = np.empty(x.shape[0], dtype=np.float32)
    lib().orc_fused_forward_f32(len(dims), _dims(dims), b32.ctypes.data_as(_fp), x.shape[0],
                                x.ctypes.data_as(_fp), out.ctypes.data_as(_fp))
    return out


def bench_fused_ns(dims, buf, x, repeats=5) -> float:
    x = _c64(x)
    out = np.empty(x.shape[0])
    return lib().orc_bench_fused_ns(len(dims), _dims(dims), _d(_c64(buf)), x.shape[0], _d(x),
                                    repeats, _d(out))


# ----------------------------------------------------------------- eval
def hard_decision_qpsk(sym: np.ndarray) -> np.ndarray:
    sym = np.asarray(sym, dtype=np.complex128)
    return np.stack([(sym.real < 0), (sym.imag < 0)], axis=1).astype(np.uint8)


def map_qpsk_bits(bits: np.ndarray) -> np.ndarray:
    a = 1.0 / np.sqrt(2.0)
    b = bits.astype(np.int64)
    return (1 - 2 * b[:, 0]) * a + 1j * (1 - 2 * b[:, 1]) * a


def bit_error_rate(pred: np.ndarray, truth: np.ndarray) -> float:
    if pred.shape != truth.shape:
        raise DimensionError(ERR_DIMENSION)
    if pred.size == 0:
        raise DimensionError(ERR_DIMENSION)
    return float(np.count_nonzero(pred != truth)) / pred.size


# ------------------------------------------------------------- pipeline
@dataclass
class SlotResult:
    w0: np.ndarray          # S x K x 2M
    gram_condition: np.ndarray
    status: np.ndarray
    plans: np.ndarray       # S x K x plan_size
    trace: np.ndarray       # S x K x epochs
    soft: np.ndarray        # S x K x ND complex (or None)
    bit_errors: np.ndarray  # S x K


def slot_cfg(sc: Scenario, hidden, epochs=50, batch=128, lr=0.005):
    dims = [2 * sc.num_antennas] + list(hidden)
    c = _SlotCfg()
    c.sc = sc._c()
    c.ndims = len(dims)
    for i, v in enumerate(dims):
        c.dims[i] = v
    c.epochs, c.batch, c.lr = epochs, batch, lr
    return c, dims


def run_slots(sc: Scenario, hidden, seeds, epochs=50, batch=128, lr=0.005, threads=1,
              want_soft=True) -> SlotResult:
    cfg, dims = slot_cfg(sc, hidden, epochs, batch, lr)
    S, K, w = len(seeds), sc.num_users, dims[0]
    ps = plan_size(dims)
    w0 = np.zeros((S, K, w))
    cond = np.zeros((S, K))
    status = np.zeros((S, K), dtype=np.int32)
    plans = np.zeros((S, K, ps))
    trace = np.zeros((S, K, max(epochs, 1)))
    soft = np.zeros((S, K, 2 * sc.data_symbols)) if want_soft else None
    errs = np.zeros((S, K), dtype=np.int64)
    sd = np.asarray(seeds, dtype=np.uint64)
    lib().orc_slots_run_threaded(C.byref(cfg), S, sd.ctypes.data_as(_u64p), threads, _d(w0),
                                 _d(cond), status.ctypes.data_as(_ip), _d(plans), _d(trace),
                                 _d(soft) if soft is not None else None,
                                 errs.ctypes.data_as(_lp))
    soft_c = soft[..., 0::2] + 1j * soft[..., 1::2] if soft is not None else None
    return SlotResult(w0, cond, status, plans, trace[..., :epochs], soft_c, errs)


# ---------------------------------------------------------------- sweep
# TEST INFRASTRUCTURE: FP64 restatement of detect_user / run_noise_sweep
# (eval.cpp:100-254) over the primitives above, the checker for
# paper_2206_05998_b200.sweep (small sizes only).
def real_design(x: np.ndarray) -> np.ndarray:
    """eval.cpp:69-74: one row [Re r; Im r] per symbol."""
    return np.concatenate([x.real, x.imag], axis=1)


def detect_user_ref(opts, rec, user, det, abl, trial_tag):
    """eval.cpp:100-166 (det in {"LLS", "HybridNN"}; abl in {"symmetry_on",
    "symmetry_off", "symmetry_on_half_data"})."""
    ms = opts.master_seed
    dims_h = list(opts.hidden_dims)
    y = rec.train_symbols[:, user - 1]
    wd = widen_design(rec.data_rx)
    if abl != "symmetry_off":
        if abl == "symmetry_on":
            design, targets = widen_design(rec.train_rx), widen_targets(y)
        else:
            half = rec.train_rx.shape[0] // 2
            design, targets = widen_design(rec.train_rx[:half]), widen_targets(y[:half])
        w = lls_fit(design, targets, user)
        if det == "LLS":
            return narrow_predictions(wd @ w.w)
        net = init_params([design.shape[1]] + dims_h, w.w,
                          Rng(substream_seed(ms, mix_tag(trial_tag, 11))))
        train(net, design, targets, opts.epochs, opts.batch_size, opts.lr,
              substream_seed(ms, mix_tag(trial_tag, 12)))
        return detect(net, wd)
    rt, rd = real_design(rec.train_rx), real_design(rec.data_rx)
    preds = []
    for slot, yy in ((1, y.real.copy()), (2, y.imag.copy())):
        w = lls_fit(rt, yy, user)
        if det == "LLS":
            preds.append(rd @ w.w)
            continue
        net = init_params([rt.shape[1]] + dims_h, w.w,
                          Rng(substream_seed(ms, mix_tag(trial_tag, 11, slot))))
        train(net, rt, yy, opts.epochs, opts.batch_size, opts.lr,
              substream_seed(ms, mix_tag(trial_tag, 12, slot)))
        preds.append(forward(net, rd))
    return preds[0] + 1j * preds[1]


def run_noise_sweep_ref(opts):
    """eval.cpp:170-254 -> {(snr_index, detector, ablation, user): [ber per trial]}."""
    sc = opts.scenario
    users = list(opts.users) or list(range(1, sc.num_users + 1))
    out = {}
    for si, snr in enumerate(opts.snr_list):
        scn = Scenario(sc.num_users, sc.num_antennas, sc.train_symbols, sc.data_symbols,
                       sc.power_step_db, snr, sc.rx_nonlinearity_gain)
        for t in range(opts.trials):
            seeds = (substream_seed(opts.master_seed, 1),
                     substream_seed(opts.master_seed, mix_tag(2, t)) if opts.fresh_channel_per_trial
                     else substream_seed(opts.master_seed, 2),
                     substream_seed(opts.master_seed, mix_tag(3, si, t)))
            rec = synthesize(scn, seeds)
            for di, det in enumerate(opts.detectors):
                for ai, abl in enumerate(opts.ablations):
                    for u in users:
                        tag = mix_tag(si, t, u, (di << 8) | ai)
                        pred = detect_user_ref(opts, rec, u, det, abl, tag)
                        ber = bit_error_rate(hard_decision_qpsk(pred),
                                             hard_decision_qpsk(rec.data_symbols[:, u - 1]))
                        out.setdefault((si, det, abl, u), []).append(ber)
    return out
