"""Python mirror of the reference detector API (proj/include/noma) on the GPU.

Names and argument meaning follow the reference headers -- lls::fit
(lls.hpp:19-21), hybrid_nn::init_params / train / detect (hybrid_nn.hpp:55-75),
fused::fused_forward_f32 (fused_inference.hpp:60), widen_* (iq_transform.hpp:
20-29), hard_decision_qpsk / bit_error_rate (eval.hpp:27-33) -- so the parity
tests read like the reference's own tests.  Every compute call goes through the
C-ABI (native.py -> libnoma_b200.so); numpy in, numpy out.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import native as N

_ctx = None


def context() -> N.Context:
    global _ctx
    if _ctx is None:
        _ctx = N.Context(0)
    return _ctx


# ------------------------------------------------------------------ lls
@dataclass
class LlsWeights:
    w: np.ndarray
    user_index: int = 0
    gram_condition: float = 0.0


def _fit(layout, S, K, rows, width, design, targets):
    w0 = np.zeros((S, K, width))
    cond = np.zeros((S, K))
    status = np.zeros((S, K), dtype=np.int32)
    try:
        context().lls_fit(layout, S, K, rows, width, design, targets, w0, cond, status)
    except N.IllConditionedError as e:
        bad = np.argwhere(status != 0)
        e.gram_condition = float(cond[tuple(bad[0])])
        e.status = status
        raise
    return w0, cond, status


def lls_fit(design: np.ndarray, targets: np.ndarray, user_index: int = 0) -> LlsWeights:
    """lls::fit(Mat, Vec, int) -- arbitrary real design (lls.cpp:10-54)."""
    x = np.ascontiguousarray(design, dtype=np.float64)
    y = np.ascontiguousarray(targets, dtype=np.float64)
    rows, cols = x.shape
    if rows < cols or rows != y.size:
        raise N.DimensionError(N.ERR_DIMENSION, "lls::fit: dimension mismatch")
    w0, cond, _ = _fit(N.LAYOUT_REAL, 1, 1, rows, cols, x, y.reshape(1, 1, rows))
    return LlsWeights(w0[0, 0], user_index, float(cond[0, 0]))


def lls_fit_widened(x: np.ndarray, y: np.ndarray, user_index: int = 0) -> LlsWeights:
    """lls::fit(widen_dataset(x, y)) with the widening done on device."""
    x = np.ascontiguousarray(x, dtype=np.complex128)
    y = np.ascontiguousarray(np.asarray(y, dtype=np.complex128).reshape(-1, 1))
    n, m = x.shape
    w0, cond, _ = _fit(N.LAYOUT_WIDEN, 1, 1, 2 * n, 2 * m, x.view(np.float64),
                       y.view(np.float64))
    return LlsWeights(w0[0, 0], user_index, float(cond[0, 0]))


def lls_fit_slots(pilot_rx: np.ndarray, pilot_sym: np.ndarray):
    """Batched: pilot_rx [S,NT,M] complex, pilot_sym [S,NT,K] complex ->
    w0 [S,K,2M], gram_condition [S,K], status [S,K] (no exception)."""
    px = np.ascontiguousarray(pilot_rx, dtype=np.complex128)
    py = np.ascontiguousarray(pilot_sym, dtype=np.complex128)
    S, NT, M = px.shape
    K = py.shape[2]
    w0 = np.zeros((S, K, 2 * M))
    cond = np.zeros((S, K))
    status = np.zeros((S, K), dtype=np.int32)
    try:
        context().lls_fit(N.LAYOUT_WIDEN, S, K, 2 * NT, 2 * M, px.view(np.float64),
                          py.view(np.float64), w0, cond, status)
    except N.IllConditionedError:
        pass
    return w0, cond, status


def lls_predict(w: np.ndarray, widened_design: np.ndarray) -> np.ndarray:
    """lls::predict (lls.cpp:62-66): narrow(X w) in FP64 on device."""
    x = np.ascontiguousarray(widened_design, dtype=np.float64)
    w = np.ascontiguousarray(w, dtype=np.float64)
    if x.shape[1] != w.size:
        raise N.DimensionError(N.ERR_DIMENSION, "lls::predict: column count does not match weights")
    if x.shape[0] % 2:
        raise N.DimensionError(N.ERR_DIMENSION, "narrow_predictions: length must be even")
    out = np.zeros(x.shape[0])
    context().lls_predict(N.LAYOUT_REAL, 1, 1, x.shape[0], x.shape[1], x, w.reshape(1, -1), out)
    return out[0::2] + 1j * out[1::2]


# ------------------------------------------------------------ hybrid_nn
def plan_layout(dims):
    """Offsets of the FusedPlan buffer (fused_inference.cpp:19-42)."""
    pad = [((d + 7) // 8) * 8 for d in dims]
    off = pad[0]
    layers = []
    for l in range(1, len(dims)):
        w = off
        off += dims[l] * pad[l - 1]
        b = off
        off += pad[l]
        layers.append((w, b))
    return pad, layers, off, off + pad[-1]


@dataclass
class HybridNet:
    """HybridNetParams held as the device FP32 FusedPlan buffer plus FP64 w0."""
    dims: list
    plan: np.ndarray                       # float32 [plan_size]
    w0: np.ndarray = field(repr=False)     # float64 [dims[0]]

    def unpack(self):
        """-> ([(W_l, b_l)], final) as float64 views of the plan."""
        pad, layers, f, _ = plan_layout(self.dims)
        out = []
        for l, (wo, bo) in enumerate(layers, start=1):
            W = self.plan[wo:wo + self.dims[l] * pad[l - 1]].reshape(self.dims[l], pad[l - 1])
            out.append((W[:, :self.dims[l - 1]].astype(np.float64),
                        self.plan[bo:bo + self.dims[l]].astype(np.float64)))
        return out, self.plan[f:f + self.dims[-1]].astype(np.float64)

    def trainable_count(self):
        return N.param_count(self.dims)


def init_params(dims, w0: np.ndarray, seed: int) -> HybridNet:
    """hybrid_nn::init_params with Rng(seed) on device (hybrid_nn.cpp:34-55)."""
    dims = [int(d) for d in dims]
    w0 = np.ascontiguousarray(w0, dtype=np.float64)
    if not dims or dims[0] != w0.size or min(dims) < 1:
        raise N.DimensionError(N.ERR_DIMENSION, "init_params: dims[0] must equal the w0 length")
    plans = np.zeros((1, N.plan_size(dims)), dtype=np.float32)
    context().init_params(dims, np.array([seed], dtype=np.uint64), w0.reshape(1, -1), plans)
    return HybridNet(dims, plans[0], w0.copy())


def init_params_state(dims, w0: np.ndarray, state):
    """init_params(dims, w0, Rng&) with an explicit xoshiro256++ state
    (4 x u64): returns (HybridNet, flat FP64 theta, advanced state)."""
    dims = [int(d) for d in dims]
    w0 = np.ascontiguousarray(w0, dtype=np.float64)
    st = np.array([list(state)], dtype=np.uint64)
    plans = np.zeros((1, N.plan_size(dims)), dtype=np.float32)
    theta = np.zeros((1, N.param_count(dims)))
    context().init_params_state(dims, st, w0.reshape(1, -1), plans, theta)
    return HybridNet(dims, plans[0], w0.copy()), theta[0], tuple(int(v) for v in st[0])


def net_from_params(dims, w0, layers, final) -> HybridNet:
    """Pack explicit (W_l, b_l), final into a plan (fused::build_plan)."""
    pad, lay, f, total = plan_layout(dims)
    plan = np.zeros(total, dtype=np.float32)
    plan[:dims[0]] = w0
    for l, ((W, b), (wo, bo)) in enumerate(zip(layers, lay), start=1):
        Wp = np.zeros((dims[l], pad[l - 1]), dtype=np.float32)
        Wp[:, :dims[l - 1]] = W
        plan[wo:wo + Wp.size] = Wp.ravel()
        plan[bo:bo + dims[l]] = b
    plan[f:f + dims[-1]] = final
    return HybridNet(list(dims), plan, np.asarray(w0, dtype=np.float64).copy())


def train(net: HybridNet, design: np.ndarray, targets: np.ndarray, epochs=50, batch_size=128,
          lr=0.005, shuffle_seed=0, widened_complex=False) -> np.ndarray:
    """hybrid_nn::train (hybrid_nn.cpp:158-195).  design: real [n, 2M] rows, or
    (widened_complex=True) the complex receive matrix [n/2, M] with complex
    targets [n/2] -- the widening is then applied on device at load time."""
    cfg = N.TrainCfg.of(epochs, batch_size, lr)
    if widened_complex:
        x = np.ascontiguousarray(design, dtype=np.complex128)
        y = np.ascontiguousarray(np.asarray(targets, dtype=np.complex128).reshape(-1, 1))
        rows, width, layout = 2 * x.shape[0], 2 * x.shape[1], N.LAYOUT_WIDEN
        xd, yd = x.view(np.float64), y.view(np.float64)
    else:
        xd = np.ascontiguousarray(design, dtype=np.float64)
        yd = np.ascontiguousarray(targets, dtype=np.float64)
        rows, width, layout = xd.shape[0], xd.shape[1], N.LAYOUT_REAL
        if yd.size != rows:
            raise N.DimensionError(N.ERR_DIMENSION, "train: targets length")
    if rows == 0:
        raise N.DimensionError(N.ERR_DIMENSION, "train: empty training set")
    trace = np.zeros(max(epochs, 0))
    plans = np.ascontiguousarray(net.plan.reshape(1, -1))
    context().train(layout, 1, 1, rows, width, xd, yd, net.dims, cfg,
                    np.ascontiguousarray(net.w0.reshape(1, -1)), plans,
                    np.array([shuffle_seed], dtype=np.uint64), trace if epochs > 0 else None)
    net.plan = plans[0]
    return trace


def train_f64(dims, w0, theta, design, targets, epochs=50, batch_size=128, lr=0.005,
              shuffle_seed=0, widened_complex=False):
    """FP64 parity mode of hybrid_nn::train: theta (reference flat order,
    W_1, b_1, ..., final) is trained in place on device; returns the trace."""
    cfg = N.TrainCfg.of(epochs, batch_size, lr)
    if widened_complex:
        x = np.ascontiguousarray(design, dtype=np.complex128)
        y = np.ascontiguousarray(np.asarray(targets, dtype=np.complex128).reshape(-1, 1))
        rows, width, layout = 2 * x.shape[0], 2 * x.shape[1], N.LAYOUT_WIDEN
        xd, yd = x.view(np.float64), y.view(np.float64)
    else:
        xd = np.ascontiguousarray(design, dtype=np.float64)
        yd = np.ascontiguousarray(targets, dtype=np.float64)
        rows, width, layout = xd.shape[0], xd.shape[1], N.LAYOUT_REAL
    th = np.ascontiguousarray(theta, dtype=np.float64).reshape(1, -1)
    trace = np.zeros(max(epochs, 0))
    context().train_f64(layout, 1, 1, rows, width, xd, yd, list(dims), cfg,
                        np.ascontiguousarray(w0, dtype=np.float64).reshape(1, -1), th,
                        np.array([shuffle_seed], dtype=np.uint64), trace if epochs > 0 else None)
    theta[...] = th[0]
    return trace


def fused_forward_f32(net: HybridNet, x: np.ndarray) -> np.ndarray:
    """fused::fused_forward_f32 (fused_inference.cpp:222-231): real rows [B, d0]."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    if x.shape[1] != net.dims[0]:
        raise N.DimensionError(N.ERR_DIMENSION, "fused_forward: input width does not match plan")
    out = np.zeros(x.shape[0], dtype=np.float32)
    context().detect(net.dims, N.LAYOUT_REAL, 1, 1, x.shape[0], x,
                     np.ascontiguousarray(net.plan.reshape(1, -1)), soft=out)
    return out


def detect(net: HybridNet, data_rx: np.ndarray, truth_symbols=None):
    """hybrid_nn::detect(net, widen_design(data_rx)) + hard decisions (+ bit
    errors vs truth).  Returns (soft complex64 [N], bits uint8 [N, 2], errors)."""
    x = np.ascontiguousarray(data_rx, dtype=np.complex64)
    nd = x.shape[0]
    soft = np.zeros(nd, dtype=np.complex64)
    codes = np.zeros(nd, dtype=np.uint8)
    errs = np.zeros(1, dtype=np.uint32)
    truth = None
    if truth_symbols is not None:
        truth = codes_of(truth_symbols).reshape(nd, 1)
    context().detect(net.dims, N.LAYOUT_WIDEN, 1, 1, nd, x.view(np.float32),
                     np.ascontiguousarray(net.plan.reshape(1, -1)), truth=truth,
                     soft=soft.view(np.float32), codes=codes,
                     bit_errors=errs if truth is not None else None)
    bits = np.stack([codes & 1, (codes >> 1) & 1], axis=1).astype(np.uint8)
    return soft, bits, (int(errs[0]) if truth is not None else None)


# ----------------------------------------------------------------- eval
def codes_of(sym: np.ndarray) -> np.ndarray:
    """2-bit QPSK code of hard_decision_qpsk (eval.cpp:38-45): bit0 | bit1 << 1."""
    sym = np.asarray(sym)
    return ((sym.real < 0).astype(np.uint8) | ((sym.imag < 0).astype(np.uint8) << 1))


# ------------------------------------------------------------- pipeline
@dataclass
class SlotBatch:
    w0: np.ndarray
    gram_condition: np.ndarray
    status: np.ndarray
    plans: np.ndarray
    trace: np.ndarray
    soft: np.ndarray
    codes: np.ndarray
    bit_errors: np.ndarray
    symbol_errors: np.ndarray = None


def pipeline(dims, pilot_rx, pilot_sym, data_rx, truth_codes, init_seeds, shuffle_seeds,
             epochs=50, batch_size=128, lr=0.005, precision=32) -> SlotBatch:
    """LLS -> init -> train -> detect for S slots x K users (one C-ABI call).
    precision=64: the reference's FP64 training (noma_pipeline_f64)."""
    px = np.ascontiguousarray(pilot_rx, dtype=np.complex128)
    py = np.ascontiguousarray(pilot_sym, dtype=np.complex128)
    dx = np.ascontiguousarray(data_rx, dtype=np.complex64)
    S, NT, M = px.shape
    K = py.shape[2]
    ND = dx.shape[1]
    nets = S * K
    ps = N.plan_size(dims)
    out = SlotBatch(np.zeros((S, K, 2 * M)), np.zeros((S, K)), np.zeros((S, K), np.int32),
                    np.zeros((S, K, ps), np.float32), np.zeros((S, K, max(epochs, 1))),
                    np.zeros((S, K, ND), np.complex64), np.zeros((S, K, ND), np.uint8),
                    np.zeros((S, K), np.uint32), np.zeros((S, K), np.uint32))
    cfg = N.TrainCfg.of(epochs, batch_size, lr)
    context().pipeline(dims, cfg, S, K, M, NT, ND, px.view(np.float64), py.view(np.float64),
                       dx.view(np.float32),
                       None if truth_codes is None else np.ascontiguousarray(truth_codes, np.uint8),
                       np.ascontiguousarray(init_seeds, np.uint64).reshape(nets),
                       np.ascontiguousarray(shuffle_seeds, np.uint64).reshape(nets),
                       out.status, w0=out.w0, cond=out.gram_condition, plans=out.plans,
                       trace=out.trace if epochs > 0 else None, soft=out.soft.view(np.float32),
                       codes=out.codes, bit_errors=out.bit_errors if truth_codes is not None else None,
                       symbol_errors=out.symbol_errors if truth_codes is not None else None,
                       precision=precision)
    out.trace = out.trace[..., :epochs]
    return out


@dataclass
class Synth:
    pilot_rx: np.ndarray
    pilot_sym: np.ndarray
    data_rx: np.ndarray
    data_codes: np.ndarray
    channel: np.ndarray
    noise_power: np.ndarray


def synthesize(num_users, num_antennas, train_symbols, data_symbols, seeds, power_step_db=3.0,
               snr_db=float("inf"), rx_nonlinearity_gain=0.0) -> Synth:
    """synthesize(cfg, SeedBundle::from_master(seed)) for each seed, on device."""
    K, M, NT, ND = num_users, num_antennas, train_symbols, data_symbols
    seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
    S = seeds.size
    sc = N.Scenario(K, M, NT, ND, power_step_db, snr_db, rx_nonlinearity_gain)
    out = Synth(np.zeros((S, NT, M), np.complex128), np.zeros((S, NT, K), np.complex128),
                np.zeros((S, ND, M), np.complex64), np.zeros((S, ND, K), np.uint8),
                np.zeros((S, M, K), np.complex128), np.zeros(S))
    context().synthesize(sc, seeds, out.pilot_rx.view(np.float64), out.pilot_sym.view(np.float64),
                         out.data_rx.view(np.float32), out.data_codes, out.channel.view(np.float64),
                         out.noise_power)
    return out


# -------------------------------------------------------------- bench rows
def bench_rows(net: HybridNet, batch: int, repeats: int = 20, naive_ns_per_sample=None) -> str:
    """GPU rows for the `noma bench` CSV (fused_inference.cpp:282-338, schema
    path,dims,batch,ns_per_sample,speedup_vs_naive): the device forward over
    `batch` rows of the plan, timed with CUDA events (median of `repeats`,
    like time_median_ns), for the FP32 FFMA kernel ("gpu_ffma") and, when the
    shape is on the tensor-core path, the tcgen05 3xTF32 kernel
    ("gpu_tcgen05").  Inputs are widened complex rows (batch/2 symbols), the
    data-phase layout; the rows are gated against the plan's FP64 forward at
    the reference FP32 tolerance (test_fused.cpp:128-130) before any timing
    is reported, as bench_compare gates its paths (:291-301).  The speedup
    column is filled when the caller supplies the CPU naive ns/sample."""
    import os

    import torch

    dims = list(net.dims)
    if batch < 2 or batch % 2 or repeats < 1:
        raise N.DimensionError(N.ERR_DIMENSION, "bench_rows: batch must be even >= 2, repeats >= 1")
    if dims[0] % 2:
        raise N.UnsupportedError(N.ERR_UNSUPPORTED, "bench_rows: widened input width must be even")
    rng = np.random.default_rng(0x9E24A)
    nsym, M = batch // 2, dims[0] // 2
    x = (rng.normal(size=(nsym, M)) + 1j * rng.normal(size=(nsym, M))).astype(np.complex64)
    # FP64 forward of the plan (the gate)
    layers, final = net.unpack()
    wd = np.empty((batch, dims[0]))
    xr, xi = x.real.astype(np.float64), x.imag.astype(np.float64)
    wd[0::2, :M], wd[0::2, M:], wd[1::2, :M], wd[1::2, M:] = xr, xi, xi, -xr
    a = wd
    for W, b in layers:
        a = np.maximum(a @ W.T + b, 0.0)
    ref = wd @ net.plan[:dims[0]].astype(np.float64) + a @ final
    ref_c = ref[0::2] + 1j * ref[1::2]
    dev = torch.device("cuda", 0)
    ctx = context()
    dx = torch.from_numpy(x.view(np.float32).copy()).to(dev)
    plan = torch.from_numpy(np.ascontiguousarray(net.plan.reshape(1, -1))).to(dev)
    soft = torch.empty((nsym, 2), dtype=torch.float32, device=dev)
    rows = []
    old = os.environ.get("NOMA_DETECT_TC")
    try:
        for path, env in (("gpu_tcgen05", None), ("gpu_ffma", "0")):
            if env is None:
                os.environ.pop("NOMA_DETECT_TC", None)
            else:
                os.environ["NOMA_DETECT_TC"] = env
            ctx.detect(dims, N.LAYOUT_WIDEN, 1, 1, nsym, dx, plan, soft=soft)
            torch.cuda.synchronize()
            if path == "gpu_tcgen05" and ctx.detect_mode != 2:
                continue
            got = soft.cpu().numpy().view(np.complex64).ravel()
            scale = max(1.0, float(np.max(np.abs(ref_c))))
            if np.max(np.abs(got - ref_c)) / scale > 1e-5:
                raise RuntimeError("bench_rows: device path disagrees with the FP64 forward")
            ns = []
            for _ in range(repeats):
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
                ctx.detect(dims, N.LAYOUT_WIDEN, 1, 1, nsym, dx, plan, soft=soft)
                e1.record()
                e1.synchronize()
                ns.append(e0.elapsed_time(e1) * 1e6)
            per = sorted(ns)[len(ns) // 2] / batch
            sp = "" if naive_ns_per_sample is None else repr(naive_ns_per_sample / per)
            rows.append(f"{path},{'x'.join(str(d) for d in dims)},{batch},{per!r},{sp}")
    finally:
        if old is None:
            os.environ.pop("NOMA_DETECT_TC", None)
        else:
            os.environ["NOMA_DETECT_TC"] = old
    return "\n".join(rows) + "\n"
