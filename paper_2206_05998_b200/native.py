"""ctypes binding of the C-ABI in include/noma_cuda.h (libnoma_b200.so).

This is plumbing: it moves numpy (host, NOMA_MEM_HOST) or torch CUDA tensors
(device, NOMA_MEM_DEVICE) into the C-ABI.  There is no CPU fallback: if the
CUDA library is missing or no device is present, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libnoma_b200.so")

OK, ERR_DIMENSION, ERR_CONFIG, ERR_ILL, ERR_UNSUPPORTED, ERR_CUDA, ERR_ARGUMENT = range(7)
MEM_HOST, MEM_DEVICE = 0, 1
LAYOUT_WIDEN, LAYOUT_REAL = 0, 1
MAX_DIMS = 9

EXPORTED = [
    "noma_version", "noma_ctx_create", "noma_ctx_destroy", "noma_ctx_last_error",
    "noma_ctx_set_stream", "noma_ctx_synchronize", "noma_ctx_kernel_launches",
    "noma_plan_size", "noma_param_count", "noma_lls_fit", "noma_init_params", "noma_train",
    "noma_detect", "noma_pipeline", "noma_synthesize", "noma_ctx_set_profiling",
    "noma_ctx_phase_ms", "noma_measure_fp32_tflops", "noma_host_alloc", "noma_host_free", "noma_init_params_state",
    "noma_lls_predict", "noma_train_f64", "noma_ctx_train_mode", "noma_ctx_detect_mode", "noma_synthesize_bundles",
    "noma_ctx_pipeline_chunks", "noma_forward_f64", "noma_forward_f32", "noma_loss_and_grad", "noma_adam_step",
    "noma_bench_forward_f64", "noma_synthesize_f64", "noma_pipeline_f64",
]
PHASES = ("lls", "init", "shuffle", "train", "detect", "total")


class NomaError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"noma status {code}: {msg}")
        self.code = code


class DimensionError(NomaError):
    pass


class ConfigError(NomaError):
    pass


class IllConditionedError(NomaError):
    def __init__(self, code, msg, gram_condition=None):
        super().__init__(code, msg)
        self.gram_condition = gram_condition


class UnsupportedError(NomaError):
    pass


_ERRS = {ERR_DIMENSION: DimensionError, ERR_CONFIG: ConfigError, ERR_UNSUPPORTED: UnsupportedError}


class NetDesc(C.Structure):
    _fields_ = [("ndims", C.c_int), ("dims", C.c_int * MAX_DIMS)]

    @classmethod
    def of(cls, dims):
        d = cls()
        d.ndims = len(dims)
        for i, v in enumerate(dims):
            d.dims[i] = int(v)
        return d


class TrainCfg(C.Structure):
    _fields_ = [("epochs", C.c_int), ("batch_size", C.c_int), ("lr", C.c_double),
                ("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double)]

    @classmethod
    def of(cls, epochs=50, batch_size=128, lr=0.005, beta1=0.9, beta2=0.999, eps=1e-8):
        return cls(epochs, batch_size, lr, beta1, beta2, eps)


class Dataset(C.Structure):
    _fields_ = [("layout", C.c_int), ("n_designs", C.c_int), ("nets_per_design", C.c_int),
                ("rows", C.c_int), ("width", C.c_int), ("design", C.c_void_p),
                ("targets", C.c_void_p)]


class Scenario(C.Structure):
    _fields_ = [("num_users", C.c_int), ("num_antennas", C.c_int), ("train_symbols", C.c_int),
                ("data_symbols", C.c_int), ("power_step_db", C.c_double), ("snr_db", C.c_double),
                ("rx_nonlinearity_gain", C.c_double)]


_lib = None


def load():
    """Load libnoma_b200.so; raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} missing: run __graft_entry__.build() "
                           "(the CUDA extension is required; there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, ip = C.c_void_p, C.c_int
    L.noma_version.restype = ip
    L.noma_ctx_create.argtypes = [ip, C.POINTER(vp)]
    L.noma_ctx_destroy.argtypes = [vp]
    L.noma_ctx_last_error.restype = C.c_char_p
    L.noma_ctx_last_error.argtypes = [vp]
    L.noma_ctx_set_stream.argtypes = [vp, vp]
    L.noma_ctx_synchronize.argtypes = [vp]
    L.noma_ctx_kernel_launches.restype = C.c_longlong
    L.noma_ctx_kernel_launches.argtypes = [vp]
    L.noma_ctx_train_mode.argtypes = [vp]
    L.noma_ctx_detect_mode.argtypes = [vp]
    L.noma_ctx_pipeline_chunks.argtypes = [vp]
    L.noma_plan_size.argtypes = [C.POINTER(NetDesc)]
    L.noma_param_count.argtypes = [C.POINTER(NetDesc)]
    L.noma_lls_fit.argtypes = [vp, C.POINTER(Dataset), vp, vp, vp, ip]
    L.noma_init_params.argtypes = [vp, C.POINTER(NetDesc), ip, vp, vp, vp, ip]
    L.noma_train.argtypes = [vp, C.POINTER(Dataset), C.POINTER(NetDesc), C.POINTER(TrainCfg),
                             vp, vp, vp, vp, vp, ip]
    L.noma_detect.argtypes = [vp, C.POINTER(NetDesc), ip, ip, ip, ip, vp, vp, vp, vp, vp, vp, vp, ip]
    L.noma_pipeline.argtypes = [vp, C.POINTER(NetDesc), C.POINTER(TrainCfg), ip, ip, ip, ip, ip,
                                vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, ip]
    L.noma_pipeline_f64.argtypes = L.noma_pipeline.argtypes
    L.noma_synthesize.argtypes = [vp, C.POINTER(Scenario), ip, vp, vp, vp, vp, vp, vp, vp, ip]
    L.noma_synthesize_bundles.argtypes = [vp, C.POINTER(Scenario), ip, vp, vp, vp, vp, vp, vp, vp, ip]
    L.noma_ctx_set_profiling.argtypes = [vp, ip]
    L.noma_ctx_phase_ms.argtypes = [vp, C.POINTER(C.c_double)]
    L.noma_measure_fp32_tflops.argtypes = [vp, ip, C.POINTER(C.c_double)]
    L.noma_host_alloc.argtypes = [C.c_size_t, C.POINTER(vp)]
    L.noma_host_free.argtypes = [vp]
    L.noma_init_params_state.argtypes = [vp, C.POINTER(NetDesc), ip, vp, vp, vp, vp, ip]
    L.noma_lls_predict.argtypes = [vp, ip, ip, ip, ip, ip, vp, vp, vp, ip]
    L.noma_train_f64.argtypes = [vp, C.POINTER(Dataset), C.POINTER(NetDesc), C.POINTER(TrainCfg),
                                 vp, vp, vp, vp, vp, ip]
    _lib = L
    return L


def plan_size(dims) -> int:
    d = NetDesc.of(dims)
    return load().noma_plan_size(C.byref(d))


def param_count(dims) -> int:
    d = NetDesc.of(dims)
    return load().noma_param_count(C.byref(d))


def _ptr(a):
    """Pointer of a numpy array (host) or a torch tensor (device); None -> NULL."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        assert a.flags.c_contiguous
        return a.ctypes.data
    # torch tensor
    assert a.is_contiguous()
    return a.data_ptr()


def pinned_empty(shape, dtype) -> np.ndarray:
    """numpy array in page-locked host memory (noma_host_alloc), freed with
    the array: the host buffers of NOMA_MEM_HOST calls whose chunked copies
    should overlap the device work."""
    import weakref

    dtype = np.dtype(dtype)
    nbytes = int(np.prod(shape)) * dtype.itemsize
    ptr = C.c_void_p()
    st = load().noma_host_alloc(max(nbytes, 1), C.byref(ptr))
    if st != OK:
        raise NomaError(st, f"noma_host_alloc({nbytes}) failed")
    raw = (C.c_uint8 * max(nbytes, 1)).from_address(ptr.value)
    base = np.frombuffer(raw, dtype=np.uint8, count=nbytes)
    arr = base.view(dtype).reshape(shape)
    weakref.finalize(raw, load().noma_host_free, ptr)
    return arr


def _mem_of(*arrays):
    kinds = {isinstance(a, np.ndarray) for a in arrays if a is not None}
    if kinds == {True}:
        return MEM_HOST
    if kinds == {False}:
        return MEM_DEVICE
    raise TypeError("mix of host (numpy) and device (torch) arrays")


class Context:
    """One per GPU (noma_ctx_create); optionally bound to a torch stream."""

    def __init__(self, device: int = 0):
        self.L = load()
        self.h = C.c_void_p()
        st = self.L.noma_ctx_create(device, C.byref(self.h))
        if st != OK:
            raise NomaError(st, f"noma_ctx_create({device}) failed (no CUDA device?)")
        self.device = device

    def close(self):
        if self.h:
            self.L.noma_ctx_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_ptr):
        self.L.noma_ctx_set_stream(self.h, C.c_void_p(stream_ptr) if stream_ptr else None)

    def use_torch_stream(self):
        """Bind to torch's current stream (must not be the legacy default
        stream, whose handle 0 means 'the context's own stream' here)."""
        import torch
        s = torch.cuda.current_stream(self.device).cuda_stream
        if not s:
            raise ValueError("torch's current stream is the legacy default stream; "
                             "set a torch.cuda.Stream first")
        self.set_stream(s)

    def synchronize(self):
        self._check(self.L.noma_ctx_synchronize(self.h))

    @property
    def pipeline_chunks(self) -> int:
        """Slot chunks of the last pipeline call (noma_ctx_pipeline_chunks)."""
        return self.L.noma_ctx_pipeline_chunks(self.h)

    @property
    def kernel_launches(self) -> int:
        return self.L.noma_ctx_kernel_launches(self.h)

    @property
    def train_mode(self) -> int:
        """Kernel shape of the last training launch (noma_ctx_train_mode)."""
        return self.L.noma_ctx_train_mode(self.h)

    @property
    def detect_mode(self) -> int:
        """Kernel of the last detection (noma_ctx_detect_mode): 1 FFMA, 2 tcgen05."""
        return self.L.noma_ctx_detect_mode(self.h)

    def set_profiling(self, on: bool):
        self._check(self.L.noma_ctx_set_profiling(self.h, 1 if on else 0))

    def phase_ms(self) -> dict:
        out = (C.c_double * 6)()
        self._check(self.L.noma_ctx_phase_ms(self.h, out))
        return dict(zip(PHASES, list(out)))

    def measure_fp32_tflops(self, form: int = 0) -> float:
        """form 0: constant-operand FFMA peak; 1: 8x4 register outer product."""
        v = C.c_double(0)
        self._check(self.L.noma_measure_fp32_tflops(self.h, form, C.byref(v)))
        return v.value

    def last_error(self) -> str:
        return self.L.noma_ctx_last_error(self.h).decode()

    def _check(self, st, ill_cond=None):
        if st == OK:
            return
        msg = self.last_error()
        if st == ERR_ILL:
            raise IllConditionedError(st, msg, ill_cond)
        raise _ERRS.get(st, NomaError)(st, msg)

    # ------------------------------------------------------------ entries
    def lls_fit(self, layout, n_designs, K, rows, width, design, targets, w0, cond, status):
        mem = _mem_of(design, targets, w0)
        ds = Dataset(layout, n_designs, K, rows, width, _ptr(design), _ptr(targets))
        st = self.L.noma_lls_fit(self.h, C.byref(ds), _ptr(w0), _ptr(cond), _ptr(status), mem)
        if st == ERR_ILL:
            raise IllConditionedError(st, self.last_error(),
                                      float(cond.ravel()[np.argmax(status.ravel() != 0)])
                                      if cond is not None and status is not None else None)
        self._check(st)

    def init_params(self, dims, seeds, w0, plans):
        mem = _mem_of(seeds, plans)
        d = NetDesc.of(dims)
        n = seeds.shape[0]
        self._check(self.L.noma_init_params(self.h, C.byref(d), n, _ptr(seeds), _ptr(w0),
                                            _ptr(plans), mem))

    def init_params_state(self, dims, states, w0, plans=None, theta=None):
        mem = _mem_of(states, w0, plans, theta)
        d = NetDesc.of(dims)
        self._check(self.L.noma_init_params_state(self.h, C.byref(d), states.shape[0],
                                                  _ptr(states), _ptr(w0), _ptr(plans),
                                                  _ptr(theta), mem))

    def lls_predict(self, layout, n_designs, K, rows, width, data, w0, out):
        mem = _mem_of(data, w0, out)
        self._check(self.L.noma_lls_predict(self.h, layout, n_designs, K, rows, width,
                                            _ptr(data), _ptr(w0), _ptr(out), mem))

    def train(self, layout, n_designs, K, rows, width, design, targets, dims, cfg: TrainCfg, w0,
              plans, shuffle_seeds, trace=None, status=None):
        mem = _mem_of(design, targets, w0, plans, shuffle_seeds)
        ds = Dataset(layout, n_designs, K, rows, width, _ptr(design), _ptr(targets))
        d = NetDesc.of(dims)
        self._check(self.L.noma_train(self.h, C.byref(ds), C.byref(d), C.byref(cfg), _ptr(w0),
                                      _ptr(plans), _ptr(shuffle_seeds), _ptr(trace),
                                      _ptr(status), mem))

    def train_f64(self, layout, n_designs, K, rows, width, design, targets, dims, cfg: TrainCfg,
                  w0, theta, shuffle_seeds, trace=None, status=None):
        mem = _mem_of(design, targets, w0, theta, shuffle_seeds)
        ds = Dataset(layout, n_designs, K, rows, width, _ptr(design), _ptr(targets))
        d = NetDesc.of(dims)
        self._check(self.L.noma_train_f64(self.h, C.byref(ds), C.byref(d), C.byref(cfg), _ptr(w0),
                                          _ptr(theta), _ptr(shuffle_seeds), _ptr(trace),
                                          _ptr(status), mem))

    def detect(self, dims, layout, n_designs, K, rows, data, plans, truth=None, soft=None,
               codes=None, bit_errors=None, symbol_errors=None):
        mem = _mem_of(data, plans)
        d = NetDesc.of(dims)
        self._check(self.L.noma_detect(self.h, C.byref(d), layout, n_designs, K, rows,
                                       _ptr(data), _ptr(plans), _ptr(truth), _ptr(soft),
                                       _ptr(codes), _ptr(bit_errors), _ptr(symbol_errors), mem))

    def pipeline(self, dims, cfg: TrainCfg, S, K, M, NT, ND, pilot_rx, pilot_sym, data_rx, truth,
                 init_seeds, shuffle_seeds, status, w0=None, cond=None, plans=None, trace=None,
                 soft=None, codes=None, bit_errors=None, symbol_errors=None, precision=32):
        mem = _mem_of(pilot_rx, pilot_sym, data_rx, status)
        d = NetDesc.of(dims)
        fn = self.L.noma_pipeline_f64 if precision == 64 else self.L.noma_pipeline
        self._check(fn(
            self.h, C.byref(d), C.byref(cfg), S, K, M, NT, ND, _ptr(pilot_rx), _ptr(pilot_sym),
            _ptr(data_rx), _ptr(truth), _ptr(init_seeds), _ptr(shuffle_seeds), _ptr(w0),
            _ptr(cond), _ptr(plans), _ptr(trace), _ptr(soft), _ptr(codes), _ptr(bit_errors),
            _ptr(symbol_errors), _ptr(status), mem))

    def synthesize_bundles(self, sc: Scenario, bundles, pilot_rx=None, pilot_sym=None, data_rx=None,
                           data_codes=None, channel=None, noise_power=None):
        """synthesize(cfg, SeedBundle{symbols, channel, noise}) per row of bundles [S, 3]."""
        mem = _mem_of(bundles, pilot_rx, pilot_sym, data_rx, data_codes, channel, noise_power)
        S = bundles.shape[0]
        self._check(self.L.noma_synthesize_bundles(self.h, C.byref(sc), S, _ptr(bundles), _ptr(pilot_rx),
                                                   _ptr(pilot_sym), _ptr(data_rx), _ptr(data_codes),
                                                   _ptr(channel), _ptr(noise_power), mem))

    def synthesize(self, sc: Scenario, seeds, pilot_rx=None, pilot_sym=None, data_rx=None,
                   data_codes=None, channel=None, noise_power=None):
        mem = _mem_of(seeds, pilot_rx, pilot_sym, data_rx, data_codes, channel, noise_power)
        S = seeds.shape[0]
        self._check(self.L.noma_synthesize(self.h, C.byref(sc), S, _ptr(seeds), _ptr(pilot_rx),
                                           _ptr(pilot_sym), _ptr(data_rx), _ptr(data_codes),
                                           _ptr(channel), _ptr(noise_power), mem))
