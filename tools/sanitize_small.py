"""Small invocations of every device kernel for compute-sanitizer runs:
LLS, init, shuffles, synthesis, the throughput and latency training kernels,
FFMA and tcgen05 detection (one slot, short training)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_05998_b200 import api  # noqa: E402
from paper_2206_05998_b200.seeds import slot_user_seeds  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "all"
sy = api.synthesize(3, 16, 100, 256, [5], snr_db=15.0, rx_nonlinearity_gain=0.05)
init, shuf = slot_user_seeds(np.array([5], np.uint64), 3)
for hidden in ([64], [64, 64]):
    if mode in ("all", "lat"):  # latency cluster kernel (default for few nets)
        out = api.pipeline([32] + hidden, sy.pilot_rx, sy.pilot_sym, sy.data_rx, sy.data_codes,
                           init, shuf, epochs=2)
        print("lat", hidden, api.context().train_mode, api.context().detect_mode, out.bit_errors.ravel())
    if mode in ("all", "tc"):  # throughput kernel + tcgen05 detect
        os.environ["NOMA_LAT_CLUSTER"] = "1"
        out = api.pipeline([32] + hidden, sy.pilot_rx, sy.pilot_sym, sy.data_rx, sy.data_codes,
                           init, shuf, epochs=2)
        print("tc", hidden, api.context().train_mode, api.context().detect_mode, out.bit_errors.ravel())
        os.environ.pop("NOMA_LAT_CLUSTER")
    if mode in ("all", "thr"):  # throughput kernel + FFMA detect
        os.environ["NOMA_LAT_CLUSTER"] = "1"
        os.environ["NOMA_DETECT_TC"] = "0"
        out = api.pipeline([32] + hidden, sy.pilot_rx, sy.pilot_sym, sy.data_rx, sy.data_codes,
                           init, shuf, epochs=2)
        print("thr", hidden, api.context().train_mode, api.context().detect_mode, out.bit_errors.ravel())
        os.environ.pop("NOMA_LAT_CLUSTER")
        os.environ.pop("NOMA_DETECT_TC")
if mode in ("all", "tcmulti"):  # detection CTAs spanning several nets (persistent grid)
    from paper_2206_05998_b200 import native as N
    from tests.helpers import random_net_fused

    for dims in ([32, 64, 64], [64, 64]):
        nd, K, rows = 2, 3, 8000  # 125 tiles per net, 750 over 148 CTAs
        nets = [api.net_from_params(o.dims, o.w0, *o.layers())
                for o in (random_net_fused(dims, 300 + i) for i in range(nd * K))]
        plans = np.ascontiguousarray(np.stack([n.plan.reshape(-1) for n in nets]))
        rng = np.random.default_rng(3)
        x = (rng.normal(size=(nd, rows, dims[0] // 2))
             + 1j * rng.normal(size=(nd, rows, dims[0] // 2))).astype(np.complex64)
        truth = rng.integers(0, 4, size=(nd, rows, K), dtype=np.uint8)
        codes = np.zeros((nd * K, rows), np.uint8)
        errs = np.zeros(nd * K, np.uint32)
        api.context().detect(dims, N.LAYOUT_WIDEN, nd, K, rows, x.view(np.float32), plans, truth=truth,
                             codes=codes, bit_errors=errs)
        print("tcmulti", dims, api.context().detect_mode, errs)
if mode in ("all", "w4"):  # the 4-warp throughput kernel (one hidden layer of 64, many nets)
    sy8 = api.synthesize(6, 16, 100, 256, [5, 6, 7, 8, 9, 10, 11, 12], snr_db=15.0, rx_nonlinearity_gain=0.05)
    i8, s8 = slot_user_seeds(np.arange(5, 13, dtype=np.uint64), 6)
    os.environ["NOMA_LAT_CLUSTER"] = "1"
    out = api.pipeline([32, 64], sy8.pilot_rx, sy8.pilot_sym, sy8.data_rx, sy8.data_codes, i8, s8, epochs=2)
    print("w4", api.context().train_mode, api.context().detect_mode, out.bit_errors.ravel()[:6])
    os.environ.pop("NOMA_LAT_CLUSTER")
if mode in ("all", "l2"):  # the two-hidden-layer 8-warp kernel (train mode 5), 8 slots x 6 users
    sy8 = api.synthesize(6, 16, 100, 256, [5, 6, 7, 8, 9, 10, 11, 12], snr_db=15.0, rx_nonlinearity_gain=0.05)
    i8, s8 = slot_user_seeds(np.arange(5, 13, dtype=np.uint64), 6)
    os.environ["NOMA_LAT_CLUSTER"] = "1"
    out = api.pipeline([32, 64, 64], sy8.pilot_rx, sy8.pilot_sym, sy8.data_rx, sy8.data_codes, i8, s8, epochs=2)
    print("l2", api.context().train_mode, api.context().detect_mode, out.bit_errors.ravel()[:6])
    os.environ.pop("NOMA_LAT_CLUSTER")
if mode in ("all", "w8"):  # the 8-warp kernel on a 128-wide input (train mode 4), 2 slots x 8 users
    sy2 = api.synthesize(8, 64, 130, 256, [5, 6], snr_db=15.0, rx_nonlinearity_gain=0.05)
    i2, s2 = slot_user_seeds(np.arange(5, 7, dtype=np.uint64), 8)
    os.environ["NOMA_LAT_CLUSTER"] = "1"
    out = api.pipeline([128, 64], sy2.pilot_rx, sy2.pilot_sym, sy2.data_rx, sy2.data_codes, i2, s2, epochs=2)
    print("w8", api.context().train_mode, api.context().detect_mode, out.bit_errors.ravel()[:6])
    os.environ.pop("NOMA_LAT_CLUSTER")
if mode in ("all", "generic"):  # shape-general training / detection, FP64 pipeline mode
    out = api.pipeline([32, 160], sy.pilot_rx, sy.pilot_sym, sy.data_rx, sy.data_codes, init, shuf, epochs=2)
    print("generic", api.context().train_mode, api.context().detect_mode, out.bit_errors.ravel())
    out = api.pipeline([32, 64], sy.pilot_rx, sy.pilot_sym, sy.data_rx, sy.data_codes, init, shuf, epochs=2,
                       precision=64)
    print("f64", api.context().train_mode, api.context().detect_mode, out.bit_errors.ravel())
if mode in ("all", "dense"):  # the C++ API's FP64 entry points (k_dense.cu)
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for t in ("fused", "hybrid_nn"):
        r = subprocess.run([os.path.join(root, "oracle", "_ref", "reftests", "test_" + t)], capture_output=True,
                           text=True)
        print("dense", t, r.returncode, r.stdout.strip().splitlines()[-1] if r.stdout else "")
print("done")
