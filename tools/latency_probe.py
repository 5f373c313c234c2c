"""Single-slot (S=1) latency breakdown of the pipeline: per-phase device ms
(CUDA events recorded by the C-ABI) and, with NOMA_PHASE_CLOCKS in a
NOMA_BUILD_TRACE=1 build (the cycle probes are compiled out otherwise), the train
kernel's per-phase cycles for net 0, for each training-cluster shape.

  python tools/latency_probe.py [--configs c1,c2] [--clusters 1,2,4]
"""
import argparse
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2206_05998_b200 import native as N  # noqa: E402
from paper_2206_05998_b200.seeds import slot_user_seeds  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="c1,c2")
ap.add_argument("--clusters", default="1,2,4")
ap.add_argument("--reps", type=int, default=6)
ap.add_argument("--lat", default="", help="NOMA_LAT_CLUSTER values to sweep (latency kernel)")
args = ap.parse_args()
dev = torch.device("cuda", 0)
ctx = N.Context(0)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx.set_stream(stream.cuda_stream)
for tag in args.configs.split(","):
    cfg = dict(bench.CONFIGS[tag])
    M, K, NT, ND = cfg["M"], cfg["K"], bench.NT, bench.ND
    dims = [2 * M] + cfg["hidden"]
    seeds = np.array([1000], dtype=np.uint64)
    px = torch.empty((1, NT, M, 2), dtype=torch.float64, device=dev)
    py = torch.empty((1, NT, K, 2), dtype=torch.float64, device=dev)
    dx = torch.empty((1, ND, M, 2), dtype=torch.float32, device=dev)
    truth = torch.empty((1, ND, K), dtype=torch.uint8, device=dev)
    ctx.synthesize(N.Scenario(K, M, NT, ND, cfg["step"], bench.SNR, bench.GAIN),
                   torch.from_numpy(seeds.astype(np.int64)).to(dev), px, py, dx, truth)
    i_s, s_s = slot_user_seeds(seeds, K)
    i_d = torch.from_numpy(i_s.astype(np.int64)).to(dev)
    s_d = torch.from_numpy(s_s.astype(np.int64)).to(dev)
    status = torch.empty((1, K), dtype=torch.int32, device=dev)
    errs = torch.empty((1, K), dtype=torch.int32, device=dev)
    codes = torch.empty((1, K, ND), dtype=torch.uint8, device=dev)
    tcfg = N.TrainCfg.of(bench.EPOCHS, bench.BATCH, bench.LR)
    sweep = [("lat", v) for v in args.lat.split(",") if v] or [("row", v) for v in args.clusters.split(",")]
    for kind, cs in sweep:
        os.environ.pop("NOMA_LAT_CLUSTER", None)
        if kind == "lat":
            os.environ["NOMA_LAT_CLUSTER"] = cs
        else:
            os.environ["NOMA_TRAIN_CLUSTER"] = cs
        os.environ.pop("NOMA_PHASE_CLOCKS", None)
        tot, ph = [], []
        ctx.set_profiling(True)
        for i in range(args.reps):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            ctx.pipeline(dims, tcfg, 1, K, M, NT, ND, px, py, dx, truth, i_d, s_d, status,
                         codes=codes, bit_errors=errs)
            b.record(stream)
            b.synchronize()
            if i >= 2:
                tot.append(a.elapsed_time(b) * 1e3)
                ph.append(ctx.phase_ms())
        ctx.set_profiling(False)
        os.environ["NOMA_PHASE_CLOCKS"] = "1"
        ctx.pipeline(dims, tcfg, 1, K, M, NT, ND, px, py, dx, truth, i_d, s_d, status,
                     codes=codes, bit_errors=errs)
        torch.cuda.synchronize()
        os.environ.pop("NOMA_PHASE_CLOCKS", None)
        print(json.dumps({"config": tag, "cluster": f"{kind}{cs}", "train_mode": ctx.train_mode, "latency_us": statistics.median(tot),
                          "phase_us": {k: round(1e3 * statistics.median(p[k] for p in ph), 1)
                                       for k in ph[0]},
                          "bit_errors": errs.cpu().tolist()}), flush=True)
