"""One pipeline step on synthetic device-resident slots, for ncu captures.

  python tools/profile_step.py [--config c2] [--slots 148] [--steps 1]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2206_05998_b200 import native as N  # noqa: E402
from paper_2206_05998_b200.seeds import slot_user_seeds  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--slots", type=int, default=0)
ap.add_argument("--steps", type=int, default=1)
args = ap.parse_args()
cfg = dict(bench.CONFIGS[args.config])
S = args.slots or cfg["slots"]
M, K = cfg["M"], cfg["K"]
NT, ND = bench.NT, bench.ND
dims = [2 * M] + cfg["hidden"]
dev = torch.device("cuda", 0)
ctx = N.Context(0)
_stream = torch.cuda.Stream()
torch.cuda.set_stream(_stream)
ctx.set_stream(_stream.cuda_stream)
seeds = np.arange(1000, 1000 + S, dtype=np.uint64)
px = torch.empty((S, NT, M, 2), dtype=torch.float64, device=dev)
py = torch.empty((S, NT, K, 2), dtype=torch.float64, device=dev)
dx = torch.empty((S, ND, M, 2), dtype=torch.float32, device=dev)
truth = torch.empty((S, ND, K), dtype=torch.uint8, device=dev)
ctx.synthesize(N.Scenario(K, M, NT, ND, cfg["step"], bench.SNR, bench.GAIN),
               torch.from_numpy(seeds.astype(np.int64)).to(dev), px, py, dx, truth)
i_s, s_s = slot_user_seeds(seeds, K)
status = torch.empty((S, K), dtype=torch.int32, device=dev)
errs = torch.empty((S, K), dtype=torch.int32, device=dev)
codes = torch.empty((S, K, ND), dtype=torch.uint8, device=dev)
for _ in range(args.steps):
    ctx.pipeline(dims, N.TrainCfg.of(bench.EPOCHS, bench.BATCH, bench.LR), S, K, M, NT, ND, px, py,
                 dx, truth, torch.from_numpy(i_s.astype(np.int64)).to(dev),
                 torch.from_numpy(s_s.astype(np.int64)).to(dev), status, codes=codes,
                 bit_errors=errs)
torch.cuda.synchronize()
print("ok", int((status != 0).sum()), int(errs.sum()))
