"""Is the single-slot latency host-bound?  Times the C1 pipeline call with the
stream idle at the first event (as bench.py does) and with the host given a
head start (a 2 ms device sleep queued before the first event), and reports
the host-side duration of the call."""
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2206_05998_b200 import native as N  # noqa: E402
from paper_2206_05998_b200.seeds import slot_user_seeds  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "c1"
dev = torch.device("cuda", 0)
ctx = N.Context(0)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx.set_stream(stream.cuda_stream)
c = bench.CONFIGS[tag]
M, K, NT, ND = c["M"], c["K"], bench.NT, bench.ND
dims = [2 * M] + c["hidden"]
px = torch.empty((1, NT, M, 2), dtype=torch.float64, device=dev)
py = torch.empty((1, NT, K, 2), dtype=torch.float64, device=dev)
dx = torch.empty((1, ND, M, 2), dtype=torch.float32, device=dev)
tr = torch.empty((1, ND, K), dtype=torch.uint8, device=dev)
ctx.synthesize(N.Scenario(K, M, NT, ND, c["step"], bench.SNR, bench.GAIN),
               torch.tensor([1000], dtype=torch.int64, device=dev), px, py, dx, tr)
i1, h1 = slot_user_seeds(np.array([1000], np.uint64), K)
i1 = torch.from_numpy(i1.view(np.int64)).to(dev)
h1 = torch.from_numpy(h1.view(np.int64)).to(dev)
st = torch.empty((1, K), dtype=torch.int32, device=dev)
er = torch.empty((1, K), dtype=torch.int32, device=dev)
se = torch.empty((1, K), dtype=torch.int32, device=dev)
co = torch.empty((1, K, ND), dtype=torch.uint8, device=dev)
tcfg = N.TrainCfg.of(bench.EPOCHS, bench.BATCH, bench.LR)
for head in (False, True, False, True):
    dev_us, host_us = [], []
    for i in range(8):
        torch.cuda.synchronize()
        if head:
            torch.cuda._sleep(4_000_000)  # ~2 ms at 1.9 GHz
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        t0 = time.perf_counter()
        ctx.pipeline(dims, tcfg, 1, K, M, NT, ND, px, py, dx, tr, i1, h1, st, codes=co, bit_errors=er,
                     symbol_errors=se)
        host_us.append((time.perf_counter() - t0) * 1e6)
        b.record(stream)
        b.synchronize()
        if i >= 2:
            dev_us.append(a.elapsed_time(b) * 1e3)
    print(f"{tag} head_start={head}: device {statistics.median(dev_us):.1f} us, host call {statistics.median(host_us):.1f} us")
