"""Print the per-warp step timeline written by NOMA_PHASE_TRACE (latency kernel)."""
import sys

import numpy as np

t = np.loadtxt(sys.argv[1])[:1024].reshape(4, 16, 16)
names = ["start", "fwd", "bar1", "ysent", "gath", "ywait", "resid", "bar2", "bwd", "bar3", "f1done", "agwait", "rsissue", "wg2done", "rswait", "-"]
for st in range(int(sys.argv[2]) if len(sys.argv) > 2 else 1):
    print("step", 100 + st, " ".join(f"{n:>6s}" for n in names))
    rel = t[st] - t[st, :, 0].min()
    for w in range(16):
        print(f"  w{w:2d}     " + " ".join(f"{int(x):6d}" if t[st, w, i] > 0 else "     -" for i, x in enumerate(rel[w])))
