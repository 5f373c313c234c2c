"""Print the per-warp step timeline written by NOMA_PHASE_TRACE (latency kernel).

usage: trace_view.py FILE [STEPS]; cycles relative to the step's earliest warp start.
"""
import sys

import numpy as np

t = np.loadtxt(sys.argv[1])[:1024].reshape(4, 16, 16)
names = ["start", "fwd", "bar1", "ysent", "gath", "ywait", "resid", "bar2", "bwd", "bar3", "f1done", "agwait", "rsissue", "wg2done", "rswait", "-"]
for st in range(int(sys.argv[2]) if len(sys.argv) > 2 else 1):
    z = t[st]
    live = [w for w in range(16) if z[w, 0] > 0]
    base = z[live, 0].min()
    print("step", 100 + st, " ".join(f"{n:>7s}" for n in names[:15]))
    for w in live:
        print(f"  w{w:2d}   " + " ".join(f"{int(z[w, i] - base):7d}" if z[w, i] > 0 else "      -" for i in range(15)))
