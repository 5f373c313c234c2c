"""Histogram of the distance (in instructions) between an FFMA2/FFMA and the
previous instruction writing its accumulator input, per SASS function."""
import re
import subprocess
import sys
from collections import Counter

obj, fun = sys.argv[1], sys.argv[2]
sass = subprocess.run(["cuobjdump", "-sass", "-fun", fun, obj], capture_output=True, text=True).stdout
ins = []
for line in sass.splitlines():
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m:
        ins.append(m.group(2).strip())
last_write = {}
hist = Counter()
for idx, s in enumerate(ins):
    mm = re.match(r"(?:@!?U?P\w+\s+)?(FFMA2|FFMA)\s+(R\d+),\s*(.*)", s)
    if mm:
        ops = [o.strip() for o in mm.group(3).split(",")]
        acc = re.match(r"(R\d+)", ops[-1])
        if acc and acc.group(1) in last_write:
            d = idx - last_write[acc.group(1)]
            hist[min(d, 40)] += 1
    dm = re.match(r"(?:@!?U?P\w+\s+)?[A-Z0-9.]+\s+(R\d+)", s)
    if dm:
        last_write[dm.group(1)] = idx
tot = sum(hist.values())
print(f"{tot} dependent FMAs; distance histogram (<=40):")
acc = 0
for d in sorted(hist):
    acc += hist[d]
    if d <= 12 or d in (16, 20, 24, 32, 40):
        print(f"  d={d:2d}: {hist[d]:5d}  cum {acc / tot:.2f}")
