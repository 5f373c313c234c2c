"""Instructions executed and stall samples per source-line range of a kernel
(needs -lineinfo): python tools/ncu_ranges.py rep file name:lo-hi ..."""
import csv
import subprocess
import sys

rep, fname = sys.argv[1], sys.argv[2]
ranges = []
for a in sys.argv[3:]:
    name, span = a.split(":")
    lo, hi = span.split("-")
    ranges.append((name, int(lo), int(hi)))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur = None
acc = {r[0]: [0, 0] for r in ranges}
acc["other"] = [0, 0]
for r in rows:
    if len(r) == 2 and r[0] in ("File Name", "File Path"):
        cur = r[1].split("/")[-1]
        continue
    if len(r) < 8 or not r[0].isdigit() or r[2] not in ("-", ""):
        continue
    ln = int(r[0])
    inst, samp = int(r[7] or 0), int(r[6] or 0)
    key = "other"
    if cur == fname:
        for name, lo, hi in ranges:
            if lo <= ln <= hi:
                key = name
                break
    acc[key][0] += inst
    acc[key][1] += samp
ti = sum(v[0] for v in acc.values()) or 1
ts = sum(v[1] for v in acc.values()) or 1
for k, v in acc.items():
    print(f"{k:12s} inst {v[0]:12d} ({100*v[0]/ti:5.1f}%)  stall samples {100*v[1]/ts:5.1f}%")
