"""Top SASS instructions of a kernel by warp-stall samples, with their source
line: python tools/ncu_sass_top.py rep.ncu-rep [top]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = None
items = []
for r in rows:
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        try:
            items.append((int(d.get("Warp Stall Sampling (All Samples)", "0") or 0), d))
        except ValueError:
            pass
tot = sum(i[0] for i in items) or 1
print("columns:", [h for h in hdr][:12] if hdr else None)
for smp, d in sorted(items, key=lambda x: -x[0])[:top]:
    print(f"{100*smp/tot:5.1f}% {d.get('Address','')} {d.get('Source','')[:70]:70s} inst={d.get('Instructions Executed','')}")
