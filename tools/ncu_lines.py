"""Per-source-line instruction and stall-sample totals of one kernel in an
ncu report (needs -lineinfo): python tools/ncu_lines.py rep.ncu-rep [top] [file]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
want = sys.argv[3] if len(sys.argv) > 3 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur, agg, src = None, {}, {}
for r in rows:
    if len(r) == 2 and r[0] in ("File Name", "File Path"):
        cur = r[1].split("/")[-1]
        continue
    if len(r) < 8 or not r[0].isdigit():
        continue
    key = (cur, int(r[0]))
    src[key] = r[1]
    if r[2] == "-" or r[2] == "":
        try:
            agg[key] = (int(r[7] or 0), int(r[6] or 0))
        except ValueError:
            pass
tot_i = sum(v[0] for v in agg.values()) or 1
tot_s = sum(v[1] for v in agg.values()) or 1
print(f"total instructions {tot_i}, samples {tot_s}")
items = [(k, v) for k, v in agg.items() if (want is None or k[0] == want)]
for k, v in sorted(items, key=lambda kv: -kv[1][0])[:top]:
    print(f"inst {100*v[0]/tot_i:5.1f}%  stall {100*v[1]/tot_s:5.1f}%  {k[0]}:{k[1]}  {src[k].strip()[:90]}")
