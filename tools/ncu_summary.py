import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[0]
want = ["Duration", "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread",
        "Achieved Occupancy", "Eligible Warps Per Scheduler", "No Eligible", "Warp Cycles Per Issued Instruction",
        "Executed Instructions", "L1/TEX Hit Rate", "DRAM Throughput", "Dynamic Shared Memory Per Block", "Memory Throughput"]
for row in r[1:]:
    d = dict(zip(h, row))
    if d.get("Metric Name") in want:
        print(f"{d['Metric Name'][:45]:45s} {d['Metric Unit'][:12]:12s} {d['Metric Value']}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
cur = None; agg = []
for x in rows:
    if len(x) == 2 and x[0] == "File Path": cur = x[1].split("/")[-1]; continue
    if len(x) < 8: continue
    try: ln = int(x[0])
    except: continue
    if x[2] == "-":
        s = int(x[4]) if x[4].isdigit() else 0
        agg.append((s, cur, ln, x[1][:80], x[7]))
tot = sum(a[0] for a in agg) or 1
for a in sorted(agg, reverse=True)[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{a[0]/tot*100:5.1f}% {a[1]}:{a[2]} inst={a[4]} | {a[3]}")
