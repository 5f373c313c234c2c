# kernel durations of single-slot (latency mode) pipelines, C1 and C2
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lat_launches.csv python tools/latency_probe.py --configs c1,c2 --lat 16 --reps 3 > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows = list(csv.reader(open("gpurun_out/lat_launches.csv")))
h = next(r for r in rows if "Kernel Name" in r)
seen = collections.defaultdict(list)
for r in rows:
    if len(r) == len(h) and r[h.index("Metric Name")] == "gpu__time_duration.sum":
        seen[r[h.index("Kernel Name")].split("(")[0][:60]].append(float(r[h.index("Metric Value")].replace(",", "")))
for k, v in sorted(seen.items(), key=lambda kv: -max(kv[1])):
    print(f"{k:60s} n={len(v):3d} median {sorted(v)[len(v)//2]/1e3:9.1f} us  max {max(v)/1e3:9.1f} us")
PY
