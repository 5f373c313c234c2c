# per-kernel device times of one single-slot C1 / C2 pipeline call (serialised by ncu)
mkdir -p gpurun_out
for c in c1 c2; do
timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lat_launches_$c.csv \
  python tools/latency_probe.py --configs $c --clusters 1 --lat 16 --reps 1 > /dev/null 2>&1
python - <<PY
import csv
rows=list(csv.reader(open('gpurun_out/lat_launches_$c.csv')))
h=rows[0]; ik=h.index('Kernel Name'); iv=h.index('Metric Value'); iid=h.index('ID')
seen=[(r[iid], r[ik][:60], float(r[iv])/1000) for r in rows[1:] if len(r)>iv]
for i,k,v in seen[-14:]: print('$c', i, k, '%.1f us'%v)
PY
done
