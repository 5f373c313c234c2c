# same-box A/B of two builds of libnoma_b200.so on the single-slot C1 latency
for v in A B A B A B; do
  cp tools/gpu/ab/lib$v.so paper_2206_05998_b200/libnoma_b200.so
  timeout 300 python tools/latency_probe.py --configs ${CFG:-c1} --clusters 1 --lat 16 --reps 8 2>/dev/null | python -c "import sys,json; [print('$v', round(d['latency_us'],1), d['phase_us']['train']) for d in map(json.loads, sys.stdin)]"
done
