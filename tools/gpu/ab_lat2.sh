# same-box A/B of single-slot latency (C1, C2) + the latency parity tests on B
for v in A B A B; do
  cp tools/gpu/ab/lib$v.so paper_2206_05998_b200/libnoma_b200.so
  timeout 600 python tools/latency_probe.py --configs c1,c2 --lat 16 --reps 8 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$v', d['config'], round(d['latency_us'],1), d['phase_us'])"
done
cp tools/gpu/ab/libB.so paper_2206_05998_b200/libnoma_b200.so
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
