for v in A B A B; do
  cp tools/gpu/ab/lib$v.so paper_2206_05998_b200/libnoma_b200.so
  timeout 600 python tools/latency_probe.py --configs c1,c2 --lat 16 --reps 8 2>&1 | grep config | python -c "
import sys, json
for line in sys.stdin:
    d = json.loads(line); print('$v', d['config'], round(d['latency_us']), d['phase_us']['train'], d['bit_errors'])"
done
