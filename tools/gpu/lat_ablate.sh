for e in 0 1 2 4 7 0; do
  NOMA_LAT_EXP=$e timeout 300 python tools/latency_probe.py --configs c1 --clusters 1 --lat 16 --reps 6 2>/dev/null | python -c "import sys,json; [print('exp=$e', round(d['latency_us'],1), d['phase_us']['train']) for d in map(json.loads, sys.stdin)]"
done
