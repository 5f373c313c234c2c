for v in A B A0 A B A0; do
  lib=${v:0:1}; e=""; [ "$v" = "A0" ] && e="NOMA_DETECT_TC=0"
  cp tools/gpu/ab/lib$lib.so paper_2206_05998_b200/libnoma_b200.so
  env $e timeout 300 python tools/latency_probe.py --configs c1 --clusters 1 --lat 16 --reps 8 2>/dev/null | python -c "import sys,json; [print('$v', round(d['latency_us'],1), d['phase_us']) for d in map(json.loads, sys.stdin)]"
done
