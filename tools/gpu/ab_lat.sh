# same-box A/B of two builds (tools/gpu/ab/libA.so, libB.so) on the single-slot
# C1 / C2 latency (tools/latency_probe.py, median of 8 after 2 warm calls)
mkdir -p gpurun_out
for v in A B A B; do
  cp tools/gpu/ab/lib$v.so paper_2206_05998_b200/libnoma_b200.so
  timeout 600 python tools/latency_probe.py --configs c1,c2 --lat 16 --reps 10 2>/dev/null | \
    python -c "import sys,json; [print('$v', d['config'], round(d['latency_us'],1), d['phase_us']['train']) for d in map(json.loads, sys.stdin)]"
done
