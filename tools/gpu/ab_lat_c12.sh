# same-box A/B of tools/gpu/ab/libA.so vs libB.so on the C1 and C2 single-slot latency,
# then the latency parity tests on B (EXTRA: more latency_probe arguments for a cluster-size check)
mkdir -p gpurun_out
for v in A B A B A B; do
  cp tools/gpu/ab/lib$v.so paper_2206_05998_b200/libnoma_b200.so
  timeout 300 python tools/latency_probe.py --configs c1,c2 --lat 16 --reps 8 2>/dev/null | python -c "import sys,json; [print('$v', d['config'], round(d['latency_us'],1), d['phase_us']['train']) for d in map(json.loads, sys.stdin)]"
done
if [ -n "$EXTRA" ]; then timeout 300 python tools/latency_probe.py $EXTRA 2>/dev/null | python -c "import sys,json; [print('X', d['config'], d['cluster'], round(d['latency_us'],1), d['phase_us']['train']) for d in map(json.loads, sys.stdin)]"; fi
cp tools/gpu/ab/libB.so paper_2206_05998_b200/libnoma_b200.so
timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_latency.py tests/test_gpu_pipeline.py tests/test_gpu_parity_full.py 2>&1 | tail -3
