# same-box comparison of several builds tools/gpu/ab/lib$V.so (V in $LIBS, first = baseline)
# on the C1 and C2 single-slot latency, three rounds; then the latency parity tests on each non-baseline build
mkdir -p gpurun_out
for rep in 1 2 3; do
  for v in $LIBS; do
    cp tools/gpu/ab/lib$v.so paper_2206_05998_b200/libnoma_b200.so
    timeout 300 python tools/latency_probe.py --configs c1,c2 --lat 16 --reps 8 2>/dev/null | python -c "import sys,json; [print('$v', d['config'], round(d['latency_us'],1), d['phase_us']['train']) for d in map(json.loads, sys.stdin)]"
  done
  cp tools/gpu/ab/libA.so paper_2206_05998_b200/libnoma_b200.so
  NOMA_LAT_WARPS=16 timeout 300 python tools/latency_probe.py --configs c2 --lat 16 --reps 8 2>/dev/null | python -c "import sys,json; [print('A-w16', d['config'], round(d['latency_us'],1), d['phase_us']['train']) for d in map(json.loads, sys.stdin)]"
done
for v in $LIBS; do
  [ "$v" = A ] && continue
  cp tools/gpu/ab/lib$v.so paper_2206_05998_b200/libnoma_b200.so
  echo "tests $v: $(timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_latency.py tests/test_gpu_pipeline.py tests/test_gpu_parity_full.py 2>&1 | tail -1)"
done
