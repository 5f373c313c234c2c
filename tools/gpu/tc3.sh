mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for impl in tc ffma; do
  if [ $impl = ffma ]; then export NOMA_DETECT_TC=0; fi
  timeout 600 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_c3_$impl.json
  python -c "
import json;d=json.load(open('gpurun_out/bench_c3_$impl.json'));print('$impl', '%.3g'%d['value'], d['ms_per_step'], d['roofline'].get('frac_of_3xtf32_ceiling'), d['roofline']['kernel'], d.get('bit_errors'))"
done
unset NOMA_DETECT_TC
timeout 900 python bench.py 2>/dev/null | tail -1 > gpurun_out/bench_default2.json
python -c "
import json;d=json.load(open('gpurun_out/bench_default2.json'));print('%.4g'%d['value'], d['phase_ms'], d['latency_us_per_slot'], d['latency_c1_us_per_slot'])"
