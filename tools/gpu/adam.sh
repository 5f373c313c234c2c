mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for c in c2 c1 c5; do
  timeout 600 python bench.py --config $c --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/bench_${c}_adam.json
  python -c "
import json;d=json.load(open('gpurun_out/bench_${c}_adam.json'));print('$c', '%.4g'%d['value'], round(d['roofline']['frac'],4), d['phase_ms']['train'], d.get('latency_us_per_slot'))"
done
