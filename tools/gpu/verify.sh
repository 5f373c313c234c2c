mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py 2>gpurun_out/bench_v25.err | tail -1 > gpurun_out/bench_v25.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 2>/dev/null | tail -1 > gpurun_out/ref_v25.json
timeout 600 python bench.py --config c3 --steps 5 --warmup 3 2>/dev/null | tail -1 > gpurun_out/c3_v25.json
python - <<'PY'
import json
d=json.load(open('gpurun_out/bench_v25.json'))
print('default', '%.4g'%d['value'], 'frac', round(d['roofline']['frac'],4), 'e2e %.4g'%d['e2e']['value'], 'lat', round(d['latency_us_per_slot']), round(d['latency_c1_us_per_slot']), d['clocks'], 'launches', d['gpu_launches'], 'cpu', round(d['cpu_baseline']['value']))
r=json.load(open('gpurun_out/ref_v25.json')); print('reference', r.get('value'), r.get('unit'), r.get('cpu_baseline',{}).get('cores'), r.get('impl'))
c=json.load(open('gpurun_out/c3_v25.json')); print('c3', '%.4g'%c['value'], round(c['roofline']['frac'],3), c.get('bit_errors'), 'e2e %.3g'%c['e2e']['value'])
PY
