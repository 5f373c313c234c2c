mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py 2>gpurun_out/bench_default.err | tail -1 > gpurun_out/bench_default.json
python -c "
import json;d=json.load(open('gpurun_out/bench_default.json'));print('%.4g'%d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d.get('latency_c1_us_per_slot'), d['clocks'], d['cpu_baseline']['value'])"
