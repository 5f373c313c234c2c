mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 300 python bench.py --config c3 --steps 5 --warmup 3 2>&1 | tail -1 > gpurun_out/bench_c3_ws.json
python -c "
import json;d=json.load(open('gpurun_out/bench_c3_ws.json'));r=d['roofline'];print('c3', '%.3g'%d['value'], d['ms_per_step'], 'frac', round(r['frac'],3), 'vs bf16/2', round(r['frac_vs_bf16_half'],3), 'attain', round(r['frac_of_attainable'],3), r['attainable_ms'], 'e2e %.3g'%d['e2e']['value'], 'cpu', d['cpu_baseline'])"
timeout 900 python bench.py 2>/dev/null | tail -1 > gpurun_out/bench_default3.json
python -c "
import json;d=json.load(open('gpurun_out/bench_default3.json'));print('%.4g'%d['value'], d['phase_ms'], d['latency_us_per_slot'], d['latency_c1_us_per_slot'])"
