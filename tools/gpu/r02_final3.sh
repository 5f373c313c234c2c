# final build check: GPU suite, smoke, the driver's default bench line, the reference arm
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/g_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/g_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g_smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/g_smoke.log
timeout 1200 python bench.py > gpurun_out/g_c5.log 2>&1; tail -1 gpurun_out/g_c5.log > gpurun_out/g_c5.json
timeout 900 python bench.py --impl reference > gpurun_out/g_ref.log 2>&1; tail -1 gpurun_out/g_ref.log > gpurun_out/g_ref.json
tail -n 2 gpurun_out/g_gpu.log; tail -n 2 gpurun_out/g_smoke.log
python -c "
import json;e=json.load(open('gpurun_out/g_c5.json'));r=e['roofline'];print('c5 %.5g'%e['value'], 'e2e %.5g'%e['e2e']['value'], 'frac %.3f'%r['frac'], 'lat', e.get('latency_c1_us_per_slot'), e.get('latency_c2_us_per_slot'), e['clocks']['sm_mhz'], e['clocks']['reasons'])
e=json.load(open('gpurun_out/g_ref.json'));print('ref %.5g'%e['value'], e.get('cpu_baseline',{}).get('cores'))"
