# verification pass: the GPU suite, smoke, then the driver's default bench line
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/v_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/v_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/v_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v_smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/v_smoke.log
timeout 1200 python bench.py > gpurun_out/v_c5.log 2>&1; tail -1 gpurun_out/v_c5.log > gpurun_out/v_c5.json
tail -3 gpurun_out/v_gpu.log; tail -2 gpurun_out/v_smoke.log
python -c "
import json;e=json.load(open('gpurun_out/v_c5.json'));r=e['roofline'];print('c5 %.5g'%e['value'], 'e2e %.5g'%e['e2e']['value'], 'frac %.3f'%r['frac'], 'lat', e.get('latency_c1_us_per_slot'), e.get('latency_c2_us_per_slot'), e['clocks'])"
