# product build without compiled-in cycle probes: C5 bench line, C3, C2 batch
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/np_c5.log 2>&1; tail -1 gpurun_out/np_c5.log > gpurun_out/np_c5.json
timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 2 2>/dev/null | tail -1 > gpurun_out/np_c3.json
timeout 600 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | tail -1 > gpurun_out/np_c2.json
for c in c5 c3 c2; do python -c "
import json;e=json.load(open('gpurun_out/np_$c.json'));r=e['roofline'];print('$c %.5g'%e['value'], 'e2e %.5g'%e['e2e']['value'], 'frac %.3f'%r['frac'], 'lat', e.get('latency_c1_us_per_slot'), e.get('latency_c2_us_per_slot'), e['clocks'])"; done
