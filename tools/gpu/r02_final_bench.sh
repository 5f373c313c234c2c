# the driver's default bench command (C5 32768 slots + C1/C2 latency), then C4, C2 and C3 lines
mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/fb_c5.log 2>&1; tail -1 gpurun_out/fb_c5.log > gpurun_out/fb_c5.json
timeout 900 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/fb_c4.json
timeout 600 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/fb_c2.json
timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/fb_c3.json
for c in c5 c4 c2 c3; do python -c "
import json;e=json.load(open('gpurun_out/fb_$c.json'));r=e['roofline'];print('$c %.5g'%e['value'], 'e2e %.5g'%e['e2e']['value'], 'frac %.3f'%r['frac'], 'lat', e.get('latency_c1_us_per_slot'), e.get('latency_c2_us_per_slot'), e['clocks']['sm_mhz'], e['clocks']['reasons'])"; done
timeout 900 python bench.py --impl reference > gpurun_out/fb_ref.log 2>&1; tail -1 gpurun_out/fb_ref.log > gpurun_out/fb_ref.json
python -c "
import json;e=json.load(open('gpurun_out/fb_ref.json'));print('ref %.5g'%e['value'], e.get('cpu_baseline',{}).get('sample','')[:80], e.get('latency_us_per_slot_1core'))"
