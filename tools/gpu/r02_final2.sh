# end-of-session evidence: build, GPU suite, smoke, the default bench line, C4/C2/C3 lines,
# ncu launch list + full capture of the C5 training kernel, sanitizers over the latency kernel
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/f_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/f_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/f_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/f_smoke.log
timeout 1200 python bench.py > gpurun_out/f_c5.log 2>&1; tail -1 gpurun_out/f_c5.log > gpurun_out/f_c5.json
timeout 900 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/f_c4.json
timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/f_c3.json
tail -n 2 gpurun_out/f_gpu.log; tail -n 2 gpurun_out/f_smoke.log
for c in c5 c4 c3; do python -c "
import json;e=json.load(open('gpurun_out/f_$c.json'));r=e['roofline'];print('$c %.5g'%e['value'], 'e2e %.5g'%e['e2e']['value'], 'frac %.3f'%r['frac'], 'lat', e.get('latency_c1_us_per_slot'), e.get('latency_c2_us_per_slot'), e['clocks']['sm_mhz'], e['clocks']['reasons'])"; done
bash tools/gpu/r02_ncu_c5.sh
S=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 900 $S --tool $tool --print-limit 10 python tools/sanitize_small.py lat > gpurun_out/san_f_${tool}_lat.log 2>&1
  echo "== $tool lat: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san_f_${tool}_lat.log | tail -1) | $(grep -E '^lat ' gpurun_out/san_f_${tool}_lat.log | tr '\n' ' ')"
done
