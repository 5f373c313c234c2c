mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_hybrid.py tests/test_gpu_pipeline.py tests/test_gpu_fp64.py -x -q 2>&1 | tail -2
for c in c2 c5 c1; do timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_${c}_pf.json; python -c "
import json;d=json.load(open('gpurun_out/bench_${c}_pf.json'));print('$c', '%.4g'%d['value'], round(d['roofline']['frac'],4), d['phase_ms'])"; done
NOMA_PHASE_CLOCKS=1 timeout 300 python tools/profile_step.py --config c5 --slots 148 2>&1 | grep PHASE
