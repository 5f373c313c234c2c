mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_detect_tc.py -x -q 2>&1 | tail -1
NOMA_DETECT_CLK=1 timeout 600 python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline 2>&1 | grep NOMA_DETECT_CLK | tail -1
timeout 300 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_c3_ws.json
python -c "
import json;d=json.load(open('gpurun_out/bench_c3_ws.json'));print('ws', '%.3g'%d['value'], d['ms_per_step'], d['roofline'].get('frac'), d['roofline'].get('frac_of_attainable'), d.get('bit_errors'))"
