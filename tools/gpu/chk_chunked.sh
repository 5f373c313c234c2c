timeout 600 python -m pytest tests/test_gpu_detect_tc.py -q -x 2>&1 | tail -4
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for i in 1 2; do timeout 300 python bench.py --config c3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/c3_e2e.json; python -c "
import json;d=json.load(open('gpurun_out/c3_e2e.json'));print('%.4g'%d['value'], d['e2e'], d['gpu_launches'])"; done
