mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 600 python tools/latency_probe.py --configs c1,c2 --lat 16 2>&1 | grep -E "config|LLS_CLOCKS"
timeout 600 python bench.py 2>/dev/null | tail -1 > gpurun_out/bench_default_chol.json
python -c "
import json;d=json.load(open('gpurun_out/bench_default_chol.json'));print('%.4g'%d['value'], d['phase_ms'], d['latency_us_per_slot'], d['latency_c1_us_per_slot'], d['e2e']['value'])"
