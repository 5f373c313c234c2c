mkdir -p gpurun_out
export NOMA_PARITY_LOG=gpurun_out/parity_full.jsonl
rm -f $NOMA_PARITY_LOG
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py 2>&1 | tail -1 > gpurun_out/bench_c2_v12.json
python -c "
import json;d=json.load(open('gpurun_out/bench_c2_v12.json'));print('%.4g'%d['value'], d['latency_us_per_slot'], d['latency_c1_us_per_slot'], d['roofline']['frac'], d['phase_ms'])"
