# end-of-round state after the latency-path changes: GPU tests, every config's bench line,
# the reference arm and the C2 launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/fin_c2.json 2>gpurun_out/fin_c2.err; tail -1 gpurun_out/fin_c2.json | cut -c1-400
for c in c1 c3 c4 c5; do
  timeout 600 python bench.py --config $c --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/fin_$c.json
  python -c "import json;d=json.load(open('gpurun_out/fin_$c.json'));print('$c', '%.4g'%d['value'], d['roofline'].get('frac'), d.get('latency_us_per_slot'), d['clocks'])"
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 2>/dev/null | tail -1 > gpurun_out/fin_ref_c2.json; cut -c1-300 gpurun_out/fin_ref_c2.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_v30.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
