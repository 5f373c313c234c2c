for i in 1 2 3; do
  timeout 600 python bench.py --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/n$i.json
  python -c "
import json;d=json.load(open('gpurun_out/n$i.json'));print('c2 run $i', '%.4g'%d['value'], d['phase_ms']['train'], d['clocks']['sm_mhz'], d['clocks'].get('power_w_max'))"
done
for i in 1 2; do
  timeout 600 python bench.py --config c5 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/m$i.json
  python -c "
import json;d=json.load(open('gpurun_out/m$i.json'));print('c5 run $i', '%.4g'%d['value'], d['phase_ms']['train'])"
done
