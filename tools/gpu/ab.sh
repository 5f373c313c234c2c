for v in A B A B; do
  cp tools/gpu/ab/lib$v.so paper_2206_05998_b200/libnoma_b200.so
  timeout 600 python bench.py --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/ab_$v.json
  timeout 600 python bench.py --config c5 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/ab5_$v.json
  python -c "
import json;d=json.load(open('gpurun_out/ab_$v.json'));e=json.load(open('gpurun_out/ab5_$v.json'));print('$v c2 %.4g'%d['value'], d['phase_ms']['train'], ' c5 %.4g'%e['value'], e['phase_ms']['train'])"
done
