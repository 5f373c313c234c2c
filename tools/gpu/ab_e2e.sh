for v in A B A B A B; do
  cp tools/gpu/ab/lib$v.so paper_2206_05998_b200/libnoma_b200.so
  timeout 600 python bench.py --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/abe_$v.json
  python -c "
import json;d=json.load(open('gpurun_out/abe_$v.json'));print('$v value %.4g'%d['value'], 'e2e %.4g'%d['e2e']['value'], d['e2e']['ms_per_step'], d['ms_per_step'])"
done
