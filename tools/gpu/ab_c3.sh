for v in A B A B; do
  cp tools/gpu/ab/lib$v.so paper_2206_05998_b200/libnoma_b200.so
  timeout 600 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/abc3_$v.json
  python -c "
import json;d=json.load(open('gpurun_out/abc3_$v.json'));print('$v c3 %.4g'%d['value'], d['ms_per_step'], d['roofline']['frac'], d['bit_errors'])"
done
cp tools/gpu/ab/libB.so paper_2206_05998_b200/libnoma_b200.so
NOMA_DETECT_CLK=1 timeout 600 python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline 2>&1 | grep NOMA_DETECT_CLK | tail -1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
