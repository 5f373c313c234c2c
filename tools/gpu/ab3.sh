for v in A B A B; do
  cp tools/gpu/ab/lib$v.so paper_2206_05998_b200/libnoma_b200.so
  line="$v"
  for c in c2 c1 c5; do
    timeout 600 python bench.py --config $c --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/ab3_${v}_$c.json
    line="$line $c $(python -c "import json;d=json.load(open('gpurun_out/ab3_${v}_$c.json'));print('%.4g'%d['value'])")"
  done
  echo $line
done
