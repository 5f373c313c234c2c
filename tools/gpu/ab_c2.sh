# same-box A/B of two builds (tools/gpu/ab/libA.so, libB.so) on the C2 148-slot batch
mkdir -p gpurun_out
for v in A B A B; do
  cp tools/gpu/ab/lib$v.so paper_2206_05998_b200/libnoma_b200.so
  timeout 600 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | tail -1 > gpurun_out/abc2_$v.json
  python -c "
import json;e=json.load(open('gpurun_out/abc2_$v.json'));print('$v c2 %.5g'%e['value'], 'mode', e['train_kernel_mode'], 'train %.2f'%e['phase_ms']['train'], 'tf %.2f'%e['roofline']['achieved'], 'frac %.3f'%e['roofline']['frac'])"
done
cp tools/gpu/ab/libA.so paper_2206_05998_b200/libnoma_b200.so
