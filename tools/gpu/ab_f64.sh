# same-box A/B of two builds on the FP64 mode at C5 (296 slots, register-tiled FP64 kernel)
mkdir -p gpurun_out
for v in A B A B; do
  cp tools/gpu/ab/lib$v.so paper_2206_05998_b200/libnoma_b200.so
  timeout 600 python bench.py --precision 64 --slots 296 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 2>/dev/null | tail -1 > gpurun_out/abf64_$v.json
  python -c "
import json;e=json.load(open('gpurun_out/abf64_$v.json'));print('$v c5f64 %.5g'%e['value'], 'mode', e['train_kernel_mode'], 'train %.2f'%e['phase_ms']['train'])"
done
cp tools/gpu/ab/libA.so paper_2206_05998_b200/libnoma_b200.so
