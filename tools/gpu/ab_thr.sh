# same-box A/B of two builds (tools/gpu/ab/libA.so, libB.so) on the throughput kernels:
# C5 (2960 slots, 4-warp kernel), C4 (1024 slots, 8-warp), C2 (148 slots, two-layer)
mkdir -p gpurun_out
for v in A B A B; do
  cp tools/gpu/ab/lib$v.so paper_2206_05998_b200/libnoma_b200.so
  for c in c5 c4 c2; do
    sl=""; [ $c = c5 ] && sl="--slots 2960"; [ $c = c4 ] && sl="--slots 1024"
    timeout 600 python bench.py --config $c $sl --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | tail -1 > gpurun_out/abt_$c_$v.json
    python -c "
import json;e=json.load(open('gpurun_out/abt_$c_$v.json'));print('$v $c %.5g'%e['value'], 'mode', e['train_kernel_mode'], 'train %.2f'%e['phase_ms']['train'], 'frac %.3f'%e['roofline']['frac'])"
  done
done
cp tools/gpu/ab/libA.so paper_2206_05998_b200/libnoma_b200.so
