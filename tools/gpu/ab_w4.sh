# same-box A/B of two builds of libnoma_b200.so (tools/gpu/ab/libA.so, libB.so)
# on C5 (2960 slots), with the 4-warp kernel's de-phasing start as a third arm
mkdir -p gpurun_out
for v in A B Bd A B Bd; do
  lib=${v:0:1}
  cp tools/gpu/ab/lib$lib.so paper_2206_05998_b200/libnoma_b200.so
  d=0; [ "$v" = "Bd" ] && d=10000
  NOMA_W4_DEPHASE=$d timeout 600 python bench.py --slots 2960 --steps 3 --warmup 1 --no-cpu-baseline --e2e-steps 1 2>/dev/null | tail -1 > gpurun_out/abw4_$v.json
  python -c "
import json;e=json.load(open('gpurun_out/abw4_$v.json'));print('$v c5 %.5g'%e['value'], 'train %.1f'%e['phase_ms']['train'], 'tf %.2f'%e['roofline']['achieved'])"
done
