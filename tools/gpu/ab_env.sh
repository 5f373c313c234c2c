# same-build A/B of an environment switch on one throughput config:
#   CFG=c5 SLOTS=2960 VAR=NOMA_W4_GATHER4 bash tools/gpu/ab_env.sh   (A: VAR unset, B: VAR=0)
mkdir -p gpurun_out
c=${CFG:-c5}; sl=${SLOTS:+--slots $SLOTS}
for v in A B A B; do
  if [ $v = B ]; then export $VAR=0; else unset $VAR; fi
  timeout 600 python bench.py --config $c $sl --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | tail -1 > gpurun_out/abe_$v.json
  python -c "
import json;e=json.load(open('gpurun_out/abe_$v.json'));print('$v $c %.5g'%e['value'], 'mode', e['train_kernel_mode'], 'train %.2f'%e['phase_ms']['train'], 'frac %.3f'%e['roofline']['frac'])"
done
unset $VAR
