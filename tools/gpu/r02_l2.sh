# two-hidden-layer kernel (k_train_l2.cu): parity tests, then C2 bench with
# the new kernel (NOMA_TRAIN_L2=1) against the 16-warp kernel (=0)
mkdir -p gpurun_out; export NOMA_PARITY_LOG=gpurun_out/l2_parity.jsonl; rm -f $NOMA_PARITY_LOG
timeout 900 python -m pytest tests/test_gpu_pipeline.py -m gpu -x -q -k "c2_shape or l2_wide" 2>&1 | tail -5
timeout 900 python -m pytest tests/test_gpu_parity_full.py -m gpu -x -q -k c2_bench148 2>&1 | tail -3
for v in 1 0 1 0; do
  NOMA_TRAIN_L2=$v timeout 600 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | tail -1 > gpurun_out/l2_$v.json
  python -c "
import json;e=json.load(open('gpurun_out/l2_$v.json'));print('l2=$v c2 %.5g'%e['value'], 'mode', e['train_kernel_mode'], 'train %.2f'%e['phase_ms']['train'], 'tf %.2f'%e['roofline']['achieved'], 'frac %.3f'%e['roofline']['frac'])"
done
cat gpurun_out/l2_parity.jsonl
