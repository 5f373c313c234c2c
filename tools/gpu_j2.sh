mkdir -p gpurun_out
export NOMA_PARITY_LOG=$PWD/gpurun_out/parity_j2.jsonl
rm -f $NOMA_PARITY_LOG
timeout 900 python -m pytest tests/test_gpu_parity_full.py -x -q 2>&1 | tail -15 > gpurun_out/j2_parity.txt
timeout 600 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_hybrid.py -x -q 2>&1 | tail -15 > gpurun_out/j2_tests.txt
for c in c5 c1; do NOMA_PHASE_CLOCKS=1 timeout 300 python tools/profile_step.py --config $c --slots 148 2>&1 | grep -E "PHASE|ok|Error|error" >> gpurun_out/j2_phase.txt; done
for c in c5 c1; do timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/j2_bench_$c.json; done
