mkdir -p gpurun_out
export NOMA_PARITY_LOG=$PWD/gpurun_out/parity_j3.jsonl
rm -f $NOMA_PARITY_LOG
NOMA_PARITY_MEASURE=1 timeout 1200 python -m pytest tests/test_gpu_parity_full.py -q 2>&1 | tail -5 > gpurun_out/j3_parity.txt
timeout 1500 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_parity_full.py 2>&1 | tail -15 > gpurun_out/j3_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/j3_smoke.txt 2>&1
for c in c5 c1 c2; do timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/j3_bench_$c.json; done
timeout 900 python bench.py --config c5 --slots 2048 --steps 2 --warmup 1 --no-cpu-baseline 2>&1 | tail -2 > gpurun_out/j3_bench_c5_2048.json
