mkdir -p gpurun_out
for c in c1 c4 c5; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_${c}_v11.json; done
NOMA_PHASE_CLOCKS=1 timeout 300 python tools/profile_step.py --config c5 --slots 148 2>&1 | grep PHASE
NOMA_PHASE_CLOCKS=1 timeout 300 python tools/profile_step.py --config c2 --slots 148 2>&1 | grep PHASE
