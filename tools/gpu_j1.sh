mkdir -p gpurun_out
(free -g; nproc; lscpu | grep -E "Model name|Socket|Thread|Core") > gpurun_out/box.txt 2>&1
for c in c5 c2 c1 c4; do NOMA_PHASE_CLOCKS=1 timeout 300 python tools/profile_step.py --config $c --slots 148 2>&1 | grep -E "PHASE|ok" >> gpurun_out/phase_r02a.txt; done
