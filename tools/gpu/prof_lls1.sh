# ncu --set full of the single-slot LLS kernel (C1 latency pipeline)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"lls_kernel" -c 1 -o gpurun_out/lls_c1_1slot python tools/latency_probe.py --configs c1 --lat 16 --reps 1 > gpurun_out/ncu_lls.log 2>&1
ls -la gpurun_out/lls_c1_1slot.ncu-rep
