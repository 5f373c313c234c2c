# one full ncu capture of the single-slot LLS kernel (C1)
mkdir -p gpurun_out
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:lls_kernel -c 1 \
  -o gpurun_out/r02_ncu_lls_c1 -f python tools/latency_probe.py --configs c1 --clusters 1 --lat 16 --reps 1 > gpurun_out/r02_ncu_lls.log 2>&1
tail -2 gpurun_out/r02_ncu_lls.log
