# LLS changes: parity tests, then same-box A/B of the single-slot latency and the LLS kernel time
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_lls.py tests/test_gpu_pipeline.py tests/test_gpu_hybrid.py -m gpu -x -q 2>&1 | tail -3
bash tools/gpu/ab_lat_tl.sh
for v in A B; do
  cp tools/gpu/ab/lib$v.so paper_2206_05998_b200/libnoma_b200.so
  timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -k regex:lls_kernel --csv \
    python tools/latency_probe.py --configs c1 --clusters 1 --lat 16 --reps 1 2>/dev/null | grep lls_kernel | tail -2 | awk -F'","' -v v=$v '{print v, $5, $NF}'
done
cp tools/gpu/ab/libA.so paper_2206_05998_b200/libnoma_b200.so
