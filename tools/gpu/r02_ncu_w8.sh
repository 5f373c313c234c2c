# one full ncu capture of the 8-warp kernel at the C4 shape (148 slots = 4736 nets)
mkdir -p gpurun_out
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:train_w8 -c 1 \
  -o gpurun_out/r02_ncu_train_w8_c4 -f python bench.py --config c4 --slots 148 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 \
  > gpurun_out/r02_ncu_w8.log 2>&1
tail -2 gpurun_out/r02_ncu_w8.log
