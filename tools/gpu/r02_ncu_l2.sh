# one full ncu capture of the two-hidden-layer kernel at the C2 bench shape
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:train_l2 -c 1 \
  -o gpurun_out/r02_ncu_train_l2_c2 -f python bench.py --config c2 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 \
  > gpurun_out/r02_ncu_l2.log 2>&1
tail -3 gpurun_out/r02_ncu_l2.log
