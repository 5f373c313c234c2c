# ncu evidence for the C5 bench line: the launch list of the bench command
# (per-launch durations, serialised) and one full capture of the training
# kernel at the C5 shape (296 slots = 4736 user nets in one launch).
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 1500 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r02_launches_c5.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 \
  > gpurun_out/r02_launches_bench.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:train_w4 -c 1 \
  -o gpurun_out/r02_ncu_train_w4_c5 -f python bench.py --slots 296 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 \
  > gpurun_out/r02_ncu_full.log 2>&1
