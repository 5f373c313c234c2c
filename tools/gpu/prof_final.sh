mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_v27.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"train_kernel" -c 1 -o gpurun_out/train_c2_v27 python tools/profile_step.py --config c2 --slots 148 > gpurun_out/ncu_train27.log 2>&1
ls -la gpurun_out/launches_c2_v27.csv gpurun_out/train_c2_v27.ncu-rep
