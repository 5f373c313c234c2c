mkdir -p gpurun_out
# launch list of the default bench command (cold-cache, serialised per-launch times)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/launches_bench.log 2>&1
# one full capture of the dominant kernel (throughput train kernel, C2, 148 slots)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"train_kernel" -c 1 -o gpurun_out/train_c2_v10 python tools/profile_step.py --config c2 --slots 148 > gpurun_out/ncu_train.log 2>&1
# latency kernel at one C2 slot
timeout 600 ncu --set full --clock-control none --import-source on -k regex:train_lat_kernel -c 1 -o gpurun_out/lat_c2 python tools/profile_step.py --config c2 --slots 1 > gpurun_out/ncu_lat2.log 2>&1
ls -la gpurun_out
