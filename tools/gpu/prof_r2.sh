mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_v16.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/launches_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"detect_ws_kernel" -c 1 -o gpurun_out/detect_ws_c3_v4 python bench.py --config c3 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_ws.log 2>&1
ls -la gpurun_out/*.csv gpurun_out/*.ncu-rep | tail -4
