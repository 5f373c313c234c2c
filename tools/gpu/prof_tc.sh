mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"detect_(tc|ws)_kernel" -c 1 -o gpurun_out/detect_ws_c3_v2 python bench.py --config c3 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_tc.log 2>&1
tail -3 gpurun_out/ncu_tc.log
ls -la gpurun_out/*.ncu-rep
