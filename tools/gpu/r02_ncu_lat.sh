# one full ncu capture of the latency kernel at C1 (one slot, 6 nets x 16 CTAs)
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:train_lat -c 1 \
  -o gpurun_out/r02_ncu_lat_c1 -f python tools/latency_probe.py --configs c1 --clusters 1 --lat 16 --reps 1 \
  > gpurun_out/r02_ncu_lat.log 2>&1
tail -3 gpurun_out/r02_ncu_lat.log
