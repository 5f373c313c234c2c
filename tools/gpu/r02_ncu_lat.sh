# one full ncu capture of the latency kernel at C1 and at C2 (one slot, 6 nets x 16 CTAs)
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
for cfg in c1 c2; do
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:train_lat -c 1 \
    -o gpurun_out/r02_ncu_lat_$cfg -f python tools/latency_probe.py --configs $cfg --clusters 1 --lat 16 --reps 3 \
    > gpurun_out/r02_ncu_lat_$cfg.log 2>&1
  tail -n 2 gpurun_out/r02_ncu_lat_$cfg.log
done
