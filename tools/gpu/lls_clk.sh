# LLS phase cycles (NOMA_BUILD_TRACE=1 builds A / B in tools/gpu/ab/)
for v in A B A B; do
  cp tools/gpu/ab/lib$v.so paper_2206_05998_b200/libnoma_b200.so
  NOMA_PHASE_CLOCKS=1 timeout 300 python tools/latency_probe.py --configs c1 --clusters 1 --lat 16 --reps 2 2>&1 | grep LLS_CLOCKS | tail -1 | sed "s/^/$v /"
done
