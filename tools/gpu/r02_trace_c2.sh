# cluster-size check on the release build, then the per-warp timeline of
# latency-kernel steps 100-103 (trace build: cycle probes compiled in)
mkdir -p gpurun_out
# (cluster size: NOMA_LAT_CLUSTER=8 measured 3.08 ms for C2)
NOMA_BUILD_TRACE=1 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/t_build.log 2>&1
NOMA_PHASE_TRACE=gpurun_out/tl_c2.txt timeout 300 python tools/latency_probe.py --configs c2 --lat 16 --reps 4 > gpurun_out/t_c2.log 2>&1
NOMA_PHASE_TRACE=gpurun_out/tl_c1.txt timeout 300 python tools/latency_probe.py --configs c1 --lat 16 --reps 4 > gpurun_out/t_c1.log 2>&1
tail -n 3 gpurun_out/t_c2.log gpurun_out/t_c1.log
