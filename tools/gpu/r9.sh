mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_latency.py -x -q 2>&1 | grep -E "Error|error|passed|failed|assert" | head -20
NOMA_PHASE_TRACE=gpurun_out/trace_c1_w8.txt timeout 300 python tools/latency_probe.py --configs c1 --lat 16 2>&1 | grep -v NOMA
NOMA_PHASE_TRACE=gpurun_out/trace_c2.txt timeout 300 python tools/latency_probe.py --configs c2 --lat 16 2>&1 | grep -v NOMA
