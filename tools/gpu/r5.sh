mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_lls.py tests/test_gpu_pipeline.py tests/test_gpu_latency.py -x -q 2>&1 | grep -E "Error|error|passed|failed|assert" | head -20
timeout 300 python tools/latency_probe.py --lat 16 2>&1 | grep -v NOMA
