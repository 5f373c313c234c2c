mkdir -p gpurun_out
export NOMA_PARITY_LOG=gpurun_out/parity_lat.jsonl
timeout 600 python -m pytest tests/test_gpu_latency.py -x -q 2>&1 | grep -E "Error|error|passed|failed|assert" | head -20
timeout 300 python tools/latency_probe.py --lat ${LAT:-16} 2>&1 | tail -8
