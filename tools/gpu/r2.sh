mkdir -p gpurun_out
export NOMA_PARITY_LOG=gpurun_out/parity_lat.jsonl
timeout 600 python -m pytest tests/test_gpu_latency.py -x -q 2>&1 | tail -15
timeout 300 python tools/latency_probe.py --clusters 1 2>&1 | tail -8
