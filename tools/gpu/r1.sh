set -x; mkdir -p gpurun_out
nvidia-smi -L; nproc
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 600 python bench.py 2>&1 | tail -2 > gpurun_out/bench_c2.json
cat gpurun_out/bench_c2.json
