mkdir -p gpurun_out
nvidia-smi --query-gpu=memory.total,memory.used --format=csv > gpurun_out/j4_mem.txt
timeout 1500 python bench.py --steps 3 --warmup 1 > gpurun_out/j4_bench.json 2> gpurun_out/j4_bench.err
nvidia-smi --query-gpu=memory.total,memory.used --format=csv >> gpurun_out/j4_mem.txt
