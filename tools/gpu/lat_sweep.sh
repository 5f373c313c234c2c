# single-slot C1 latency over latency-kernel shapes (cluster size, warps per CTA)
mkdir -p gpurun_out
for v in "16:" "16:NOMA_LAT_WARPS=16" "8:" "8:NOMA_LAT_WARPS=16" "16:"; do
  cs=${v%%:*}; e=${v#*:}
  env $e timeout 600 python tools/latency_probe.py --configs c1 --lat $cs --reps 8 2>/dev/null | \
    python -c "import sys,json; [print('cs=$cs $e', d['config'], d['train_mode'], round(d['latency_us'],1), d['phase_us']['train']) for d in map(json.loads, sys.stdin)]"
done
