# single-slot latency under NOMA_LAT_EXP variants of the latency kernel (one
# build; the variants are runtime switches), interleaved twice
mkdir -p gpurun_out
for round in 1 2; do
  for x in ${LAT_EXPS:-0 1}; do
    NOMA_LAT_EXP=$x timeout 600 python tools/latency_probe.py --configs c1,c2 --lat 16 --reps 10 2>/dev/null | \
      python -c "import sys,json; [print('exp=$x', d['config'], round(d['latency_us'],1), d['phase_us']['train']) for d in map(json.loads, sys.stdin)]"
  done
done
