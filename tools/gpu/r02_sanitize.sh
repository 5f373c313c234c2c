# compute-sanitizer over the round-2 kernels (4-warp training, shape-general
# training / detection, FP64 pipeline mode, the C++ API's FP64 kernels through
# the reference tests) and the latency kernel again
mkdir -p gpurun_out
S=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  for m in w4 generic lat; do
    timeout 900 $S --tool $tool --print-limit 10 python tools/sanitize_small.py $m > gpurun_out/san_r02_${tool}_${m}.log 2>&1
    echo "== $tool $m: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san_r02_${tool}_${m}.log | tail -1) | $(grep -E '^(w4|generic|f64|lat) ' gpurun_out/san_r02_${tool}_${m}.log | tr '\n' ' ')"
  done
  timeout 900 $S --tool $tool --print-limit 10 --target-processes all python tools/sanitize_small.py dense > gpurun_out/san_r02_${tool}_dense.log 2>&1
  echo "== $tool dense: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san_r02_${tool}_dense.log | tail -3 | tr '\n' ' ') | $(grep -E '^dense ' gpurun_out/san_r02_${tool}_dense.log | tr '\n' ' ')"
done
