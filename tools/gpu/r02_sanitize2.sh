# compute-sanitizer over the kernels changed late in round 2: LLS (Cholesky /
# warp solves / r0 kernel), init, shuffles, the 4-warp, 8-warp and
# two-hidden-layer training kernels, detection, and the latency kernel
mkdir -p gpurun_out
S=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  for m in w4 l2 w8 generic lat; do
    timeout 1200 $S --tool $tool --print-limit 10 python tools/sanitize_small.py $m > gpurun_out/san2_${tool}_${m}.log 2>&1
    echo "== $tool $m: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san2_${tool}_${m}.log | tail -1) | $(grep -E '^(w4|l2|w8|generic|f64|lat) ' gpurun_out/san2_${tool}_${m}.log | tr '\n' ' ')"
  done
done
