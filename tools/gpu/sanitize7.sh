# compute-sanitizer over the tcgen05 detection path after the persistent grid,
# the per-half A2 hand-off and the row-stride launches: the pipeline (tc) and
# CTAs spanning several nets (tcmulti)
mkdir -p gpurun_out
S=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  for m in tc tcmulti; do
    timeout 900 $S --tool $tool --print-limit 10 python tools/sanitize_small.py $m > gpurun_out/san7_${tool}_${m}.log 2>&1
    echo "== $tool $m: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san7_${tool}_${m}.log | tail -1) | $(grep -E '^(tc|tcmulti) ' gpurun_out/san7_${tool}_${m}.log | tr '\n' ' ')"
  done
done
