S=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 1200 $S --tool $tool --print-limit 10 python tools/sanitize_small.py w8 > gpurun_out/san2_${tool}_w8.log 2>&1
  echo "== $tool w8: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san2_${tool}_w8.log | tail -1) | $(grep -E '^w8 ' gpurun_out/san2_${tool}_w8.log)"
done
