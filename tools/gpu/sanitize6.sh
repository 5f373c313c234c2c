mkdir -p gpurun_out
S=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  for m in tc thr; do
    timeout 900 $S --tool $tool --print-limit 10 python tools/sanitize_small.py $m > gpurun_out/san2_${tool}_${m}.log 2>&1
    echo "== $tool $m: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san2_${tool}_${m}.log | tail -1) $(grep -c '^tc\|^thr' gpurun_out/san2_${tool}_${m}.log) lines"
  done
done
