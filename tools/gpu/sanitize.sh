mkdir -p gpurun_out
S=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  echo "== $tool repro"
  timeout 300 $S --tool $tool --print-limit 4 tools/microbench/bulk_sanitizer_repro > gpurun_out/san_${tool}_repro.log 2>&1
  grep -E "OK|BAD|SUMMARY|Error:|Invalid" gpurun_out/san_${tool}_repro.log | head -5
  echo "== $tool tc"
  timeout 900 $S --tool $tool --print-limit 20 python tools/sanitize_small.py tc > gpurun_out/san_${tool}_tc.log 2>&1
  tail -4 gpurun_out/san_${tool}_tc.log
done
echo "== plain repro"; tools/microbench/bulk_sanitizer_repro
