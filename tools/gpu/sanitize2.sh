mkdir -p gpurun_out
S=/usr/local/cuda/bin/compute-sanitizer
for iss in 0 96; do echo "== racecheck repro issuer $iss"; timeout 300 $S --tool racecheck --print-limit 4 tools/microbench/bulk_sanitizer_repro $iss 2>&1 | grep -E "OK|BAD|SUMMARY|Error:" | head -4; done
for tool in racecheck synccheck; do
  echo "== $tool lat"
  timeout 900 $S --tool $tool --print-limit 20 python tools/sanitize_small.py lat > gpurun_out/san_${tool}_lat.log 2>&1
  tail -3 gpurun_out/san_${tool}_lat.log
done
timeout 600 python -m pytest tests/test_gpu_latency.py -x -q 2>&1 | tail -2
