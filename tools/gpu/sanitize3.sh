S=/usr/local/cuda/bin/compute-sanitizer
R=tools/microbench/bulk_sanitizer_repro
for args in "224 16 0 256 0 2 2 4" "224 2 0 256 0 2 2 4"; do
  echo "== $args: $($R $args)"; timeout 300 $S --tool synccheck --print-limit 1000 $R $args > /tmp/s.log 2>&1; grep -E "SUMMARY" /tmp/s.log; grep -o "by thread ([0-9]*,0,0) in block ([0-9]*,0,0)" /tmp/s.log | awk '{print $NF}' | sort | uniq -c; grep -m3 -E "Missing|located|at .*repro" /tmp/s.log
done
