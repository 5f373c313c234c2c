S=/usr/local/cuda/bin/compute-sanitizer
for d in 1 33 32; do
  NOMA_LAT_DBG=$d timeout 600 $S --tool synccheck --print-limit 100000 python tools/sanitize_var.py 1 1 64 > /tmp/s.log 2>&1
  echo "dbg $d: $(grep 'ERROR SUMMARY' /tmp/s.log) $(grep -o 'by thread ([0-9]*,0,0) in block ([0-9]*,0,0)' /tmp/s.log | awk '{print $NF}' | sort | uniq -c | tr '\n' ' ') $(grep -o 'k_train_lat.cu:[0-9]*' /tmp/s.log | sort | uniq -c | tr '\n' ' ')"
done
