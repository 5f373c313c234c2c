S=/usr/local/cuda/bin/compute-sanitizer
run() { echo "== $*: $(timeout 300 $S --tool synccheck --print-limit 1 python tools/sanitize_var.py $* 2>&1 | grep -E '^ok|ERROR SUMMARY: [0-9]+ errors$|by thread|located' | tr '\n' ' ')"; }
run 1 1 64
run 1 2 64
run 3 2 64
NOMA_LAT_CLUSTER=8 run 1 2 64
NOMA_LAT_CLUSTER=4 run 1 2 64
NOMA_LAT_WARPS=16 run 1 2 64
run 1 2 32
run 1 0 64
