# NOMA_DETECT_CLK per-role counters for C3 (cycles of CTA 0; roles: loaders,
# epilogue 1, epilogue 2, L1 issuers even/odd, L2 issuers even/odd; each
# [total, wait site 0, wait site 1, TMEM load, dot | compute, emit | store wait])
NOMA_DETECT_CLK=1 timeout 600 python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline 2>&1 | grep NOMA_DETECT_CLK | tail -1
