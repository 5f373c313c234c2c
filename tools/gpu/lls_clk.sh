# single-slot LLS phase cycles (NOMA_LLS_CLOCKS) and the latency breakdown
timeout 600 python tools/latency_probe.py --configs c1,c2 --lat 16 2>&1 | grep -E "NOMA_LLS|latency_us" | tail -6
