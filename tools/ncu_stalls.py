"""Stall-reason and pipe summary of one kernel in an ncu report."""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h, v = r[0], r[2]
items = []
for k, val in zip(h, v):
    if "smsp__average_warps_issue_stalled_" in k and k.endswith("_per_issue_active.ratio"):
        try:
            items.append((float(val), k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
        except ValueError:
            pass
print("stalls per issued instruction:", ", ".join(f"{n} {x:.2f}" for x, n in sorted(items, reverse=True)[:9]))
for k in ["gpu__time_duration.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
          "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
          "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__inst_executed.sum",
          "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
          "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active"]:
    if k in h:
        print(k, r[1][h.index(k)], v[h.index(k)])
