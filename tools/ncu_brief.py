"""Key metrics of every kernel in an .ncu-rep (raw page)."""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum", "launch__grid_size",
        "launch__registers_per_thread", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h, u = r[0], r[1]
for v in r[2:]:
    print(v[h.index("Kernel Name")][:90])
    for i, k in enumerate(h):
        if k in KEYS or ("stall" in k and k.endswith("per_issue_active.ratio") and float(v[i] or 0) > 0.3):
            print(f"  {k} {v[i]} {u[i]}")
