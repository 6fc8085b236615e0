"""Key metrics per kernel launch of an ncu report: python tools/ncu_summary.py X.ncu-rep"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__inst_executed.avg.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
for r in rows[2:]:
    name = r[h.index("Kernel Name")].split("(")[0]
    vals = []
    for k in KEYS:
        if k in h:
            vals.append(f"{k.split('.')[0].split('__')[-1]}={r[h.index(k)]}")
    print(name, " ".join(vals))
