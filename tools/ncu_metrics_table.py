"""Table of an `ncu --metrics ... --csv` capture (one row per kernel launch, one column per metric)."""
import csv
import sys
from collections import OrderedDict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) == 15]
h = rows[0]
iI, iK, iM, iV = h.index("ID"), h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
d = OrderedDict()
for r in rows[1:]:
    d.setdefault((int(r[iI]), r[iK].split("(")[0].replace("void ", "")), OrderedDict())[r[iM]] = r[iV]
metrics = list(next(iter(d.values())).keys())
short = {m: m.replace(".avg.pct_of_peak_sustained_active", "%").replace("l1tex__data_pipe_lsu_wavefronts_mem_shared", "smem_wf")
         .replace("l1tex__", "").replace(".sum", "") for m in metrics}
print("| launch | kernel | " + " | ".join(short[m] for m in metrics) + " |")
print("|" + "---|" * (len(metrics) + 2))
for (i, k), v in d.items():
    print(f"| {i} | {k} | " + " | ".join(v.get(m, "") for m in metrics) + " |")
