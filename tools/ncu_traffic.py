"""DRAM traffic per launch of each kernel class from an `ncu --set full` report.

  python tools/ncu_traffic.py FRAMES_PER_LAUNCH SOURCE_NAME REPORT.ncu-rep [...] > profiles/ncu_traffic.json

bench.py reads profiles/ncu_traffic.json for the `traffic` field of its roofline object.
"""
import csv
import io
import json
import re
import subprocess
import sys

CLASSES = {"fwd_rows": r"k_fwd_rows", "fwd_cols": r"k_fwd_cols|k_toep_cols", "adj_cols": r"k_adj_cols",
           "adj_rows": r"k_adj_rows"}
frames, source = int(sys.argv[1]), sys.argv[2]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
acc = {}
allrows = []
for rep in sys.argv[3:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    allrows += [(rows[0], rows[1], r) for r in rows[2:]]
for h, units, r in allrows:
    name = r[h.index("Kernel Name")]
    cls = next((c for c, pat in CLASSES.items() if re.search(pat, name)), None)
    if cls is None:
        continue
    b = 0.0
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = h.index(k)
        b += float(r[i].replace(",", "")) * scale[units[i]]
    t = float(r[h.index("gpu__time_duration.sum")].replace(",", ""))
    a = acc.setdefault(cls, [0.0, 0.0, 0, name.split("(")[0]])
    a[0] += b
    a[1] += t
    a[2] += 1
res = {"source": source, "frames_per_launch": frames,
       "note": "cold-cache (ncu --cache-control all) dram__bytes_read.sum + dram__bytes_write.sum, mean per launch",
       "kernels": {c: {"kernel": v[3], "dram_bytes_per_launch": v[0] / v[2], "frames_per_launch": frames,
                       "gpu_time_us_per_launch": v[1] / v[2], "launches": v[2]} for c, v in acc.items()}}
print(json.dumps(res, indent=1))
