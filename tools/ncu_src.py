"""Summarise an ncu --page source --csv dump: stall samples aggregated per CUDA source line."""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
rows = list(csv.reader(open(path)))
his = [i for i, r in enumerate(rows) if r and r[0] in ("Address", "# Address", "Line")]
for n, hi in enumerate(his):
    name = rows[hi - 1][1] if hi > 0 and len(rows[hi - 1]) > 1 else "?"
    end = his[n + 1] - 1 if n + 1 < len(his) else len(rows)
    hdr = rows[hi]
    data = [r for r in rows[hi + 1:end] if len(r) == len(hdr)]
    iS = hdr.index("Warp Stall Sampling (All Samples)")
    iSrc = hdr.index("Source")
    iL = hdr.index("Line") if "Line" in hdr else None
    def f(x):
        try:
            return float(x)
        except ValueError:
            return 0.0
    tot = sum(f(r[iS]) for r in data)
    print(f"=== {name[:100]}  samples={tot:.0f}")
    for r in sorted(data, key=lambda r: -f(r[iS]))[:top]:
        loc = r[iL] if iL is not None else r[0]
        print(f"{f(r[iS]) / max(tot, 1) * 100:5.1f}%  {loc:>6}  {r[iSrc].strip()[:110]}")
