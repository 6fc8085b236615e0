"""Top SASS instructions of an `ncu --page source --csv` dump with their stall-reason breakdown."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
hdr = rows[hi]
data = [r for r in rows[hi + 1:] if len(r) == len(hdr)]
iS = hdr.index("Warp Stall Sampling (All Samples)")
st = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


tot = sum(f(r[iS]) for r in data)
agg = {}
for r in data:
    for i in st:
        agg[hdr[i]] = agg.get(hdr[i], 0) + f(r[i])
print("total", int(tot), sorted(((int(v), k) for k, v in agg.items()), reverse=True)[:8])
for r in sorted(data, key=lambda r: -f(r[iS]))[:top]:
    rs = sorted(((f(r[i]), hdr[i][6:]) for i in st), reverse=True)[:3]
    print(f"{f(r[iS]) / tot * 100:5.1f}%  {r[1].strip()[:60]:60s} " + " ".join(f"{n}={int(v)}" for v, n in rs if v))
