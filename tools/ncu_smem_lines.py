"""Shared-memory wavefronts (ideal / excessive) per CUDA source line of one kernel.

  ncu -i X --page source --csv --print-source cuda,sass > src.csv
  python tools/ncu_smem_lines.py src.csv k_fwd_cols [items]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
target = sys.argv[2]
items = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
hdr = [r for r in rows if r and r[0] == "Line No"][0]
iw, iwi, iwe = hdr.index("L1 Wavefronts Shared"), hdr.index("L1 Wavefronts Shared Ideal"), hdr.index("L1 Wavefronts Shared Excessive")
fname, func, out = "?", "?", {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        func = r[1]
        continue
    if target not in func or not r[0].isdigit() or len(r) <= iwe or r[2] != "-":
        continue
    try:
        w, wi, we = float(r[iw] or 0), float(r[iwi] or 0), float(r[iwe] or 0)
    except ValueError:
        continue
    if w:
        out[(fname, int(r[0]))] = (w, wi, we, r[1].strip()[:70])
tot = sum(v[0] for v in out.values())
print(f"{target}: {tot / items:.0f} shared wavefronts per item")
for k, (w, wi, we, src) in sorted(out.items(), key=lambda x: -x[1][0])[:20]:
    print(f"{k[0]}:{k[1]:4d} wf {w / items:7.0f} ideal {wi / items:7.0f} excess {we / items:6.0f}  {src}")
