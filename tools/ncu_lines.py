"""Per-CUDA-source-line stall samples from `ncu -i X --page source --csv --print-source cuda,sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
fname, func, out = "?", "?", {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        func = r[1][:60]
        continue
    if r[0] == "Line No":
        continue
    if r[0] and r[0].isdigit() and len(r) > 4 and r[2] == "-":
        try:
            s = float(r[4])
        except ValueError:
            continue
        key = (func, fname, int(r[0]))
        out[key] = (out.get(key, (0, ""))[0] + s, r[1].strip()[:90])
by_func = {}
for (func, f, l), (s, src) in out.items():
    by_func.setdefault(func, []).append((s, f, l, src))
for func, lst in by_func.items():
    tot = sum(x[0] for x in lst)
    print(f"=== {func}  samples={tot:.0f}")
    for s, f, l, src in sorted(lst, reverse=True)[:top]:
        print(f"{s / tot * 100:5.1f}%  {f}:{l:<4} {src}")
