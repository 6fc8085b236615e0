"""Group an `ncu --metrics gpu__time_duration.sum --csv` launch list into repeated call sequences
that start with a kernel whose name contains sys.argv[2]; print every `every`-th sequence."""
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) == 15]
h = rows[0]
iK, iV = h.index("Kernel Name"), h.index("Metric Value")
seq = [(r[iK].split("(")[0].replace("void ", ""), float(r[iV]) / 1000) for r in rows[1:]]
starts = [i for i, s in enumerate(seq) if sys.argv[2] in s[0]]
every = int(sys.argv[3]) if len(sys.argv) > 3 else 1
off = int(sys.argv[4]) if len(sys.argv) > 4 else 0
for j, st in enumerate(starts):
    en = starts[j + 1] if j + 1 < len(starts) else len(seq)
    if j % every == off:
        print(f"---- call {j}: {sum(s[1] for s in seq[st:en]):.1f} us")
        for name, us in seq[st:en]:
            print(f"   {name:44s} {us:9.1f} us")
