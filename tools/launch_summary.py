"""Per-kernel totals and shares of an `ncu --metrics gpu__time_duration.sum --csv` launch list."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[i]
kn, mn, v = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
tot, cnt = collections.Counter(), collections.Counter()
for r in rows[i + 1:]:
    if len(r) <= v or r[mn] != "gpu__time_duration.sum":
        continue
    name = r[kn].split("(")[0].replace("void ", "")
    tot[name] += float(r[v].replace(",", ""))
    cnt[name] += 1
T = sum(tot.values())
print(f"{'kernel':58s} {'launches':>8s} {'total us':>10s} {'avg us':>8s} {'share':>6s}")
for k, t in tot.most_common():
    print(f"{k[:58]:58s} {cnt[k]:8d} {t / 1e3:10.1f} {t / cnt[k] / 1e3:8.2f} {t / T:6.3f}")
print(f"{'total':58s} {sum(cnt.values()):8d} {T / 1e3:10.1f}")
