"""Summarise an ncu --metrics gpu__time_duration.sum CSV: per-kernel totals."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
tot, cnt = collections.defaultdict(float), collections.Counter()
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    name = r[ki].split("(")[0].split("<")[0].replace("void ", "")
    tot[name] += v
    cnt[name] += 1
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
grand = sum(tot.values())
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k:36s} launches={cnt[k]:4d} total={v:10.1f}us per-step={v / steps:9.1f}us "
          f"share={100 * v / grand:5.1f}%")
print(f"{'TOTAL':36s} {grand:10.1f}us per-step={grand / steps:9.1f}us")
