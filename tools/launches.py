"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hi]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
agg = collections.defaultdict(list)
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    agg[r[ki].split("(")[0][:70]].append(float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-3))
tot = sum(sum(v) for v in agg.values())
print(f"{'total us':>10} {'n':>4} {'avg us':>10} {'share':>6}  kernel")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{sum(v):10.1f} {len(v):4d} {sum(v)/len(v):10.1f} {100*sum(v)/tot:5.1f}%  {k}")
