"""Sum an ncu launch list (gpu__time_duration.sum CSV) per kernel name."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
div = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
d = collections.defaultdict(list)
for r in rows[hi + 1:]:
    if len(r) > vi:
        d[r[ki][:70]].append(float(r[vi].replace(",", "")))
tot = sum(sum(v) for v in d.values())
for k, v in sorted(d.items(), key=lambda x: -sum(x[1])):
    print(f"{sum(v) / 1e3 / div:9.1f} us/unit {len(v) / div:6.1f} launches {sum(v) / len(v) / 1e3:8.1f} us  {k}")
print(f"total {tot / 1e3 / div:.1f} us per unit")
