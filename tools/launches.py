"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list."""
import collections
import csv
import sys

path = sys.argv[1]
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
rows = list(csv.reader(open(path)))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, vi, ui, gi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit"), h.index("Grid Size")
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hi + 1:][skip:]:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0].split("::")[-1]
    agg[name][0] += 1
    agg[name][1] += float(r[vi].replace(",", "")) * scale[r[ui]]
tot = sum(a[1] for a in agg.values())
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:28s} n={n:5d} total={t / 1e3:9.3f} ms  avg={t / n:9.1f} us  share={t / tot:6.1%}")
print(f"total {tot / 1e3:.3f} ms over {sum(a[0] for a in agg.values())} launches")
