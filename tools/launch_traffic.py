"""Per-launch time and DRAM traffic from an ncu CSV with gpu__time_duration.sum,
dram__bytes_read.sum, dram__bytes_write.sum (one row per launch and metric)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, mi, vi, ui, idi = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
d = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(",", ""))
    u = r[ui]
    v *= {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "byte": 1e-9,
          "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0}.get(u, 1.0)
    d.setdefault(int(r[idi]), {"k": r[ki]})[r[mi]] = v
tot = [0.0, 0.0, 0.0]
for i, x in d.items():
    if i < skip:
        continue
    name = x["k"].split("(")[0]
    name = name.replace("ntt16::", "").replace("<unnamed>::", "").replace("void ", "")
    t, r, w = x.get("gpu__time_duration.sum", 0), x.get("dram__bytes_read.sum", 0), x.get("dram__bytes_write.sum", 0)
    tot[0] += t
    tot[1] += r
    tot[2] += w
    print(f"{i:4d} {name[-58:]:58s} {t:7.3f} ms  r {r:6.2f}  w {w:6.2f} GB")
print(f"total {tot[0]:.3f} ms, read {tot[1]:.2f} GB, written {tot[2]:.2f} GB")
