"""Per-kernel-name totals of an ncu `--metrics gpu__time_duration.sum --csv` launch list.

  python tools/launch_table.py launches.csv"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
tot, cnt = defaultdict(float), defaultdict(int)
seen = set()
for r in rows[hi + 1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0].replace("void ", "")
    t = float(r[vi].replace(",", ""))
    unit = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}[r[h.index("Metric Unit")]]
    tot[name] += t * unit
    cnt[name] += 1
T = sum(tot.values())
print(f"total {T:.1f} us over {sum(cnt.values())} launches")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{tot[k]:10.1f} us {100 * tot[k] / T:5.1f}%  {cnt[k]:5d}  {k[:110]}")
