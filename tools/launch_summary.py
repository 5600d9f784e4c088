"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: python tools/launch_summary.py file.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, mi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hi + 1:]:
    if len(r) <= mi:
        continue
    us = float(r[mi].replace(",", "")) * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6, "second": 1e6}.get(r[ui], 1.0)
    a = agg[r[ki].split("(")[0][:60]]
    a[0] += 1
    a[1] += us
tot = sum(v for _, v in agg.values())
for k, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:60s} n={n:5d} mean={us / n:9.2f} us total={us / 1000:9.3f} ms share={us / tot:6.1%}")
