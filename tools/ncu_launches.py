#!/usr/bin/env python
"""Per-kernel averages from an `ncu --metrics a,b,c --csv` launch list.
usage: python tools/ncu_launches.py LAUNCHES.csv [OUT.txt]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
st = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[st]
ik, im, iv, iu = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = defaultdict(lambda: defaultdict(list))
units = {}
order = []
for r in rows[st + 1:]:
    if len(r) <= iv:
        continue
    k = r[ik].split("(")[0][:70]
    if k not in agg:
        order.append(k)
    agg[k][r[im]].append(float(r[iv].replace(",", "")))
    units[r[im]] = r[iu]
metrics = sorted(units)
lines = ["launches  " + "  ".join(f"{m} [{units[m]}]" for m in metrics) + "  kernel"]
for k in order:
    v = agg[k]
    n = max(len(x) for x in v.values())
    lines.append(f"{n:8d}  " + "  ".join(f"{sum(v[m]) / len(v[m]):.4g}" if v.get(m) else "-" for m in metrics)
                 + f"  {k}")
out = "\n".join(lines) + "\n"
print(out, end="")
if len(sys.argv) > 2:
    open(sys.argv[2], "w").write(out)
