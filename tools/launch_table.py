"""Summarise an ncu --csv launch list (gpu__time_duration.sum): per-kernel time and share."""
import csv
import re
import sys
from collections import OrderedDict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = OrderedDict()
for r in rows[1:]:
    name = re.sub(r"\(.*", "", r[ki].replace("(anonymous namespace)::", "").replace("<unnamed>::", ""))
    name = name.replace("void ", "")
    v = float(r[vi].replace(",", "")) * {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(r[ui], 1e-3)
    c, t = agg.get(name, (0, 0.0))
    agg[name] = (c + 1, t + v)
tot = sum(t for _, t in agg.values())
print(f"{'kernel':60s} {'n':>3s} {'us':>10s} {'share':>7s}")
for k, (c, t) in agg.items():
    print(f"{k[:60]:60s} {c:3d} {t:10.1f} {100 * t / tot:6.2f}%")
print(f"{'total':60s} {'':3s} {tot:10.1f}")
