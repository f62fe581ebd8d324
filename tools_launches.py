"""Summarise an ncu --metrics gpu__time_duration.sum launch list per kernel."""
import collections
import csv
import sys

path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/launches.csv"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
rows = list(csv.reader(open(path)))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
data = rows[hi + 1:]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6}
tot = collections.OrderedDict()
cnt = collections.Counter()
allsum = 0.0
for r in data:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0].replace("void ", "")
    v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    tot[name] = tot.get(name, 0) + v
    cnt[name] += 1
    allsum += v
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{v / steps:9.1f} us/step  x{cnt[k] // steps:2d}  {100 * v / allsum:5.1f}%  {k[:80]}")
print(f"total per step {allsum / steps:.1f} us")
