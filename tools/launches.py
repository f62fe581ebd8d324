"""Summarise an ncu `--metrics gpu__time_duration.sum` launch list per kernel:
launches, mean duration per launch and share of the total kernel time."""
import collections
import csv
import sys

path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/launches.csv"
rows = list(csv.reader(open(path)))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
data = rows[hi + 1:]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
         "second": 1e6, "s": 1e6}
tot = collections.OrderedDict()
cnt = collections.Counter()
allsum = 0.0
for r in data:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0].replace("void ", "")
    v = float(r[vi].replace(",", "")) * scale[r[ui]]
    tot[name] = tot.get(name, 0) + v
    cnt[name] += 1
    allsum += v
print(f"{'mean us':>9} {'launches':>8} {'share':>6}  kernel")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{v / cnt[k]:9.1f} {cnt[k]:8d} {100 * v / allsum:5.1f}%  {k[:80]}")
print(f"total kernel time {allsum:.1f} us over {sum(cnt.values())} launches")
