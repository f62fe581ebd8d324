"""Instruction-count profile of one kernel's SASS from an .ncu-rep: the
share of executed instructions and stall samples per 100-instruction window
and the hot loop's op mix.   python tools/ncu_hot.py rep.ncu-rep"""
import csv
import subprocess
import sys
from collections import Counter

out = subprocess.run(['ncu', '-i', sys.argv[1], '--page', 'source', '--csv', '--print-source',
                      'sass'], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, data = rows[1], rows[2:]
ie, src = h.index("Instructions Executed"), h.index("Source")
smp = h.index("Warp Stall Sampling (All Samples)")
cnt = [int(r[ie]) for r in data]
tot, tsm = sum(cnt), sum(int(r[smp]) for r in data)
mx = max(cnt)
hot = [i for i, c in enumerate(cnt) if c >= 0.6 * mx]
print("sass", len(data), "executed", tot, "hot", len(hot), "share %.2f" % (sum(cnt[i] for i in hot) / tot))
ops = Counter(data[i][src].split()[1] if data[i][src].strip().startswith('@') else data[i][src].split()[0]
              for i in hot)
print(ops.most_common(20))
for i in range(0, len(data), 100):
    seg = data[i:i + 100]
    s = sum(int(r[ie]) for r in seg)
    sm = sum(int(r[smp]) for r in seg)
    if s > tot * 0.01 or sm > tsm * 0.02:
        print("%5d %5.1f%% inst %5.1f%% samples  %s" % (i, 100 * s / tot, 100 * sm / tsm, seg[0][src].strip()[:50]))
