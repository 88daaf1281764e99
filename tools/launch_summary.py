"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) per kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) > vi:
        v = float(r[vi].replace(",", ""))
        k = r[ki][:80]
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += v
tot = sum(v[1] for v in agg.values())
print("%6s %12s %12s %6s  %s" % ("count", "total_us", "mean_us", "share", "kernel"))
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print("%6d %12.1f %12.1f %5.1f%%  %s" % (v[0], v[1] / 1e3, v[1] / v[0] / 1e3, 100 * v[1] / tot, k))
