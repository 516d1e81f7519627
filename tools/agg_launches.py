"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) by kernel name: total us, count."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
t = collections.OrderedDict()
for r in rows[1:]:
    if r[mi] == "gpu__time_duration.sum":
        t[(r[ii], r[ki])] = float(r[vi].replace(",", ""))
agg = collections.defaultdict(lambda: [0, 0.0])
for (i, k), v in t.items():
    agg[k.split("(")[0]][0] += 1
    agg[k.split("(")[0]][1] += v
print("total us %.1f over %d launches" % (sum(v for _, v in agg.values()) / 1e3, len(t)))
for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{v / 1e3:9.1f} us {n:5d}x {k[:90]}")
