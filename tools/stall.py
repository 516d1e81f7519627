"""Top warp-stall SASS lines of an `ncu --page source --csv --print-source sass` export."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ci = {k: i for i, k in enumerate(h)}
key = "Warp Stall Sampling (All Samples)"
data = []
for idx, r in enumerate(rows[2:]):
    if r and r[0] == "Kernel Name":
        break  # first kernel of the export only
    if len(r) <= ci[key] or not r[ci[key]].replace(".", "").isdigit():
        continue
    data.append((float(r[ci[key]] or 0), idx, r[ci["Source"]].strip()))
tot = sum(d[0] for d in data)
print("total samples", tot, "instructions", len(data))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
for d in sorted(data, key=lambda x: -x[0])[:n]:
    print(f"{d[0]:7.0f} {100 * d[0] / tot:5.1f}% {d[1]:5d} {d[2][:100]}")
