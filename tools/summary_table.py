"""Per-kernel table of one AMGF apply from an ncu launch list (tools/launches.py format source CSV): kernels grouped
by name, launches, total and mean time, DRAM bytes per launch, DRAM GB/s and its fraction of the measured copy
peak (MEASURED_PEAKS.json) and of 8 TB/s.  Usage: summary_table.py launches.csv"""
import json
import os
import re
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from launches import load  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6458.1)
k = load(sys.argv[1])
agg, order = {}, []
for (i, name), m in sorted(k.items()):
    short = re.sub(r"\(.*", "", name).replace("void ", "")
    if short not in agg:
        agg[short] = [0, 0.0, 0.0]
        order.append(short)
    a = agg[short]
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0.0) / 1e3
    a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
tot = sum(a[1] for a in agg.values())
print(f"| kernel | launches | total µs | share | mean µs | DRAM MB / launch | DRAM GB/s | of measured {peak:.0f} | of 8,000 |")
print("|---|---|---|---|---|---|---|---|---|")
for s in order:
    n, t, b = agg[s]
    gbs = b / max(t, 1e-9) / 1e3
    print(f"| `{s}` | {n} | {t:.1f} | {100 * t / tot:.1f} % | {t / n:.1f} | {b / n / 1e6:.1f} | {gbs:.0f} | {gbs / peak:.2f} | {gbs / 8000:.2f} |")
print(f"| total | {sum(a[0] for a in agg.values())} | {tot:.1f} | | | {sum(a[2] for a in agg.values()) / 1e6:.0f} (all) | {sum(a[2] for a in agg.values()) / tot / 1e3:.0f} | | |")
