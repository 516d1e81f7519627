"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes per launch)."""
import csv
import sys


def load(path):
    hdr, k = None, {}
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            k.setdefault((int(d["ID"]), d["Kernel Name"]), {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    return k


if __name__ == "__main__":
    k = load(sys.argv[1])
    tot = 0.0
    for (i, name), m in sorted(k.items()):
        t = m.get("gpu__time_duration.sum", 0.0)
        rb = m.get("dram__bytes_read.sum", 0.0)
        wb = m.get("dram__bytes_write.sum", 0.0)
        tot += t
        print(f"{i:>4} {name[:58]:58s} {t / 1e3:9.1f} us  R {rb / 1e6:8.1f} MB  W {wb / 1e6:7.1f} MB  "
              f"{(rb + wb) / max(t, 1):7.0f} GB/s")
    print(f"total {tot / 1e3:.1f} us over {len(k)} launches")
