"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per kernel count, total, share."""
import csv
import re
import sys
from collections import defaultdict


def short(name: str) -> str:
    m = re.search(r"(k_\w+|ensi::\w+)", name)
    if m:
        return m.group(1)
    return name.split("(")[0][:60]


def main(path: str):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if r[hdr.index("Metric Name")] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}.get(r[ui], 1e-6)
        a = agg[short(r[ki])]
        a[0] += 1
        a[1] += v * scale
    tot = sum(a[1] for a in agg.values())
    print(f"{'kernel':40s} {'launches':>8s} {'total ms':>10s} {'share':>7s}")
    for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:40s} {c:8d} {t:10.3f} {100 * t / tot:6.1f}%")
    print(f"{'TOTAL':40s} {sum(a[0] for a in agg.values()):8d} {tot:10.3f}")


if __name__ == "__main__":
    main(sys.argv[1])
