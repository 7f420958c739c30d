#!/usr/bin/env python
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): per kernel count,
mean/min device time, and share of the total (cold-cache, serialised: compare SHARES)."""
import collections
import csv
import sys


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in rows[1:]:
        name = r[ki].split("(")[0].replace("void ", "").split("::")[-1]
        agg[name].append(float(r[vi].replace(",", "")) / 1e3)
    tot = sum(sum(v) for v in agg.values())
    print(f"{'kernel':28s} {'n':>5s} {'mean us':>9s} {'min us':>8s} {'share':>7s}")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k:28s} {len(v):5d} {sum(v) / len(v):9.2f} {min(v):8.2f} {100 * sum(v) / tot:6.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
