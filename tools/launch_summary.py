#!/usr/bin/env python
"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per (kernel, grid)
count, mean duration and share of the listed device time."""
import collections
import csv
import sys


def summary(path, skip_prefixes=("at::", "void at::")):
    rows = list(csv.reader(open(path)))
    i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr, data = rows[i], rows[i + 1:]
    ki, vi, gi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Grid Size"), hdr.index("Metric Unit")
    agg = collections.defaultdict(list)
    for r in data:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        if r[ui] == "usecond":
            v *= 1000.0
        elif r[ui] == "msecond":
            v *= 1e6
        agg[(r[ki].split("(")[0].replace("void ", ""), r[gi])].append(v)
    tot = sum(sum(v) for v in agg.values())
    out = []
    for (k, g), v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        out.append((k, g, len(v), sum(v) / len(v) / 1000.0, 100.0 * sum(v) / tot))
    return out


if __name__ == "__main__":
    print(f"{'kernel':40s} {'grid':>16s} {'n':>5s} {'mean us':>9s} {'share':>7s}")
    for k, g, n, mean, share in summary(sys.argv[1]):
        print(f"{k[:40]:40s} {g:>16s} {n:5d} {mean:9.2f} {share:6.1f}%")
