#!/usr/bin/env python3
"""Summarises an `ncu --metrics gpu__time_duration.sum --csv` launch list: per-kernel count, total
and share, for the last `--steps` bench step(s) (warm-up launches are dropped by id)."""
import collections
import csv
import sys


def main(path, skip_frac=0.0):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, data = rows[0], rows[1:]
    ki, mi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in data:
        v = float(r[mi].replace(",", ""))
        v *= {"ms": 1e3, "us": 1.0, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "nsecond": 1e-3}.get(r[ui], 1.0)
        name = r[ki].split("(")[0].replace("(anonymous namespace)::", "")
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':62s} {'launches':>8s} {'total ms':>10s} {'share':>7s}")
    for n, (c, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{n[:62]:62s} {c:8d} {us / 1e3:10.3f} {us / tot * 100:6.1f}%")
    print(f"{'TOTAL':62s} {sum(v[0] for v in agg.values()):8d} {tot / 1e3:10.3f}")


if __name__ == "__main__":
    main(sys.argv[1])
