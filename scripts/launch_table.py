#!/usr/bin/env python3
"""Summarise an ncu `--metrics gpu__time_duration.sum --csv` launch list:
per-kernel count, total device time and share."""
import collections
import csv
import io
import sys


def load(path):
    lines = [ln for ln in open(path) if not ln.startswith("==")]
    return list(csv.DictReader(io.StringIO("".join(lines))))


def main(path):
    rows = load(path)
    agg = collections.OrderedDict()
    tot = 0.0
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
             "second": 1e6, "s": 1e6}
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0]
        v = float(r["Metric Value"].replace(",", "")) * scale.get(r["Metric Unit"], 1.0)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
        tot += v
    print(f"{'total_us':>10} {'launches':>8} {'share':>6}  kernel")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{t:10.1f} {n:8d} {100 * t / tot:5.1f}%  {k}")
    print(f"{tot:10.1f} {sum(n for n, _ in agg.values()):8d} 100.0%  (sum of serialized launch times)")


if __name__ == "__main__":
    main(sys.argv[1])
