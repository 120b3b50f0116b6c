#!/usr/bin/env python3
"""Per-kernel totals / shares of an ncu launch list (gpu__time_duration.sum
--csv) of scripts/fwd_launches.py; load-time weight quantize / pack launches
of that first forward are excluded.
usage: python scripts/launch_summary.py launches.csv > summary.txt"""
import csv
import sys
from collections import defaultdict

LOAD_TIME = ("quantize", "pack", "elementwise", "copy")
rows = [line for line in open(sys.argv[1]) if not line.startswith("==")]
tot, cnt = defaultdict(float), defaultdict(int)
for r in csv.DictReader(rows):
    if r["Metric Name"] != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"]
    if any(s in name for s in LOAD_TIME):
        continue
    short = name.split("(")[0]
    scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(r["Metric Unit"], 1e-3)
    tot[short] += float(r["Metric Value"].replace(",", "")) * scale
    cnt[short] += 1
total = sum(tot.values())
print("# one eager PVTv2-B0 forward (B=256), ncu gpu__time_duration per launch (serialised, cold);")
print("# load-time weight quantize / pack launches of this first forward excluded")
print(f"{'total_us':>10s} {'launches':>8s} {'share':>6s}  kernel")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{tot[k]:10.1f} {cnt[k]:8d} {100 * tot[k] / total:5.1f}%  {k}")
print(f"{total:10.1f} {sum(cnt.values()):8d} 100.0%  total")
