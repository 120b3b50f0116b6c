#!/usr/bin/env python3
"""Top stall-sampled SASS instructions of an ncu report (source page)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True,
                     text=True).stdout.splitlines()
rows = list(csv.reader(out[1:]))
hdr = rows[0]
ia, isrc, iw = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
data = []
tot = 0
for r in rows[1:]:
    try:
        w = float(r[iw] or 0)
    except ValueError:
        continue
    tot += w
    data.append((w, r[ia], r[isrc]))
data.sort(reverse=True)
for w, a, s in data[:top]:
    print(f"{100 * w / max(tot, 1):5.1f}%  {a}  {s[:110]}")
