#!/usr/bin/env python3
"""Per-CUDA-source-line instruction counts and stall samples of an ncu report
(needs -lineinfo): python ncu_lines.py REPORT [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda"],
                     capture_output=True, text=True).stdout
rows = []
fname = None
lines = out.splitlines()
i = 0
while i < len(lines):
    if lines[i].startswith('"File Name"'):
        fname = lines[i].split(",", 1)[1].strip('"').split("/")[-1]
        hdr = next(csv.reader([lines[i + 1]]))
        i += 2
        while i < len(lines) and not lines[i].startswith('"File Name"'):
            r = next(csv.reader([lines[i]]))
            if len(r) == len(hdr):
                d = dict(zip(hdr, r))
                rows.append((fname, d))
            i += 1
    else:
        i += 1
ie = "Instructions Executed"
iw = "Warp Stall Sampling (All Samples)"
def f(x):
    try:
        return float(x)
    except Exception:
        return 0.0
tot_e = sum(f(d.get(ie, 0)) for _, d in rows)
tot_w = sum(f(d.get(iw, 0)) for _, d in rows)
rows.sort(key=lambda x: -f(x[1].get(iw, 0)))
print(f"total instructions {tot_e:.0f}, stall samples {tot_w:.0f}")
for fn, d in rows[:top]:
    print(f"{fn[:16]:16s}:{d['Line No']:>4} inst {100*f(d.get(ie,0))/max(tot_e,1):5.1f}%  stall {100*f(d.get(iw,0))/max(tot_w,1):5.1f}%  {d['Source'].strip()[:70]}")
