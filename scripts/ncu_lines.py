#!/usr/bin/env python3
"""Per-CUDA-source-line instruction counts and stall samples of an ncu report
(needs -lineinfo): python ncu_lines.py REPORT [top] [kernel-regex]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
       "--launch-count", "1"]
if len(sys.argv) > 3:
    cmd += ["-k", f"regex:{sys.argv[3]}"]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
rows, fname, hdr = [], None, None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0]:
        continue
    d = dict(zip(["line", "src", "addr", "sass"] + hdr[4:], r))
    try:
        inst = float(d["Instructions Executed"] or 0)
        st = float(d["Warp Stall Sampling (All Samples)"] or 0)
    except (KeyError, ValueError):
        continue
    rows.append((fname, int(r[0]), r[1].strip(), inst, st))
ti = sum(x[3] for x in rows) or 1
ts = sum(x[4] for x in rows) or 1
print(f"total instructions {ti:.0f}, stall samples {ts:.0f}")
for f, ln, src, inst, st in sorted(rows, key=lambda x: -(x[3] / ti + x[4] / ts))[:top]:
    print(f"{f[:16]:16s}:{ln:4d} inst {100 * inst / ti:5.1f}%  stall {100 * st / ts:5.1f}%  {src[:70]}")
