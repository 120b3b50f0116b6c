#!/usr/bin/env python3
"""Per-SASS-instruction execution counts and stall samples for one kernel of
an ncu report: python ncu_src.py REPORT KERNEL_REGEX [min_share]"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
thr = float(sys.argv[3]) if len(sys.argv) > 3 else 0.05
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                      "--launch-count", "1"], capture_output=True, text=True).stdout.splitlines()
start = [i for i, ln in enumerate(out) if ln.startswith('"Address"')][0]
rows = list(csv.reader(out[start:]))
hdr = rows[0]
ia, isrc = hdr.index("Address"), hdr.index("Source")
ie, iw = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
body = [r for r in rows[1:] if len(r) == len(hdr) and r[ie].replace(".", "").isdigit()]
tot = sum(float(r[iw] or 0) for r in body)
ti = sum(float(r[ie] or 0) for r in body)
mx = max(float(r[ie] or 0) for r in body)
print(f"total warp-instructions {ti:.0f}")
for r in body:
    e, w = float(r[ie] or 0), float(r[iw] or 0)
    if e >= thr * mx or w > 0.01 * tot:
        print(f"{r[ia][-5:]} {int(e):>10} {100 * w / max(tot, 1):5.1f}%  {r[isrc][:72]}")
