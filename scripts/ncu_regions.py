#!/usr/bin/env python3
"""Stall samples of one kernel's source page grouped into address regions cut
at the SYNCS wait / arrive instructions (to attribute stalls to warp roles):
python ncu_regions.py SOURCE_CSV [top_n]"""
import csv
import sys

out = open(sys.argv[1]).read().splitlines()
top = int(sys.argv[2]) if len(sys.argv) > 2 else 12
start = [i for i, ln in enumerate(out) if ln.startswith('"Address"')][0]
rows = list(csv.reader(out[start:]))
h = rows[0]
ia, isrc, ie, iw = (h.index("Address"), h.index("Source"), h.index("Instructions Executed"),
                    h.index("Warp Stall Sampling (All Samples)"))
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
body = [r for r in rows[1:] if len(r) == len(h) and r[ie].replace(".", "").isdigit()]
tot = sum(float(r[iw] or 0) for r in body)
print(f"samples {tot:.0f}, warp-instructions {sum(float(r[ie]) for r in body):.0f}")
for r in body:
    w = float(r[iw] or 0)
    src = r[isrc]
    mark = "SYNCS" in src or "EXIT" in src or "UTCHMMA" in src[:20] or "UTCBAR" in src
    if w > 0.004 * tot or ("SYNCS" in src):
        rs = sorted(((float(r[h.index(c)] or 0), c[6:]) for c in reasons), reverse=True)[:2]
        print(f"{r[ia][-5:]} {int(float(r[ie])):>9} {100 * w / tot:5.1f}%  {src[:64]:64s} "
              + " ".join(f"{c}:{v:.0f}" for v, c in rs if v > 0))
