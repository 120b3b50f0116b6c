#!/usr/bin/env python3
"""SASS opcode histogram (executed warp-instructions) and per-address hot spots
of an ncu report: python ncu_ops.py REPORT [top]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True,
                     text=True).stdout.splitlines()
start = [i for i, ln in enumerate(out) if ln.startswith('"Address"')][0]
rows = list(csv.reader(out[start:]))
hdr = rows[0]
ia, isrc, ie = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed")
hist = collections.Counter()
tot = 0
for r in rows[1:]:
    if len(r) != len(hdr):
        continue
    try:
        e = float(r[ie] or 0)
    except ValueError:
        continue
    src = r[isrc].strip()
    toks = src.split()
    if toks and toks[0].startswith("@"):
        toks = toks[1:]
    op = toks[0].split(".")[0] if toks else "?"
    hist[op] += e
    tot += e
print(f"total warp-instructions {tot:.0f}")
for op, e in hist.most_common(top):
    print(f"  {op:12s} {e:14.0f} {100 * e / tot:5.1f}%")
