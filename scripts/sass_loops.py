#!/usr/bin/env python3
"""Loop bodies of one kernel in an object's SASS (backward branches): size and
opcode mix, for offline instruction-count checks.
    python sass_loops.py OBJ KERNEL_SUBSTRING"""
import collections
import re
import subprocess
import sys

obj, name = sys.argv[1], sys.argv[2]
sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", sass)
fn = next(f for f in funcs if name in f.split("\n")[0])
ins = []
for ln in fn.splitlines():
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
addr_idx = {a: i for i, (a, _) in enumerate(ins)}
for i, (a, s) in enumerate(ins):
    m = re.search(r"BRA\s+(?:\S+\s+)?(0x[0-9a-f]+)", s)
    if m:
        tgt = int(m.group(1), 16)
        if tgt < a and tgt in addr_idx:
            body = ins[addr_idx[tgt]:i + 1]
            ops = collections.Counter(x[1].split()[0] if not x[1].startswith("@") else x[1].split()[1]
                                      for x in body)
            ops = collections.Counter({k.split(".")[0]: 0 for k in ops}) + collections.Counter(
                [k.split(".")[0] for k in (x[1].split()[0] if not x[1].startswith("@") else x[1].split()[1] for x in body)])
            print(f"loop {tgt:#x}-{a:#x}: {len(body)} instr  " +
                  " ".join(f"{k}:{v}" for k, v in ops.most_common(10)))
