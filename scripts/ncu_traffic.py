#!/usr/bin/env python3
"""Attribute an ncu launch list (dram__bytes_read/write.sum, gpu__time_duration.sum,
--csv) to the library calls recorded by profile_forward.py --record, and write
per-op DRAM traffic per launch-of-the-op (profiles/ncu_traffic.json).
    python ncu_traffic.py LAUNCH_CSV CALLS_JSON OUT_JSON"""
import collections
import csv
import io
import json
import sys

csv_path, calls_path, out_path = sys.argv[1:4]
lines = [ln for ln in open(csv_path) if not ln.startswith("==")]
rows = list(csv.DictReader(io.StringIO("".join(lines))))
per = collections.OrderedDict()
unit = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "ns": 1e-9,
        "usecond": 1e-6, "us": 1e-6, "ms": 1e-3,
        "msecond": 1e-3}
for r in rows:
    lid = int(r["ID"])
    d = per.setdefault(lid, {"kernel": r["Kernel Name"].split("(")[0]})
    d[r["Metric Name"]] = float(r["Metric Value"].replace(",", "")) * unit.get(r["Metric Unit"], 1)
launches = [per[k] for k in sorted(per)]
calls = json.load(open(calls_path))
assert sum(n for _, n in calls) == len(launches), (sum(n for _, n in calls), len(launches))
ops = collections.OrderedDict()
i = 0
for name, n in calls:
    o = ops.setdefault(name, {"calls": 0, "dram_bytes": 0.0, "time_s": 0.0, "kernels": set()})
    o["calls"] += 1
    for L in launches[i:i + n]:
        o["dram_bytes"] += L.get("dram__bytes_read.sum", 0) + L.get("dram__bytes_write.sum", 0)
        o["time_s"] += L.get("gpu__time_duration.sum", 0)
        o["kernels"].add(L["kernel"])
    i += n
out = {name: {"dram_bytes_per_call": o["dram_bytes"] / o["calls"], "calls": o["calls"],
              "ncu_time_us_per_call": 1e6 * o["time_s"] / o["calls"],
              "kernels": sorted(o["kernels"])} for name, o in ops.items()}
json.dump(out, open(out_path, "w"), indent=1)
for name, o in out.items():
    print(f"{name:24s} calls {o['calls']:3d}  dram/call {o['dram_bytes_per_call'] / 1e6:9.2f} MB  "
          f"ncu {o['ncu_time_us_per_call']:8.1f} us")
