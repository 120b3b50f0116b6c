#!/usr/bin/env python3
"""One-line-per-kernel summary of `ncu --set full` reports: duration, DRAM
bytes, DRAM throughput, SM / tensor-pipe activity, registers, occupancy."""
import csv
import io
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "dur",
    "dram__bytes_read.sum": "rd",
    "dram__bytes_write.sum": "wr",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram%",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm%",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor%",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed": "smem%",
    "launch__registers_per_thread": "regs",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occ%",
    "smsp__inst_executed.sum": "inst",
    "lts__t_bytes.sum": "l2B",
}


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rd = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rd[0], rd[1], rd[2:]
    for r in data:
        d = {"kernel": r[hdr.index("Kernel Name")][:60]}
        for k, short in KEYS.items():
            if k in hdr:
                i = hdr.index(k)
                d[short] = (r[i], units[i])
        yield d


for rep in sys.argv[1:]:
    for d in rows(rep):
        print(d["kernel"])
        print("   " + "  ".join(f"{k}={v[0]}{v[1]}" for k, v in d.items() if k != "kernel"))
