#!/usr/bin/env python3
"""Per-CTA phase timeline of the tensor-core binary attention kernel (clock64
marks, -DBAT_PROF build of binattn_tc.cu): median cycles per phase."""
import ctypes
import os
import subprocess
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2306_06446_b200 import quantize as Q  # noqa: E402

so = os.environ.get("BAT_SO", "/tmp/libbatprof.so")
if not os.path.exists(so):
    c = os.path.join(ROOT, "paper_2306_06446_b200", "csrc")
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                           "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr", "-DBAT_PROF", "-shared",
                           "-I", os.path.join(ROOT, "include"), "-I", c,
                           os.path.join(c, "binattn_tc.cu"), os.path.join(c, "lib.cu"), "-o", so])
lib = ctypes.CDLL(so)
B, n, d, h = [int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (256, 3136, 32, 1))]
g = np.random.default_rng(0)
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
M = B * n
x, k, v = (dev(g.standard_normal((M, d)).astype(np.float32)) for _ in range(3))
dw = dev((g.standard_normal((3, 3, d)) * 0.1).astype(np.float32))
cq, gq = Q.sign_hash(x, h, B)
ck, gk = Q.sign_hash(k, h, B)
out = torch.empty_like(v)
P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
buf = torch.zeros(B * 64 * 16 * 16, dtype=torch.int64, device="cuda")
lib.sa_bat_prof_set(P(buf))
args = [P(cq), P(ck), P(gq), P(gk), P(v), P(dw), P(out), ctypes.c_int64(B), ctypes.c_int64(n),
        ctypes.c_int64(d), ctypes.c_int64(h), ctypes.c_float(1e-6)]
for _ in range(3):
    assert lib.sa_bat_prof_launch(*args) == 0
torch.cuda.synchronize()
buf.zero_()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
lib.sa_bat_prof_launch(*args)
e1.record()
torch.cuda.synchronize()
print("kernel us", e0.elapsed_time(e1) * 1e3)
m = buf.cpu().numpy().reshape(-1, 16)
m = m[m[:, 7] != 0]
names = ["setup", "phaseA", "readout+sync", "exchange+planes+den", "->B", "phaseB", "dealloc"]
order = [7, 0, 1, 2, 3, 4, 5, 6]
for i in range(7):
    dlt = m[:, order[i + 1]] - m[:, order[i]]
    print(f"{names[i]:22s} median {np.median(dlt):8.0f}  p90 {np.percentile(dlt, 90):8.0f}")
for nm, c in (("first MMA issued (from start)", 9), ("sc0 planes done", 10), ("sc0 B done", 11),
              ("sc0 st wait done", 12), ("sc0 sync done", 13)):
    dlt = m[:, c] - m[:, 7]
    print(f"{nm:22s} median {np.median(dlt):8.0f}  p90 {np.percentile(dlt, 90):8.0f}")
tot = m[:, 6] - m[:, 7]
print(f"{'total':22s} median {np.median(tot):8.0f}  p90 {np.percentile(tot, 90):8.0f}  ctas {len(m)}")
