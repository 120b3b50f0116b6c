#!/usr/bin/env python3
"""Time the classifier head (sa_tc_linear, M = 256 images, 256 → 1000, dense)
at column-tile widths bn = 32 / 64 / 128, and check the outputs are equal."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_06446_b200 import _lib, model as MD  # noqa: E402

M, K, N = int(os.environ.get("M", 256)), 256, 1000
layer = MD.Linear((np.random.Generator(np.random.PCG64(0)).standard_normal((K, N)) * 0.05).astype(np.float32))
x = torch.randn(M, K, device="cuda")
outs = {}
for bn in (32, 64, 128):
    pk, b, kind = layer.tc_pack(bn)
    y = torch.empty(M, N, device="cuda")

    def run():
        _lib.call("sa_tc_linear", _lib.ptr(x), _lib.ptr(pk), kind, b, _lib.ptr(y), M, K, N,
                  None, 0, MD._stream())

    run()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(int(1e8))
    s.record()
    for _ in range(20):
        run()
    e.record()
    torch.cuda.synchronize()
    outs[bn] = y.clone()
    print(f"bn={b:4d}: {s.elapsed_time(e) / 20 * 1000:6.1f} us")
print("equal:", all(torch.equal(outs[32], o) for o in outs.values()))
