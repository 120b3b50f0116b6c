#!/usr/bin/env python3
"""K3 shift-Linear (tcgen05) at the PVTv2-B0 stage-1 fc1 shape, timed with the
tc GEMM debug switches (1 no A loads, 2 no C stores, 4 no MMAs)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_06446_b200 import _lib, model as MD  # noqa: E402

lib = _lib.load()
M, K, N = (int(a) for a in sys.argv[1:4])
modes = [int(a) for a in sys.argv[4:]] or [0, 1, 2, 4, 7]
g = np.random.default_rng(0)
w = (g.standard_normal((K, N)) / np.sqrt(K)).astype(np.float32)
lay = MD.ShiftLinearLayer(w)
x = torch.from_numpy(g.standard_normal((M, K)).astype(np.float32)).cuda()
y = torch.empty((M, N), dtype=torch.float32, device="cuda")
pk, bn, kind = lay.tc_pack()
for mode in modes:
    lib.sa_debug_tc_mode(mode)
    f = lambda: _lib.call("sa_tc_linear", _lib.ptr(x), _lib.ptr(pk), kind, bn, _lib.ptr(y), M, K, N,  # noqa: E731
                          None, 0, _lib.stream())
    f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10):
        f()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 10
    gbs = (M * K * 4 + M * N * 4 + K * N) / ms / 1e6
    print(f"M={M} K={K} N={N} bn={bn} mode={mode}: {ms * 1000:7.1f} us  {gbs:7.0f} GB/s")
lib.sa_debug_tc_mode(0)
