#!/usr/bin/env python3
"""tc GEMM role isolation (debug): one MoE projection at (M, K) timed with the
producers' A loads (1), the epilogue stores (2) or the MMAs (4) switched off."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_06446_b200 import _lib, model as MD, moe as MOE  # noqa: E402

lib = _lib.load()
M, K = int(sys.argv[1]), int(sys.argv[2])
g = np.random.default_rng(0)
w = (g.standard_normal((K, K)) / np.sqrt(K)).astype(np.float32)
wg = (g.standard_normal((K, 2)) * 0.3).astype(np.float32)
mod = MD.MoeModule(wg, [MD.Linear(w), MD.ShiftLinearLayer(w.copy())], MD.MoeConfig())
x = torch.from_numpy(g.standard_normal((M, K)).astype(np.float32)).cuda()
plan, _ = MOE.route_plan(x, mod.wg.value)
MODES = [int(a) for a in sys.argv[3:]] or [0, 1, 2, 3, 4, 5, 7]
for mode in MODES:
    lib.sa_debug_tc_mode(mode)
    mod.forward(x, plan=plan)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10):
        mod.forward(x, plan=plan)
    e.record()
    torch.cuda.synchronize()
    print(f"M={M} K={K} mode={mode}: {s.elapsed_time(e) / 10 * 1000:7.1f} us")
lib.sa_debug_tc_mode(0)
