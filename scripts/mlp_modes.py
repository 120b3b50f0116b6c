#!/usr/bin/env python3
"""Fused-MLP role isolation (debug): time one stage-1 MoE MLP with producers
(2), GELU (4) or both (6) reduced to barrier traffic, plus the MMA thread's
busy cycles from the wait-site profile."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_06446_b200 import _lib, model as MD, moe as MOE  # noqa: E402
from oracle import ops  # noqa: E402

lib = _lib.debug_library().__enter__()   # the whole script runs on the debug build
lib.sa_debug_mlp_profile.argtypes = [ctypes.c_void_p]
lib.sa_debug_mlp_mode.argtypes = [ctypes.c_int]
MODES = [int(a) for a in sys.argv[1:]] or [0, 2, 4, 6, 8]
for d, hidden, M in ((32, 256, 802816), (64, 512, 200704)):
    g = ops.rng(0)
    w1 = (g.standard_normal((d, hidden)) / np.sqrt(d)).astype(np.float32)
    w2 = (g.standard_normal((hidden, d)) / np.sqrt(hidden)).astype(np.float32)
    wg = (g.standard_normal((d, 2)) * 0.3).astype(np.float32)
    mod = MD.MoeModule(wg, [MD.Mlp(MD.Linear(w1), MD.Linear(w2)),
                            MD.Mlp(MD.ShiftLinearLayer(w1.copy()), MD.ShiftLinearLayer(w2.copy()))],
                       MD.MoeConfig())
    x = torch.from_numpy(g.standard_normal((M, d)).astype(np.float32)).cuda()
    plan, _ = MOE.route_plan(x, mod.wg.value)
    for mode in MODES:
        lib.sa_debug_mlp_mode(mode)
        mod.forward(x, plan=plan)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(5):
            mod.forward(x, plan=plan)
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / 5
        buf = torch.zeros(32, dtype=torch.int64, device="cuda")
        lib.sa_debug_mlp_profile(buf.data_ptr())
        mod.forward(x, plan=plan)
        torch.cuda.synchronize()
        lib.sa_debug_mlp_profile(None)
        v = buf.cpu().numpy().astype(np.float64) / 148
        waits = v[3] + v[4] + v[5] + v[6] + v[7] + v[8]
        print(f"d={d} mode={mode}: {ms * 1000:7.1f} us   T_mma {v[13] / 1e3:7.1f}k  mma waits {waits / 1e3:7.1f}k"
              f"  gelu h_full wait {v[9] / 4 / 1e3:7.1f}k  prod a1_empty wait {v[0] / 4 / 1e3:7.1f}k")
    lib.sa_debug_mlp_mode(0)
