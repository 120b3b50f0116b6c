#!/usr/bin/env python3
"""Cycle profile of the fused MLP kernel's wait sites (debug): runs one
stage-1 MoE MLP at bench size and prints cycles per site per warp."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_06446_b200 import _lib, model as MD  # noqa: E402
from oracle import ops  # noqa: E402

SITES = ["prod a1_empty", "w1stream empty", "w2stream empty", "mma a1_full", "mma w1_full",
         "mma h_empty(fc1)", "mma o_empty", "mma w2_full", "mma h_empty(fc2)", "gelu h_full",
         "gelu a2_empty", "epi o_full", "T prod", "T mma", "T gelu", "mma issue fc1", "mma issue fc2"]
lib = _lib.debug_library().__enter__()   # the whole script runs on the debug build
lib.sa_debug_mlp_profile.argtypes = [ctypes.c_void_p]
lib.sa_debug_mlp_mode.argtypes = [ctypes.c_int]
MODE = int(sys.argv[1]) if len(sys.argv) > 1 else 0
lib.sa_debug_mlp_mode(MODE)
for d, hidden in ((32, 256), (64, 512)):
    M = 802816 if d == 32 else 200704
    g = ops.rng(0)
    w1 = (g.standard_normal((d, hidden)) / np.sqrt(d)).astype(np.float32)
    w2 = (g.standard_normal((hidden, d)) / np.sqrt(hidden)).astype(np.float32)
    wg = (g.standard_normal((d, 2)) * 0.3).astype(np.float32)
    mod = MD.MoeModule(wg, [MD.Mlp(MD.Linear(w1), MD.Linear(w2)),
                            MD.Mlp(MD.ShiftLinearLayer(w1.copy()), MD.ShiftLinearLayer(w2.copy()))],
                       MD.MoeConfig())
    x = torch.from_numpy(g.standard_normal((M, d)).astype(np.float32)).cuda()
    mod.forward(x)
    buf = torch.zeros(32, dtype=torch.int64, device="cuda")
    lib.sa_debug_mlp_profile(buf.data_ptr())
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    mod.forward(x)
    e.record()
    torch.cuda.synchronize()
    lib.sa_debug_mlp_profile(None)
    v = buf.cpu().numpy().astype(np.float64)
    ncta = 148
    print(f"d={d} hidden={hidden} M={M}  forward(route+mlp) {s.elapsed_time(e):.3f} ms   share1={mod.last_plan.share(1):.2f}")
    warps = {"prod": 4, "w1": 1, "w2": 1, "mma": 1, "gelu": 8, "epi": 8}
    for i, name in enumerate(SITES):
        key = name.split()[0]
        w = {"prod": 4, "w1stream": 1, "w2stream": 1, "mma": 1, "gelu": 4, "epi": 4, "T": 1}[key]
        if name.startswith("T "):
            w = {"T prod": 4, "T mma": 1, "T gelu": 8}[name]
        print(f"  {name:22s} {v[i] / ncta / w / 1e3:10.1f} kcycles/warp")
