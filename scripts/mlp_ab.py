#!/usr/bin/env python3
"""Fused MoE MLP device time per call with the product library or an A/B
variant (SA_LIB=_scratch/lib_X.so): d = 32, 64, 160 PVTv2-B0 shapes."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_06446_b200 import _lib, model as MD, moe as MOE  # noqa: E402

if os.environ.get("SA_LIB"):
    _lib.LIB_PATH = os.environ["SA_LIB"]
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
out = []
for d, hidden, M in ((32, 256, 802816), (64, 512, 200704), (160, 640, 50176)):
    g = np.random.default_rng(0)
    w1 = (g.standard_normal((d, hidden)) / np.sqrt(d)).astype(np.float32)
    w2 = (g.standard_normal((hidden, d)) / np.sqrt(hidden)).astype(np.float32)
    wg = (g.standard_normal((d, 2)) * 0.3).astype(np.float32)
    mod = MD.MoeModule(wg, [MD.Mlp(MD.Linear(w1), MD.Linear(w2)),
                            MD.Mlp(MD.ShiftLinearLayer(w1.copy()), MD.ShiftLinearLayer(w2.copy()))],
                       MD.MoeConfig())
    x = torch.from_numpy(g.standard_normal((M, d)).astype(np.float32)).cuda()
    res = torch.from_numpy(g.standard_normal((M, d)).astype(np.float32)).cuda()
    plan, _ = MOE.route_plan(x, mod.wg.value)
    f = lambda: mod.forward(x, plan=plan, residual=res)  # noqa: E731
    f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        a, b = ev(), ev()
        torch.cuda._sleep(20_000_000)
        a.record()
        for _ in range(10):
            f()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 100)
    out.append(f"d={d}: {np.median(ts):.1f}")
print(os.environ.get("SA_LIB", "product"), "  ".join(out), flush=True)
