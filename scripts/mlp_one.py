#!/usr/bin/env python3
"""One fused MoE MLP call at the PVTv2-B0 stage-1 (or, with argv[1] == 64,
stage-2) shape inside a profiler range, after a warm-up (for ncu
--profile-from-start off -k regex:mlp_kernel)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_06446_b200 import model as MD, moe as MOE  # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 32
hidden, M = (256, 802816) if d == 32 else (512, 200704)
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
mod.forward(x, plan=plan, residual=res)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
mod.forward(x, plan=plan, residual=res)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
