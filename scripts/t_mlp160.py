#!/usr/bin/env python3
"""Stage-3 MoE MLP (d=160, hidden 640, M=50176) through the two-GEMM
tensor-core path, timed with the tc debug knobs (KQ = stage-alternation
threshold)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_06446_b200 import _lib, model as MD, moe as MOE  # noqa: E402

lib = _lib.load()
d, hidden, M = 160, 640, 50176
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
MODE = os.environ.get("MODES")
runs = [(4, int(m)) for m in MODE.split(",")] if MODE else [(int(a), 0) for a in sys.argv[1:]] or [(4, 0)]
for kq, dbg in runs:
    lib.sa_debug_tc_kq(kq)
    lib.sa_debug_tc_mode(dbg)
    mod.forward(x, plan=plan, residual=res)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(int(5e7))
    s.record()
    for _ in range(10):
        mod.forward(x, plan=plan, residual=res)
    e.record()
    torch.cuda.synchronize()
    print(f"kq={kq} dbg={dbg}: {s.elapsed_time(e) / 10 * 1000:7.1f} us")
lib.sa_debug_tc_kq(4)
lib.sa_debug_tc_mode(0)
