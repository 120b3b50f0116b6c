"""Debug: time one MoE (Linear, Shift) projection at (M, K)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
from paper_2306_06446_b200 import model as MD, moe as MOE  # noqa: E402

M, K = int(sys.argv[1]), int(sys.argv[2])
g = np.random.default_rng(0)
w = (g.standard_normal((K, K)) / np.sqrt(K)).astype(np.float32)
wg = (g.standard_normal((K, 2)) * 0.3).astype(np.float32)
mod = MD.MoeModule(wg, [MD.Linear(w), MD.ShiftLinearLayer(w.copy())], MD.MoeConfig())
x = torch.from_numpy(g.standard_normal((M, K)).astype(np.float32)).cuda()
plan, _ = MOE.route_plan(x, mod.wg.value)
y = mod.forward(x, plan=plan)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(20):
    mod.forward(x, plan=plan)
e.record()
torch.cuda.synchronize()
print(f"M={M} K={K} bn={os.environ.get('SA_BN_OVERRIDE', 'auto')}: {s.elapsed_time(e) / 20 * 1000:.1f} us  sum {float(y.abs().sum()):.6g}")
