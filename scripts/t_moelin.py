"""Debug: one MoE (Linear, Shift) projection at (M, K) with the tc staging mode argv[3]."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
from paper_2306_06446_b200 import _lib, model as MD  # noqa: E402

M, K = int(sys.argv[1]), int(sys.argv[2])
if len(sys.argv) > 3:
    _lib.load().sa_debug_tc_stage(int(sys.argv[3]))
g = np.random.default_rng(0)
w = (g.standard_normal((K, K)) / np.sqrt(K)).astype(np.float32)
wg = (g.standard_normal((K, 2)) * 0.3).astype(np.float32)
mod = MD.MoeModule(wg, [MD.Linear(w), MD.ShiftLinearLayer(w.copy())], MD.MoeConfig())
x = torch.from_numpy(g.standard_normal((M, K)).astype(np.float32)).cuda()
y = mod.forward(x)
torch.cuda.synchronize()
print("ok", M, K, float(y.abs().sum()))
