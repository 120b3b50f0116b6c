#!/usr/bin/env python3
"""Time the fused attention output projection (sa_fused_moe_linear: router +
both experts + residual) at the PVTv2-B0 stage-1 / stage-2 shapes (B = 256)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_06446_b200 import _lib, model as MD  # noqa: E402

if os.environ.get("SA_LIB"):   # A/B variant library (scripts/build_variant.py)
    _lib.LIB_PATH = os.environ["SA_LIB"]

ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
net = MD.pvt_v2_b0()
g = np.random.default_rng(0)
for si in (0, 1):
    S = net.stages[si]
    o = S.blocks[0].attn.proj["o"]
    M = 256 * S.rows
    x = torch.from_numpy(g.standard_normal((M, S.d)).astype(np.float32)).cuda()
    r = torch.from_numpy(g.standard_normal((M, S.d)).astype(np.float32)).cuda()
    f = lambda: o.forward(x, residual=r)  # noqa: E731
    f()
    torch.cuda.synchronize()
    a, b = ev(), ev()
    torch.cuda._sleep(20_000_000)
    a.record()
    for _ in range(10):
        f()
    b.record()
    torch.cuda.synchronize()
    print(f"W_O stage {si + 1} (M={M}, d={S.d}): {a.elapsed_time(b) * 100:.1f} us", flush=True)
