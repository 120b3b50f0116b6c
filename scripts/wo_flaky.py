#!/usr/bin/env python3
"""Per-call device times of the fused W_O kernel at the stage-2 shape (d = 64),
to catch intermittent stalls: python scripts/wo_flaky.py [calls]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_06446_b200 import _lib, model as MD  # noqa: E402

if os.environ.get("SA_LIB"):
    _lib.LIB_PATH = os.environ["SA_LIB"]
net = MD.pvt_v2_b0()
g = np.random.default_rng(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
for si in (1, 0):
    S = net.stages[si]
    o = S.blocks[0].attn.proj["o"]
    M = 256 * S.rows
    x = torch.from_numpy(g.standard_normal((M, S.d)).astype(np.float32)).cuda()
    r = torch.from_numpy(g.standard_normal((M, S.d)).astype(np.float32)).cuda()
    o.forward(x, residual=r)
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        o.forward(x, residual=r)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ts = np.array(ts)
    print(f"d={S.d}: median {np.median(ts):.1f} us, max {ts.max():.1f}, "
          f"calls > 2x median: {int((ts > 2 * np.median(ts)).sum())}/{n}", flush=True)
