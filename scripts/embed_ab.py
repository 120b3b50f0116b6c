#!/usr/bin/env python3
"""Patch embed + LayerNorm (sa_tc_patch_embed_ln) device time per call at the
PVTv2-B0 stage-1 / stage-2 shapes with the product library or an A/B variant
(SA_LIB=_scratch/lib_X.so)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_06446_b200 import _lib, model as MD  # noqa: E402

if os.environ.get("SA_LIB"):
    _lib.LIB_PATH = os.environ["SA_LIB"]
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
g = np.random.default_rng(0)
out = []
for B, H, C, patch, d in ((256, 224, 3, 4, 32), (256, 56, 32, 2, 64)):
    grid = torch.from_numpy(g.uniform(0, 1, (B, H, H, C)).astype(np.float32)).cuda()
    K = patch * patch * C
    lay = MD.Linear((g.standard_normal((K, d)) / np.sqrt(K)).astype(np.float32))
    pk, bn, _ = lay.tc_pack()
    gain = torch.ones(d, device="cuda")
    bias = torch.zeros(d, device="cuda")
    side = H // patch
    y = torch.empty((B * side * side, d), device="cuda")
    f = lambda: _lib.call("sa_tc_patch_embed_ln", _lib.ptr(grid), B, H, H, C, patch, 0.5,  # noqa: E731
                          _lib.ptr(pk), bn, d, _lib.ptr(gain), _lib.ptr(bias), 1e-5, _lib.ptr(y),
                          _lib.stream())
    f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
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
