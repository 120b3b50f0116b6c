#!/usr/bin/env python3
"""Time sa_softmax_attn at the PVTv2-B0 stage-4 shape (B=256, n=49, d=256,
8 heads) for the generic kernel and the dk=32 kernel at QB = 2/4/8."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_06446_b200 import _lib, attention as A  # noqa: E402

lib = _lib.load()
B, n, d, h = 256, 49, 256, 8
q, k, v = (torch.randn(B * n, d, device="cuda") for _ in range(3))
for name, gen, qb in (("generic", 1, 4), ("qb2", 0, 2), ("qb4", 0, 4), ("qb8", 0, 8)):
    lib.sa_debug_softmax_generic(gen)
    lib.sa_debug_softmax_qb(qb)
    A.softmax_core_flat(q, k, v, B, h)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20):
        A.softmax_core_flat(q, k, v, B, h)
    e.record()
    torch.cuda.synchronize()
    us = s.elapsed_time(e) / 20 * 1000
    print(f"{name:8s} {us:7.1f} us  {4 * q.numel() * 4 / us / 1e3:6.0f} GB/s")
lib.sa_debug_softmax_generic(0)
lib.sa_debug_softmax_qb(4)
