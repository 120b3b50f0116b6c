#!/usr/bin/env python3
"""Time sa_sign_hash at the PVTv2-B0 stage-3 / stage-2 / stage-4 shapes."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_06446_b200 import quantize as Q
for B, n, d, h in ((256, 196, 160, 5), (256, 784, 64, 2), (256, 49, 256, 8)):
    x = torch.randn(B * n, d, device="cuda")
    Q.sign_hash(x, h, B); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(int(5e7)); s.record()
    for _ in range(20): Q.sign_hash(x, h, B)
    e.record(); torch.cuda.synchronize()
    print(B, n, d, h, f"{s.elapsed_time(e) / 20 * 1000:.1f} us")
