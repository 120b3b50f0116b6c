#!/usr/bin/env python3
"""Time sa_ln_route / sa_moe_route at the PVTv2-B0 stage-3 shape (M=50176,
d=160) with 1 and 3 routers."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_06446_b200 import moe as MOE  # noqa: E402

M, d = int(os.environ.get("M", 50176)), int(os.environ.get("D", 160))
x = torch.randn(M, d, device="cuda")
gain = torch.ones(d, device="cuda")
bias = torch.zeros(d, device="cuda")
wgs = [torch.randn(d, 2, device="cuda") * 0.3 for _ in range(3)]


def timeit(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(int(1e8))
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1000


from paper_2306_06446_b200 import _lib  # noqa: E402
for rt in (1, 2):   # rows per thread of the 8-lanes-per-row kernel (d >= 96)
    _lib.load().sa_debug_oct_rows(rt)
    for nr in (1, 3):
        us = timeit(lambda: MOE.ln_route_plans(x, gain, bias, wgs[:nr]))
        print(f"rt={rt} ln_route M={M} d={d} nr={nr}: {us:7.1f} us")
    us = timeit(lambda: MOE.route_plan(x, wgs[0]))
    print(f"rt={rt} moe_route M={M} d={d}: {us:7.1f} us")
_lib.load().sa_debug_oct_rows(2)
