#!/usr/bin/env python3
"""One-GPU forward used under ncu: builds PVTv2-B0 (bench config), runs
`--warm` eager forwards, then `--iters` more between cudaProfilerStart/Stop
(capture with --profile-from-start off). With --record PATH, the library
calls of the profiled forwards are written as [op, n_launches] in order, so a
launch list can be attributed to C-ABI calls. Never used for timing numbers."""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_06446_b200 import _lib, model as MD, specs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=256)
ap.add_argument("--warm", type=int, default=1)
ap.add_argument("--iters", type=int, default=1)
ap.add_argument("--variant", default="moe")
ap.add_argument("--record", default=None)
a = ap.parse_args()
m = MD.Network(specs.pvt_v2_b0(variant=a.variant))
x = torch.from_numpy(np.random.default_rng(0).uniform(0, 1, (a.batch, 224, 224, 3)).astype(np.float32)).cuda()
for _ in range(a.warm):
    m.forward(x)
torch.cuda.synchronize()
calls = []
if a.record:
    from bench import op_key   # the bench's per-op rows (MLP split by model dim)
    orig = _lib.call

    def rec(name, *args):
        c0 = _lib.launch_count()
        r = orig(name, *args)
        calls.append([op_key(name, args), _lib.launch_count() - c0])
        return r
    _lib.call = rec
torch.cuda.cudart().cudaProfilerStart()
for _ in range(a.iters):
    m.forward(x)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
if a.record:
    json.dump(calls, open(a.record, "w"))
print("done")
