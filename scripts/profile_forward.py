#!/usr/bin/env python3
"""One-GPU forward used under ncu: builds PVTv2-B0 (bench config), runs
`--warm` eager forwards, then `--iters` more (the ones ncu should capture with
-s/-c). Never used for timing numbers."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_06446_b200 import model as MD, specs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=256)
ap.add_argument("--warm", type=int, default=1)
ap.add_argument("--iters", type=int, default=1)
ap.add_argument("--variant", default="moe")
a = ap.parse_args()
m = MD.Network(specs.pvt_v2_b0(variant=a.variant))
x = torch.from_numpy(np.random.default_rng(0).uniform(0, 1, (a.batch, 224, 224, 3)).astype(np.float32)).cuda()
for _ in range(a.warm):
    m.forward(x)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for _ in range(a.iters):
    m.forward(x)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("done")
