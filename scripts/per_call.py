#!/usr/bin/env python3
"""Per-call device time of one PVTv2-B0 forward (CUDA events around every
C-ABI call), with the call's algorithmic bytes and achieved GB/s. The forward
is enqueued behind a device sleep, so the host is far ahead of the GPU and the
events time the kernels, not host launch gaps."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2306_06446_b200 import model as MD, specs  # noqa: E402
from paper_2306_06446_b200.runtime import OpTimer  # noqa: E402

m = MD.Network(specs.pvt_v2_b0())
x = torch.from_numpy(np.random.default_rng(0).uniform(0, 1, (256, 224, 224, 3)).astype(np.float32)).cuda()
m.forward(x)
m.forward(x)
torch.cuda.synchronize()
t = OpTimer()
torch.cuda._sleep(int(3e8))   # ~150 ms of device time: the whole forward is queued before it runs
with t.record():
    m.forward(x)
torch.cuda.synchronize()
tot = 0.0
for name, s, e, args in t.events:
    ms = s.elapsed_time(e)
    tot += ms
    nb = bench.op_bytes(name, args)
    shape = [a for a in args if isinstance(a, int) and 1 < a < 10**7][:5]
    gbs = f"{nb / ms / 1e6:7.0f} GB/s" if nb else ""
    print(f"{name:22s} {str(shape):34s} {ms * 1000:8.1f} us {gbs}")
print(f"total {tot:.3f} ms")
