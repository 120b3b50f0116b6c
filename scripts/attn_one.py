#!/usr/bin/env python3
"""One product binary-attention call at the PVTv2-B0 stage-1 shape inside a
profiler range, after a warm-up (for ncu --profile-from-start off)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_06446_b200 import attention as A, quantize as Q  # noqa: E402

B, n, d, h = (int(a) for a in (sys.argv[1:5] if len(sys.argv) > 4 else (256, 3136, 32, 1)))
g = np.random.default_rng(0)
dev = lambda a: torch.from_numpy(a).cuda()  # noqa: E731
x, k, v = (dev(g.standard_normal((B * n, d)).astype(np.float32)) for _ in range(3))
dw = dev((g.standard_normal((3, 3, d)) * 0.1).astype(np.float32))
cq, gq = Q.sign_hash(x, h, B)
ck, gk = Q.sign_hash(k, h, B)
f = lambda: A.binary_core_codes(cq, ck, gq, gk, v, B, h, dw, A.EPS_NORM, "linear")  # noqa: E731
f()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
f()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
