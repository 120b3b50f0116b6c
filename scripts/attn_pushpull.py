#!/usr/bin/env python3
"""K2a exchange A/B (debug build): push (st.async to owners / peers) vs pull
(cluster barrier + DSMEM loads), stage-1 and stage-2 PVTv2-B0 shapes, median
of 20 launches, alternating the two forms."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_06446_b200 import _lib, attention as A, quantize as Q  # noqa: E402

lib = _lib._lib = _lib._open(_lib.DEBUG_LIB_PATH)
lib.sa_debug_attn_pull.argtypes = [ctypes.c_int]
g = np.random.default_rng(0)
dev = lambda a: torch.from_numpy(a).cuda()  # noqa: E731
for B, n, d, h in ((256, 3136, 32, 1), (256, 784, 64, 2)):
    x, k, v = (dev(g.standard_normal((B * n, d)).astype(np.float32)) for _ in range(3))
    dw = dev((g.standard_normal((3, 3, d)) * 0.1).astype(np.float32))
    cq, gq = Q.sign_hash(x, h, B)
    ck, gk = Q.sign_hash(k, h, B)
    f = lambda: A.binary_core_codes(cq, ck, gq, gk, v, B, h, dw, A.EPS_NORM, "linear")  # noqa: E731
    outs, res = {}, {0: [], 1: []}
    for rep in range(3):
        for pull in (0, 1):
            lib.sa_debug_attn_pull(pull)
            outs[pull] = f().clone()
            torch.cuda.synchronize()
            ts = []
            for _ in range(20):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                f()
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b) * 1e3)
            res[pull].append(np.median(ts))
    lib.sa_debug_attn_pull(0)
    same = torch.equal(outs[0], outs[1])
    print(f"n={n} d={d}: push {np.median(res[0]):.1f} us, pull {np.median(res[1]):.1f} us, "
          f"bit-identical {same}", flush=True)
