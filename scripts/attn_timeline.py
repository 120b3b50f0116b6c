#!/usr/bin/env python3
"""Streaming binary-attention event timeline of CTA 0 (debug build): per tile
the clock of pass-A conversion start / end, pass-A MMA issue, pass-B epilogue
start / end and MMA issue, producer row issues; relative to the first event."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_06446_b200 import _lib, attention as A, quantize as Q  # noqa: E402

lib = _lib._lib = _lib._open(_lib.DEBUG_LIB_PATH)
lib.sa_debug_attn_mode.argtypes = [ctypes.c_int]
lib.sa_debug_attn_mode(5)   # the streaming kernel
lib.sa_debug_attn_timeline.argtypes = [ctypes.c_void_p]
B, n, d, h = 256, 3136, 32, 1
g = np.random.default_rng(0)
dev = lambda a: torch.from_numpy(a).cuda()  # noqa: E731
x, k, v = (dev(g.standard_normal((B * n, d)).astype(np.float32)) for _ in range(3))
dw = dev((g.standard_normal((3, 3, d)) * 0.1).astype(np.float32))
cq, gq = Q.sign_hash(x, h, B)
ck, gk = Q.sign_hash(k, h, B)
f = lambda: A.binary_core_codes(cq, ck, gq, gk, v, B, h, dw, A.EPS_NORM, "linear")  # noqa: E731
f()
tl = torch.zeros(9 * 256, dtype=torch.int64, device="cuda")
lib.sa_debug_attn_timeline(tl.data_ptr())
f()
torch.cuda.synchronize()
lib.sa_debug_attn_timeline(None)
t = tl.view(9, 256).cpu().numpy()
t0 = t[6, 0]
names = ["A conv start", "A conv end", "A mma", "switch", "B epi start", "B epi end", "row issue", "B mma",
         "A rows+sync"]
for e in range(9):
    row = t[e, :60]
    row = [int(x - t0) if x else None for x in row]
    print(f"{names[e]:12s}", row[:60])
