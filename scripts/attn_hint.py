#!/usr/bin/env python3
"""Streaming binary attention at the PVTv2-B0 stage shapes vs the mbarrier
try_wait suspend-time hint (diagnostic, debug build): device time per call
(calls queued behind a device sleep)."""
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
lib.sa_debug_attn_hint.argtypes = [ctypes.c_uint32]
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
for B, n, d, h in ((256, 3136, 32, 1), (256, 784, 64, 2), (256, 196, 160, 5)):
    g = np.random.default_rng(0)
    dev = lambda a: torch.from_numpy(a).cuda()  # noqa: E731
    x, k, v = (dev(g.standard_normal((B * n, d)).astype(np.float32)) for _ in range(3))
    dw = dev((g.standard_normal((3, 3, d)) * 0.1).astype(np.float32))
    cq, gq = Q.sign_hash(x, h, B)
    ck, gk = Q.sign_hash(k, h, B)
    f = lambda: A.binary_core_codes(cq, ck, gq, gk, v, B, h, dw, A.EPS_NORM, "linear")  # noqa: E731
    row = []
    for hint in [int(a, 0) for a in sys.argv[1:]] or [0, 32, 256, 2000, 0x100000]:
        lib.sa_debug_attn_hint(hint)
        f()
        torch.cuda.synchronize()
        a, b = ev(), ev()
        torch.cuda._sleep(20_000_000)
        a.record()
        for _ in range(10):
            f()
        b.record()
        torch.cuda.synchronize()
        row.append(f"hint {hint}: {a.elapsed_time(b) * 100:.1f} us")
    print((B, n, d, h), "; ".join(row), flush=True)
    lib.sa_debug_attn_hint(0x100000)
