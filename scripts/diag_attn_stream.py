#!/usr/bin/env python3
"""Streaming binary-attention kernel against the oracle and the tensor-core
cluster kernel (diagnostic): per shape, max error, the tokens / heads / images
that differ, and run-to-run determinism."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_06446_b200 import _lib, attention as A  # noqa: E402
from oracle import ops  # noqa: E402

lib = _lib._lib = _lib._open(_lib.DEBUG_LIB_PATH)
lib.sa_debug_attn_mode.argtypes = [ctypes.c_int]
for (B, n, d, h, with_dw, seed) in [(2, 3136, 32, 1, True, 7 + 3136), (3, 3136, 32, 1, True, 11 + 3136 + 32),
                                    (2, 784, 64, 2, True, 7 + 784), (2, 196, 160, 5, True, 7 + 196)]:
    g = ops.rng(seed)
    q, kk, v = (g.standard_normal((B * n, d)).astype(np.float32) for _ in range(3))
    dw = (g.standard_normal((3, 3, d)) * 0.1).astype(np.float32) if with_dw else None
    dev = lambda a: torch.from_numpy(a).cuda()  # noqa: E731
    args = (dev(q), dev(kk), dev(v), B, h, dev(dw) if with_dw else None)
    runs = []
    for _ in range(3):
        lib.sa_debug_attn_mode(5)
        runs.append(A.binary_core(*args).cpu().numpy())
    lib.sa_debug_attn_mode(3)
    tc = A.binary_core(*args).cpu().numpy()
    lib.sa_debug_attn_mode(0)
    prod = runs[0]
    det = all(np.array_equal(r, prod) for r in runs)
    diff = np.abs(prod - tc).reshape(B, n, h, d // h).max(axis=3)
    bad = np.argwhere(diff > 1e-4)
    print((B, n, d, h), "deterministic", det, "max |prod - tc|", diff.max(), "bad", len(bad), flush=True)
    if len(bad):
        toks = sorted(set(int(t) for _, t, _ in bad))
        side = int(np.ceil(np.sqrt(n)))
        print("  tokens", toks[:10], "...", toks[-5:], "rows", sorted(set(t // side for t in toks))[:20],
              "heads", sorted(set(int(x) for _, _, x in bad)), "images", sorted(set(int(x) for x, _, _ in bad)))
