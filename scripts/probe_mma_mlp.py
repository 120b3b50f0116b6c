#!/usr/bin/env python3
"""MLP MMA-pattern probe (diagnostic): cycles per MMA of the fused MLP's issue
pattern on one CTA, for ring / accumulator / commit variants."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_06446_b200 import _lib  # noqa: E402

lib = _lib.debug_library().__enter__()   # the whole script runs on the debug build
lib.sa_probe_mma_mlp.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
out = torch.zeros(2, dtype=torch.int64, device="cuda")
chunks = 400
for np_ in (3, 1):
    for variant in (0, 8, 16, 24, 28):
        lib.sa_probe_mma_mlp(chunks, np_, variant, out.data_ptr(), torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        issue, total = out.tolist()
        nmma = chunks * 2 * 2 * (6 if np_ == 3 else 3)
        print(f"np={np_} variant={variant}: {total / nmma:6.1f} cyc/mma (issue {issue / nmma:6.1f})")
