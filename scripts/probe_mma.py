#!/usr/bin/env python3
"""tcgen05.mma issue/completion rate (diagnostic): cycles per M=128 K=16 MMA."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_06446_b200 import _lib  # noqa: E402

lib = _lib.load()
lib.sa_probe_mma.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
out = torch.zeros(2, dtype=torch.int64, device="cuda")
for layout in (0, 1):
    for n in (32, 64, 128, 256):
        for iters in (64, 512):
            lib.sa_probe_mma(n, iters, layout, out.data_ptr(), torch.cuda.current_stream().cuda_stream)
            torch.cuda.synchronize()
            issue, total = out.tolist()
            print(f"layout={'sw64' if layout else 'intl'} N={n:3d} iters={iters:4d}: issue {issue/iters:7.1f} cyc/mma, "
                  f"complete {total/iters:7.1f} cyc/mma (floor 128*N/256 = {128*n/256:.0f})")
