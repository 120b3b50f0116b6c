#!/usr/bin/env python3
"""tcgen05.mma issue/completion rate (diagnostic): cycles per M=128 K=16 MMA.
layout 0/1: one repeated operand pair (interleaved / SW64 descriptors);
layout 2: the GEMM kernels' split-precision pattern (3x3 planes, 2 k-steps)."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_06446_b200 import _lib  # noqa: E402

lib = _lib._lib = _lib._open(_lib.DEBUG_LIB_PATH)   # the debug build, loaded alone
lib.sa_probe_mma.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
out = torch.zeros(2, dtype=torch.int64, device="cuda")
for layout in (0, 2, 10, 12):
    for n in (32, 64, 96, 128, 256):
        iters = 4800
        lib.sa_probe_mma(n, iters, layout, out.data_ptr(), torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        issue, total = out.tolist()
        print(f"layout={layout} N={n:3d}: issue {issue/iters:7.1f} cyc/mma, complete {total/iters:7.1f} "
              f"cyc/mma (floor 128*N/256 = {128*n/256:.0f})")
