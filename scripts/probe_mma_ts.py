#!/usr/bin/env python3
"""A-in-TMEM tcgen05.mma probe (diagnostic): checks the TMEM A-operand layout
against torch and measures cycles per M=128 K=16 MMA with A in TMEM."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_06446_b200 import _lib  # noqa: E402

lib = _lib._lib = _lib._open(_lib.DEBUG_LIB_PATH)   # the debug build, loaded alone
lib.sa_probe_mma_ts.argtypes = [ctypes.c_int, ctypes.c_int] + [ctypes.c_void_p] * 5
torch.manual_seed(0)
out = torch.zeros(2, dtype=torch.int64, device="cuda")
for n in (32, 64, 96, 128, 256):
    a = torch.randint(-4, 5, (128, 16), device="cuda").to(torch.bfloat16)
    b = torch.randint(-4, 5, (n, 16), device="cuda").to(torch.bfloat16)
    d = torch.zeros(128, n, device="cuda")
    lib.sa_probe_mma_ts(n, 0, a.data_ptr(), b.data_ptr(), d.data_ptr(), out.data_ptr(),
                        torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    ref = a.float() @ b.float().T
    err = (d - ref).abs().max().item()
    iters = 4096
    lib.sa_probe_mma_ts(n, iters, a.data_ptr(), b.data_ptr(), d.data_ptr(), out.data_ptr(),
                        torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    issue, total = out.tolist()
    print(f"N={n:3d}: layout max|err| {err:g}; issue {issue/iters:6.1f} complete {total/iters:6.1f} cyc/mma "
          f"(floor {128*n/256:.0f})")
