#!/usr/bin/env python3
"""GELU + bf16-split throughput probe (diagnostic): SM cycles per element for
the fused MLP's GELU pair (MUFU or FMA-pipe reciprocal) and plane split, at
several warps per SM (see sa_probe_gelu)."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_06446_b200 import _lib  # noqa: E402

lib = _lib._lib = _lib._open(_lib.DEBUG_LIB_PATH)
lib.sa_probe_gelu.argtypes = [ctypes.c_int] * 4 + [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
out = torch.zeros(1, dtype=torch.int64, device="cuda")
sink = torch.zeros(1, device="cuda")
iters = 400
for mode, name in ((0, "gelu+split"), (4, "gelu+tsplit"), (1, "gelu only"), (2, "split only"),
                   (6, "tsplit only")):
    for nf in (0, 4, 8):
        row = []
        for threads in (128, 256, 512):
            lib.sa_probe_gelu(iters, mode, nf, threads, sink.data_ptr(), out.data_ptr(),
                              torch.cuda.current_stream().cuda_stream)
            torch.cuda.synchronize()
            elems = iters * 16 * threads
            row.append(out.item() / elems)
        print(f"{name:11s} nf={nf}: cycles/element/SM " +
              "  ".join(f"{t // 32:2d} warps: {c:.3f}" for t, c in zip((128, 256, 512), row)), flush=True)
