#!/usr/bin/env python3
"""Patch embed + LayerNorm at the PVTv2-B0 stage-1 and stage-2 shapes (B=256):
device time per call for the product kernel and the GEMM path (debug build),
then one call of each stage inside a profiler range (for ncu
--profile-from-start off -k regex:embed_ln)."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_06446_b200 import _lib, model as MD  # noqa: E402

lib = _lib._lib = _lib._open(_lib.DEBUG_LIB_PATH)
lib.sa_debug_embed_mode.argtypes = [ctypes.c_int]
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
g = np.random.default_rng(0)
calls = []
for B, H, C, patch, d in ((256, 224, 3, 4, 32), (256, 56, 32, 2, 64)):
    grid = torch.from_numpy(g.uniform(0, 1, (B, H, H, C)).astype(np.float32)).cuda()
    K = patch * patch * C
    lay = MD.Linear((g.standard_normal((K, d)) / np.sqrt(K)).astype(np.float32))
    pk, bn, _ = lay.tc_pack()
    gain = torch.ones(d, device="cuda")
    bias = torch.zeros(d, device="cuda")
    side = H // patch
    y = torch.empty((B * side * side, d), device="cuda")
    f = lambda: _lib.call("sa_tc_patch_embed_ln", _lib.ptr(grid), B, H, H, C, patch, 0.5,  # noqa: E731
                          _lib.ptr(pk), bn, d, _lib.ptr(gain), _lib.ptr(bias), 1e-5, _lib.ptr(y),
                          _lib.stream())
    for mode in (0, 1):
        lib.sa_debug_embed_mode(mode)
        f()
        torch.cuda.synchronize()
        a, b = ev(), ev()
        torch.cuda._sleep(20_000_000)
        a.record()
        for _ in range(10):
            f()
        b.record()
        torch.cuda.synchronize()
        mb = (grid.numel() + y.numel()) * 4 / 1e6
        us = a.elapsed_time(b) * 100
        print(f"B={B} H={H} C={C} p={patch} d={d} mode {mode}: {us:.1f} us ({mb / us:.2f} TB/s, {mb:.0f} MB)",
              flush=True)
    lib.sa_debug_embed_mode(0)
    calls.append((f, grid, y, pk, gain, bias))
torch.cuda.cudart().cudaProfilerStart()
for c in calls:
    c[0]()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
