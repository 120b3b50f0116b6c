#!/usr/bin/env python3
"""tcgen05.mma operand-pattern probe (diagnostic): cycles per M=128 K=16 MMA
for constant / cycling A (TMEM or shared memory) and B operands, ones vs
pseudo-random data, one CTA vs one CTA per SM (see sa_probe_mma_seq)."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_06446_b200 import _lib  # noqa: E402

lib = _lib._lib = _lib._open(_lib.DEBUG_LIB_PATH)   # the debug build, loaded alone
lib.sa_probe_mma_seq.argtypes = [ctypes.c_int] * 5 + [ctypes.c_void_p, ctypes.c_void_p]
out = torch.zeros(2, dtype=torch.int64, device="cuda")
iters = 3000
names = {0: "A,B const", 1: "A cycles", 2: "A,B cycle", 3: "A smem cycles", 4: "A,B cycle, 2 acc",
         8: "warp: A,B cycle", 9: "warp: +2 acc", 10: "warp: unrolled x6", 11: "warp: N alternates", 12: "warp: 12 MMAs per D/N", 13: "D 96/288 A 416", 14: "D 0/256 A 416",
         15: "D 96/288 A 384", 16: "2 warps, commits", 17: "1 warp, commits", 18: "2 warps, no commit", 19: "MMA + 3 warps ld/st", 20: "3 warps ld/st only"}
for grid in (1,):
    for rnd in (0,):
        for mode in (sys.argv[1:] and [int(a) for a in sys.argv[1:]]) or names:
            row = []
            for n in (32, 64, 128):
                lib.sa_probe_mma_seq(n, iters, mode, rnd, grid, out.data_ptr(),
                                     torch.cuda.current_stream().cuda_stream)
                torch.cuda.synchronize()
                row.append(out[1].item() / (iters * (2 if mode in (16, 18) else 1)))
            print(f"grid={grid:3d} rnd={rnd} {names[mode]:18s}: " +
                  "  ".join(f"N={n}: {c:6.1f}" for n, c in zip((32, 64, 128), row)), flush=True)
