#!/usr/bin/env python3
"""Patch-embed role isolation (debug): the PVTv2-B0 stage-`si` patch embed at
batch 256 timed with tc debug bits (1: no A loads, 2: no C stores, 4: no MMA,
32: no split/stage stores, 16: no TMA epilogue)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_06446_b200 import _lib, model as MD  # noqa: E402

lib = _lib.load()
if os.environ.get("KQ"):
    lib.sa_debug_tc_kq(int(os.environ["KQ"]))
si = int(sys.argv[1]) if len(sys.argv) > 1 else 0
modes = [int(a) for a in sys.argv[2:]] or [0, 1, 2, 4, 32, 16, 3, 35]
m = MD.pvt_v2_b0()
S = m.stages[si]
side = [224, 56, 28, 14][si]
cin = [3, 32, 64, 160][si]
B = 256
grid = torch.rand((B, side, side, cin), device="cuda")
tok = torch.empty((B * S.rows, S.d), device="cuda")
pk, bn, _ = S.patch_embed.tc_pack()


def run():
    _lib.call("sa_tc_patch_embed", _lib.ptr(grid), B, side, side, cin, S.patch, 0.5, _lib.ptr(pk),
              bn, S.d, None, None, _lib.ptr(tok), 0)


for mode in modes:
    lib.sa_debug_tc_mode(mode)
    run()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10):
        run()
    e.record()
    torch.cuda.synchronize()
    us = s.elapsed_time(e) / 10 * 1000
    gb = (grid.numel() + tok.numel()) * 4 / us / 1e3
    print(f"stage {si} bn={bn} mode={mode:3d}: {us:7.1f} us  {gb:6.0f} GB/s")
lib.sa_debug_tc_mode(0)
