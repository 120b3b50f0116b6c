#!/usr/bin/env python3
"""tcgen05 GEMM path (tc_gemm_kernel) role isolation at the PVTv2-B0 stage-3 MoE
MLP (d=160, hidden 640) and stage-4 dense MLP (d=256, hidden 1024) shapes
(diagnostic, debug build): device time per call for sa_debug_tc_mode bits
(1 no A loads, 2 no C stores, 4 no MMAs, 32 no A conversion / stage stores)."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_06446_b200 import _lib, model as MD, moe as MOE  # noqa: E402

lib = _lib._lib = _lib._open(_lib.DEBUG_LIB_PATH)
lib.sa_debug_tc_mode.argtypes = [ctypes.c_int]
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    a, b = ev(), ev()
    torch.cuda._sleep(20_000_000)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / reps


MODES = [int(a) for a in sys.argv[1:]] or [0, 1, 2, 4, 5, 32, 33, 36, 37]
g = np.random.default_rng(0)
SHAPES = (("s3-moe", 160, 640, 50176, True), ("s4-dense", 256, 1024, 12544, False))
if os.environ.get("GEMM_SHAPES"):   # e.g. "deit-moe,192,768,100864,1"
    SHAPES = tuple((t.split(",")[0], *[int(v) for v in t.split(",")[1:4]], t.split(",")[4] == "1")
                   for t in os.environ["GEMM_SHAPES"].split(";"))
for label, d, hidden, M, moe in SHAPES:
    w1 = (g.standard_normal((d, hidden)) / np.sqrt(d)).astype(np.float32)
    w2 = (g.standard_normal((hidden, d)) / np.sqrt(hidden)).astype(np.float32)
    x = torch.from_numpy(g.standard_normal((M, d)).astype(np.float32)).cuda()
    res = torch.from_numpy(g.standard_normal((M, d)).astype(np.float32)).cuda()
    if moe:
        wg = (g.standard_normal((d, 2)) * 0.3).astype(np.float32)
        mod = MD.MoeModule(wg, [MD.Mlp(MD.Linear(w1), MD.Linear(w2)),
                                MD.Mlp(MD.ShiftLinearLayer(w1.copy()), MD.ShiftLinearLayer(w2.copy()))],
                           MD.MoeConfig())
        plan, _ = MOE.route_plan(x, mod.wg.value)
        f = lambda: mod.forward(x, plan=plan, residual=res)  # noqa: E731
    else:
        mlp = MD.Mlp(MD.Linear(w1), MD.Linear(w2))
        f = lambda: mlp.forward(x, residual=res)  # noqa: E731
    row = []
    for mode in MODES:
        lib.sa_debug_tc_mode(mode)
        row.append(f"{mode}: {timed(f):.1f}")
    lib.sa_debug_tc_mode(0)
    print(label, "us per call by debug mode —", "  ".join(row), flush=True)
