#!/usr/bin/env python3
"""W_O + LN2 + MLP router kernel (sa_fused_moe_linear_ln_route) at the
PVTv2-B0 stage-1 / stage-2 shapes: device time per call by debug role bits
(sa_debug_qkv_mode: 1 producers skip the router, 2 epilogue handshakes only,
4 no MMAs, 8 producers skip loads), debug build."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_06446_b200 import _lib, model as MD, moe as MOE  # noqa: E402

lib = _lib._lib = _lib._open(_lib.DEBUG_LIB_PATH)
lib.sa_debug_qkv_mode.argtypes = [ctypes.c_int]
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
MODES = [int(a) for a in sys.argv[1:]] or [0, 1, 2, 4, 8]
net = MD.pvt_v2_b0()
g = np.random.default_rng(0)
for si in (0, 1):
    S = net.stages[si]
    blk = S.blocks[0]
    o = blk.attn.proj["o"]
    M, d = 256 * S.rows, S.d
    x = torch.from_numpy(g.standard_normal((M, d)).astype(np.float32)).cuda()
    r = torch.from_numpy(g.standard_normal((M, d)).astype(np.float32)).cuda()
    outs = [torch.empty(M, dtype=torch.int32, device="cuda"), torch.empty(M, device="cuda"),
            torch.empty_like(x), torch.empty_like(x), torch.empty(M, dtype=torch.int32, device="cuda"),
            torch.empty(M, device="cuda")]
    args = (_lib.ptr(x), _lib.ptr(o.wg.value), _lib.ptr(o.experts[0].tc_pack(d)[0]),
            _lib.ptr(o.experts[1].tc_pack(d)[0]), _lib.ptr(r), MOE.tie_threshold(), M, d,
            _lib.ptr(outs[0]), _lib.ptr(outs[1]), _lib.ptr(outs[2]), _lib.ptr(blk.ln2.gain.value),
            _lib.ptr(blk.ln2.bias.value), 1e-5, _lib.ptr(blk.mlp.wg.value), _lib.ptr(outs[3]),
            _lib.ptr(outs[4]), _lib.ptr(outs[5]), _lib.stream())
    f = lambda: _lib.call("sa_fused_moe_linear_ln_route", *args)  # noqa: E731
    row = []
    for mode in MODES:
        lib.sa_debug_qkv_mode(mode)
        f()
        torch.cuda.synchronize()
        a, b = ev(), ev()
        torch.cuda._sleep(20_000_000)
        a.record()
        for _ in range(10):
            f()
        b.record()
        torch.cuda.synchronize()
        row.append(f"{mode}: {a.elapsed_time(b) * 100:.1f}")
    lib.sa_debug_qkv_mode(0)
    print(f"stage {si + 1} (M={M}, d={d}) us per call by mode —", "  ".join(row), flush=True)
