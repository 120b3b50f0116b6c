#!/usr/bin/env python3
"""Fused q/k/v input kernel (sa_ln_qkv_hash) role isolation at the PVTv2-B0
stage-1 (d=32) and stage-2 (d=64) shapes (diagnostic, debug build): device
time per call for sa_debug_qkv_mode bits (1 producers skip LN / routers,
2 epilogue handshakes only, 4 no MMAs, 8 producers skip x loads)."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_06446_b200 import _lib, model as MD, moe as MOE  # noqa: E402

PRODUCT = os.environ.get("QKV_PRODUCT") == "1"   # product library, modes ignored (for ncu)
if os.environ.get("SA_LIB"):   # A/B variant of the product library (scripts/build_variant.py)
    _lib.LIB_PATH = os.environ["SA_LIB"]
lib = _lib.load() if PRODUCT else _lib._open(_lib.DEBUG_LIB_PATH)
_lib._lib = lib
if not PRODUCT:
    lib.sa_debug_qkv_mode.argtypes = [ctypes.c_int]
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


MODES = [int(a) for a in sys.argv[1:]] or [0, 1, 2, 4, 8, 9, 3, 6, 7, 15]
net = MD.pvt_v2_b0()
g = np.random.default_rng(0)
B = 256
for si in (0, 1):
    S = net.stages[si]
    blk = S.blocks[0]
    n, d = S.rows, S.d
    x2 = torch.from_numpy(g.standard_normal((B * n, d)).astype(np.float32)).cuda()
    qkv = [blk.attn.proj[k] for k in ("q", "k", "v")]
    assert blk._fused_qkv_ok(d, n, qkv)
    M, H = B * n, blk.cfg.h
    expert_of = torch.empty((3, M), dtype=torch.int32, device="cuda")
    gate = torch.empty((3, M), dtype=torch.float32, device="cuda")
    cq = torch.empty((B, H, n, 1), dtype=torch.int32, device="cuda")
    ck = torch.empty_like(cq)
    gq = torch.empty((B, H), dtype=torch.float32, device="cuda")
    gk = torch.empty_like(gq)
    v = torch.empty((M, d), dtype=torch.float32, device="cuda")
    ws = _lib.Workspace.get(lib.sa_ln_qkv_hash_workspace(B, n, d), slot=4)
    packs = []
    for proj in qkv:
        packs += [_lib.ptr(proj.experts[0].tc_pack(d)[0]), _lib.ptr(proj.experts[1].tc_pack(d)[0])]
    args = (_lib.ptr(x2), _lib.ptr(blk.ln1.gain.value), _lib.ptr(blk.ln1.bias.value), 1e-5,
            *[_lib.ptr(p.wg.value) for p in qkv], *packs, MOE.tie_threshold(), B, n, d,
            _lib.ptr(expert_of), _lib.ptr(gate), _lib.ptr(cq), _lib.ptr(ck), _lib.ptr(gq),
            _lib.ptr(gk), _lib.ptr(v), _lib.ptr(ws), ws.numel(), _lib.stream())
    f = lambda: _lib.call("sa_ln_qkv_hash", *args)  # noqa: E731
    if PRODUCT:
        f()
        f()
        torch.cuda.synchronize()
        print(f"stage {si + 1}: {timed(f):.1f} us", flush=True)
        continue
    row = []
    for mode in MODES:
        lib.sa_debug_qkv_mode(mode)
        row.append(f"{mode}: {timed(f):.1f}")
    lib.sa_debug_qkv_mode(0)
    print(f"stage {si + 1} (M={M}, d={d}) us per call by qkv debug mode —", "  ".join(row), flush=True)
