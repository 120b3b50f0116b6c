#!/usr/bin/env python3
"""Fused MoE MLP (K5) at the PVTv2-B0 stage-1 / stage-2 shapes (diagnostic,
debug build): for each GELU FMA-reciprocal split (sa_debug_mlp_mode = pairs of
16 on the FMA pipe) the CUDA-event time of one call (median of 20, inputs
larger than L2) and the relative error against the two-kernel tcgen05 MLP."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_06446_b200 import _lib, model as MD, moe as MOE  # noqa: E402

# the whole script runs on the debug build, loaded alone (the product library
# exports the same template kernel names)
lib = _lib._lib = _lib._open(_lib.DEBUG_LIB_PATH)
lib.sa_debug_mlp_mode.argtypes = [ctypes.c_int]
lib.sa_debug_mlp_profile.argtypes = [ctypes.c_void_p]
SITES = ["o_full(prod)", "a1_empty(prod)", "w_ring", "o_empty(fc2)", "h_empty(fc2)",
         "a1_full(fc1)", "buf_free(fc1)", "h_full(gelu)", "w_full(mma)", "T_prod", "T_fc1", "T_fc2",
         "T_gelu"]
lib.sa_debug_mlp_roles.argtypes = [ctypes.c_int]
# args: GELU FMA splits to time; "r<bits>" adds a role-isolation run (1 GELU,
# 2 producers reduced to handshakes, 4 no MMAs)
MODES = [int(a) for a in sys.argv[1:] if not a.startswith("r")] or [0, 2, 4]
ROLES = [int(a[1:]) for a in sys.argv[1:] if a.startswith("r")]
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731


def timed(fn, reps=10):
    """Device time per call: the calls are queued behind a device sleep so
    the host launch path is off the clock; returns [mean us]."""
    fn()
    torch.cuda.synchronize()
    a, b = ev(), ev()
    torch.cuda._sleep(20_000_000)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return [a.elapsed_time(b) * 1e3 / reps]
SHAPES = ((32, 256, 802816), (64, 512, 200704))
if os.environ.get("MLP_SHAPES"):   # e.g. "160,640,50176;128,1024,200704"
    SHAPES = tuple(tuple(int(v) for v in t.split(",")) for t in os.environ["MLP_SHAPES"].split(";"))
for d, hidden, M in SHAPES:
    g = np.random.default_rng(0)
    w1 = (g.standard_normal((d, hidden)) / np.sqrt(d)).astype(np.float32)
    w2 = (g.standard_normal((hidden, d)) / np.sqrt(hidden)).astype(np.float32)
    wg = (g.standard_normal((d, 2)) * 0.3).astype(np.float32)
    mod = MD.MoeModule(wg, [MD.Mlp(MD.Linear(w1), MD.Linear(w2)),
                            MD.Mlp(MD.ShiftLinearLayer(w1.copy()), MD.ShiftLinearLayer(w2.copy()))],
                       MD.MoeConfig())
    x = torch.from_numpy(g.standard_normal((M, d)).astype(np.float32)).cuda()
    res = torch.from_numpy(g.standard_normal((M, d)).astype(np.float32)).cuda()
    plan, _ = MOE.route_plan(x, mod.wg.value)
    fuse = MD.FUSE_MLP
    MD.FUSE_MLP = False
    ref = mod.forward(x, plan=plan, residual=res).clone()
    MD.FUSE_MLP = fuse
    share = float((plan.counts_dev[1].item()) / M)
    for mode in MODES:
        lib.sa_debug_mlp_mode(mode)
        y = mod.forward(x, plan=plan, residual=res)
        torch.cuda.synchronize()
        err = ((y - ref).abs().max() / (ref - res).abs().max()).item()
        ts = timed(lambda: mod.forward(x, plan=plan, residual=res))
        print(f"d={d} hidden={hidden} M={M} shift share {share:.2f} gelu_fma={mode:2d}: "
              f"{np.median(ts):7.1f} us  rel err vs two-kernel {err:.2e}", flush=True)
    for r in ROLES:
        lib.sa_debug_mlp_roles(r)
        mod.forward(x, plan=plan, residual=res)
        ts = timed(lambda: mod.forward(x, plan=plan, residual=res))
        print(f"   roles {r}: {np.median(ts):7.1f} us", flush=True)
        if r & 8:   # profile of the MMA issuer alone
            buf = torch.zeros(24, dtype=torch.int64, device="cuda")
            lib.sa_debug_mlp_profile(buf.data_ptr())
            mod.forward(x, plan=plan, residual=res)
            torch.cuda.synchronize()
            lib.sa_debug_mlp_profile(None)
            pr = buf.tolist()
            ctas = min(148, M // 128)
            print(f"      T_fc1 {pr[10] / ctas / 1e3:.1f} kcyc, T_fc2 {pr[11] / ctas / 1e3:.1f}",
                  flush=True)
        lib.sa_debug_mlp_roles(0)
    buf = torch.zeros(24, dtype=torch.int64, device="cuda")
    lib.sa_debug_mlp_profile(buf.data_ptr())
    mod.forward(x, plan=plan, residual=res)
    torch.cuda.synchronize()
    lib.sa_debug_mlp_profile(None)
    prof = buf.tolist()
    ctas = min(148, M // 128)
    # per-CTA cycles: waits are summed over the warps of a role (4 producer, 1 MMA, 8 GELU)
    warps = [4, 4, 1, 1, 1, 1, 1, 12, 2, 4, 1, 1, 12]
    print("   per CTA (kcycles): " + ", ".join(
        f"{n}={prof[i] / ctas / warps[i] / 1e3:.1f}" for i, n in enumerate(SITES)), flush=True)
    lib.sa_debug_mlp_mode(0)
