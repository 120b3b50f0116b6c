#!/usr/bin/env python3
"""Time the binary linear attention (+DWConv) at the PVTv2-B0 / PVTv1-Tiny /
PVTv2-B2 stage shapes: product kernel (tensor cores) and, with --debug, the
CUDA-core variants of the debug library. CUDA events on the launching stream,
median of 20 launches; algorithmic bytes = V read + out write + q/k codes."""
import argparse
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_06446_b200 import _lib, attention as A, quantize as Q  # noqa: E402

if os.environ.get("SA_LIB"):   # A/B variant library (scripts/build_variant.py)
    _lib.LIB_PATH = os.environ["SA_LIB"]

SHAPES = [  # (label, B, n, d, heads)
    ("b0-s1", 256, 3136, 32, 1), ("b0-s2", 256, 784, 64, 2), ("b0-s3", 256, 196, 160, 5),
    ("t-s1", 256, 3136, 64, 1), ("t-s2", 256, 784, 128, 2), ("t-s3", 256, 196, 320, 5),
    ("deit-q", 512, 197, 192, 3),   # quadratic (Hamming) order, DeiT-T block
    ("deit-sm", 512, 197, 192, 3),  # softmax core of the exempt DeiT-T block
    ("t-s4-sm", 256, 49, 512, 8),   # PVTv1-Tiny / PVTv2-B2 stage-4 softmax core
]


def time_it(f, iters=20):
    s = _lib.stream()
    st = torch.cuda.current_stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(iters)]
    f()
    torch.cuda.synchronize()
    out = []
    for a, b in ev:
        a.record(st)
        f()
        b.record(st)
    torch.cuda.synchronize()
    out = sorted(a.elapsed_time(b) * 1e3 for a, b in ev)
    return out[len(out) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--debug", action="store_true")
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json"))).get("hbm_gbs", 6416.1)
    g = np.random.default_rng(0)
    rows = []
    for label, B, n, d, h in SHAPES:
        if a.only and a.only not in label:
            continue
        M = B * n
        dev = lambda t: torch.from_numpy(np.ascontiguousarray(t)).cuda()  # noqa: E731
        x = dev(g.standard_normal((M, d)).astype(np.float32))
        k = dev(g.standard_normal((M, d)).astype(np.float32))
        v = dev(g.standard_normal((M, d)).astype(np.float32))
        dw = dev((g.standard_normal((3, 3, d)) * 0.1).astype(np.float32))
        cq, gq = Q.sign_hash(x, h, B)
        ck, gk = Q.sign_hash(k, h, B)
        dk = d // h
        byt = 8 * M * d + 2 * M * h * ((dk + 31) // 32) * 4
        order = "quadratic" if label.endswith("-q") else "linear"
        f = lambda: A.binary_core_codes(cq, ck, gq, gk, v, B, h, dw, A.EPS_NORM, order)  # noqa
        if label.endswith("-sm"):
            order = "softmax"
            byt = 4 * M * d * 4
            f = lambda: A.softmax_core_flat(x, k, v, B, h)  # noqa
        res = {"shape": label, "B": B, "n": n, "d": d, "heads": h}
        us = time_it(f)
        res["prod_us"] = round(us, 1)
        res["prod_frac"] = round(byt / us / 1e3 / peak, 3)
        if a.debug:
            with _lib.debug_library() as lib:
                setm = {"quadratic": lib.sa_debug_ham_mode, "softmax": lib.sa_debug_softmax_tc}.get(
                    order, lib.sa_debug_attn_mode)
                setm.argtypes = [ctypes.c_int]
                modes = {"quadratic": ((1, "cuda_core"),), "softmax": ((1, "cuda_core"),)}.get(
                    order, ((3, "tc_cluster"), (5, "stream"), (1, "multi")))
                for mode, name in modes:
                    setm(mode)
                    us = time_it(f)
                    res[name + "_us"] = round(us, 1)
                setm(0)
        print(json.dumps(res), flush=True)
        rows.append(res)
        del x, k, v
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
