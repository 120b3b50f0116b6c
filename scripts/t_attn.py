#!/usr/bin/env python3
"""Time sa_linear_binary_attn at a PVTv2-B0 stage shape (default stage 1:
B=256, n=3136, d=32, 1 head, with DWConv) for the fused single-pass kernel
(mode 0) and the multi-kernel path (mode 1)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_06446_b200 import _lib, attention as A  # noqa: E402

lib = _lib.load()
B = int(os.environ.get("B", 256))
n = int(os.environ.get("N", 3136))
d = int(os.environ.get("D", 32))
h = d // 32
g = torch.Generator(device="cuda").manual_seed(0)
cq = torch.randint(-2**31, 2**31 - 1, (B, h, n, 1), dtype=torch.int32, device="cuda", generator=g)
ck = torch.randint(-2**31, 2**31 - 1, (B, h, n, 1), dtype=torch.int32, device="cuda", generator=g)
gq = torch.rand(B, h, device="cuda") + 0.5
gk = torch.rand(B, h, device="cuda") + 0.5
v = torch.randn(B * n, d, device="cuda")
dw = torch.randn(9, d, device="cuda") * 0.1
modes = [int(a) for a in sys.argv[1:]] or [0, 1]
ref = None
for mode in modes:
    lib.sa_debug_attn_mode(mode)
    fn = lambda: A.binary_core_codes(cq, ck, gq, gk, v, B, h, dw, A.EPS_NORM, "linear")  # noqa: E731
    out = fn()
    torch.cuda.synchronize()
    if ref is None:
        ref = out.clone()
    err = float((out - ref).abs().max() / ref.abs().max())
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(int(1e8))
    s.record()
    for _ in range(10):
        fn()
    e.record()
    torch.cuda.synchronize()
    us = s.elapsed_time(e) / 10 * 1000
    alg = 2 * B * n * d // 8 + 2 * B * n * d * 4
    print(f"mode {mode}: {us:7.1f} us  {alg / us / 1e3:6.0f} GB/s (alg)  rel diff vs mode {modes[0]}: {err:.2e}")
lib.sa_debug_attn_mode(0)
