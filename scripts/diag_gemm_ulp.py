"""Accuracy of the tensor-core fp32-parity GEMM against the reference's
fp64-accumulate-then-round matmul (ref tensor.py:68-75): ulp histogram and
max |err| / rms(y) per (K, N) shape, dense and shift weights (GPU box)."""

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import ops  # noqa: E402
from paper_2306_06446_b200 import model as MD  # noqa: E402


def ulps(a, b):
    ai = a.view(np.int32).astype(np.int64)
    bi = b.view(np.int32).astype(np.int64)
    ai = np.where(ai < 0, -(ai & 0x7FFFFFFF), ai)
    bi = np.where(bi < 0, -(bi & 0x7FFFFFFF), bi)
    return np.abs(ai - bi)


def main():
    g = np.random.default_rng(0)
    M = 4096
    for K, N in ((32, 256), (64, 512), (128, 128), (160, 640), (256, 32), (320, 1280),
                 (512, 64), (512, 2048), (1280, 320), (2048, 512)):
        x = g.standard_normal((M, K)).astype(np.float32)
        w = (g.standard_normal((K, N)) / np.sqrt(K)).astype(np.float32)
        for kind in ("dense", "shift"):
            if kind == "dense":
                L = MD.Linear(w)
                wr = w
            else:
                L = MD.ShiftLinearLayer(w)
                s, p = ops.shift_quantize(w)
                wr = ops.shift_weights(s, p)
            y = L.forward(torch.from_numpy(x).cuda()).cpu().numpy()
            ref = (x.astype(np.float64) @ wr.astype(np.float64)).astype(np.float32)
            u = ulps(y, ref)
            err = np.abs(y.astype(np.float64) - ref)
            rms = np.sqrt(np.mean(ref.astype(np.float64) ** 2))
            print(f"K={K:5d} N={N:5d} {kind:5s} exact={np.mean(u == 0):.4f} <=1ulp={np.mean(u <= 1):.4f} "
                  f"max_ulp={u.max():6d} max|err|/rms={err.max() / rms:.2e} "
                  f"mean|err|/rms={err.mean() / rms:.2e}", flush=True)


if __name__ == "__main__":
    main()
