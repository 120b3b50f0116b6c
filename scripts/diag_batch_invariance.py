"""Is each library call batch invariant? Runs a model on a batch and on a
sub-batch and compares every C-ABI call's outputs (by call order) for the
shared images. Prints the first calls whose outputs differ (GPU box).

    python scripts/diag_batch_invariance.py [pvt_small|pvt_v2_b0] [B] [lo] [hi]
"""

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import ops  # noqa: E402
from paper_2306_06446_b200 import _lib, specs  # noqa: E402
from paper_2306_06446_b200 import model as MD  # noqa: E402


def run(m, images):
    """Record (name, args) of every call, and snapshot every tensor the
    forward creates afterwards by hooking torch.empty-like outputs: we
    clone each pointer argument's tensor after the call via a registry."""
    calls = []
    orig = _lib.call
    reg = {}
    orig_ptr = _lib.ptr

    def ptr(t):
        p = orig_ptr(t)
        if p is not None:
            reg[p] = t
        return p

    def call(name, *args):
        orig(name, *args)
        torch.cuda.synchronize()
        outs = []
        for a in args:
            if isinstance(a, int) and a in reg:
                outs.append(reg[a].detach().clone())
        calls.append((name, outs))
    _lib.call = call
    _lib.ptr = ptr
    try:
        y = m.forward(images)
    finally:
        _lib.call = orig
        _lib.ptr = orig_ptr
    return y, calls


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "pvt_small"
    B = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    lo = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    hi = int(sys.argv[4]) if len(sys.argv) > 4 else 4
    spec = specs.pvt_v2_b0(img=64, classes=10) if name == "pvt_small" else specs.BUILDERS[name]()
    m = MD.Network(spec)
    img = ops.rng(5).uniform(0, 1, (B, spec["img"], spec["img"], 3)).astype(np.float32)
    x = torch.from_numpy(img).cuda()
    y_full, c_full = run(m, x)
    y_sub, c_sub = run(m, x[lo:hi].contiguous())
    print("logits max diff", float((y_full[lo:hi] - y_sub).abs().max()))
    shown = 0
    for i, ((n1, o1), (n2, o2)) in enumerate(zip(c_full, c_sub)):
        assert n1 == n2, (i, n1, n2)
        for j, (a, b) in enumerate(zip(o1, o2)):
            if a.dtype != b.dtype or a.ndim == 0 or a.shape[0] == 0:
                continue
            # rows of the shared images: leading dim proportional to the batch
            if a.shape[0] % B or b.shape[0] % (hi - lo) or a.shape[0] // B != b.shape[0] // (hi - lo):
                continue
            per = a.shape[0] // B
            sa = a[lo * per: hi * per]
            if sa.shape != b.shape:
                continue
            if sa.dtype.is_floating_point:
                diff = float((sa - b).abs().max())
            else:
                diff = float((sa != b).sum())
            if diff != 0 and shown < 12:
                print(f"call {i} {n1} arg#{j} shape {tuple(a.shape)} dtype {a.dtype}: diff {diff}")
                shown += 1


if __name__ == "__main__":
    main()
