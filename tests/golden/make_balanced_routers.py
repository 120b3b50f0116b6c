#!/usr/bin/env python3
"""Latency-aware routers for the benchmark models, trained by the REFERENCE's
router-only procedure (ref scripts/moe_balance_demo.py:31-51,
tests/test_acceptance.py:241-266; losses ref moe.py:111-189), run in the build
container on the unmodified reference package:

    python tests/golden/make_balanced_routers.py [pvt_v2_b0 ...]

For every MoE module in forward order, the module's inputs are captured from
the reference composition (make_golden.RefNet) with all EARLIER routers
already trained, and its W_g is trained from zero with momentum SGD
(momentum 0.9, batch 128, 5000 steps) on the importance + load losses with the
expert latencies of MoeConfig.lat = (3, 1) (mult, shift), i.e. latency
coefficients alpha = (0.75, 0.25): the latency-balanced split sends ~75 % of
the tokens to the shift expert. Experts are frozen (router-only training).
The step size is the demo's lr 0.3 rescaled by the layer's mean squared token
norm (the demo's tokens have 20); unscaled, larger-norm inputs saturate the
router into a one-expert split (share 1.0), in which case the step is retried
10x smaller (recorded per layer as "lr:<name>"). Stage-1 inputs of the first block are
LayerNorm outputs with a near-zero channel mean (|mean| 0.07 vs token norm
5.7), which no bias-free linear router can split far from 50/50 (the
reference's own note, ref tests/test_acceptance.py:252-253): those layers end
near 0.55.

Output: paper_2306_06446_b200/data/routers_<model>_balanced.npz with one f32
(d, 2) array per module name ("s0.b0.attn.q", ..., "s2.b1.mlp"), the share of
expert 1 on the training tokens, and the image seed; bench.py --router
balanced and the parity tests load it.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, HERE)

import make_golden as G  # noqa: E402  (puts the reference on sys.path)
from shiftadd import moe as MOE  # noqa: E402
from shiftadd import tensor as T  # noqa: E402

from paper_2306_06446_b200 import specs  # noqa: E402

OUT_DIR = os.path.join(REPO, "paper_2306_06446_b200", "data")
STEPS, BATCH, MOMENTUM, SIGMA = 5000, 128, 0.9, 0.1
# step size: the reference's lr 0.3 for its tokens N(0.5, 1) in d = 16, i.e.
# mean |x|^2 = 20, rescaled to each layer's mean squared token norm
LR_REF, NORM2_REF = 0.3, 20.0
LAT = (3.0, 1.0)           # MoeConfig.lat (ref model.py:84-88): mult, shift
TRAIN_IMAGES, IMAGE_SEED = 2, 808


def train_router(x, seed, lr):
    """The reference router-only loop (ref tests/test_acceptance.py:249-261),
    on tokens drawn from the captured layer inputs x (M, d)."""
    rng = T.make_rng(seed)
    alpha = MOE.latency_coefficients(LAT)
    wg = np.zeros((x.shape[1], 2), dtype=np.float64)
    vel = np.zeros_like(wg)
    x64 = x.astype(np.float64)
    for _ in range(STEPS):
        xb = x64[rng.integers(0, x64.shape[0], BATCH)]
        p, logits = MOE.route(xb, MOE.Router(w_g=wg, sigma=SIGMA))
        dlogits = (T.softmax_backward(MOE.importance_loss_grad(p, alpha), p, -1)
                   + MOE.load_loss_grad(logits, alpha, SIGMA))
        vel = MOMENTUM * vel + xb.T @ dlogits
        wg -= lr * vel
    return wg.astype(np.float32)


def capture_input(net, images, target):
    rec = {}
    mods = dict(net.moe_modules())
    mod = mods[target]
    orig = mod.forward

    def wrapped(x, train=False):
        rec["x"] = x
        return orig(x, train)
    mod.forward = wrapped
    try:
        net.forward(images)
    finally:
        mod.forward = orig
    return rec["x"]


def make(model_name):
    spec = specs.BUILDERS[model_name]()
    net = G.RefNet(spec)
    images = T.make_rng(IMAGE_SEED).uniform(0, 1, (TRAIN_IMAGES, spec["img"], spec["img"], 3)) \
        .astype(np.float32)
    out = {"image_seed": np.int64(IMAGE_SEED), "train_images": np.int64(TRAIN_IMAGES)}
    names = [n for n, _ in net.moe_modules()]
    for i, name in enumerate(names):
        t0 = time.perf_counter()
        x = capture_input(net, images, name)
        lr = LR_REF * NORM2_REF / float(np.mean(np.sum(x.astype(np.float64) ** 2, axis=1)))
        for _ in range(3):   # a saturated (one-expert) split: retry with a 10x smaller step
            wg = train_router(x, seed=i, lr=lr)
            p, logits = MOE.route(x, MOE.Router(w_g=wg))
            share = MOE.dispatch(p, logits).share(1)
            if 0.05 < share < 0.95:
                break
            lr *= 0.1
        mod = dict(net.moe_modules())[name]
        mod.wg.value[...] = wg
        out[name] = wg
        out["share:" + name] = np.float32(share)
        out["lr:" + name] = np.float32(lr)
        print(f"{name}: d={x.shape[1]} tokens={x.shape[0]} lr {lr:.2e} shift share {share:.3f} "
              f"({time.perf_counter() - t0:.1f}s)", flush=True)
    os.makedirs(OUT_DIR, exist_ok=True)
    path = os.path.join(OUT_DIR, f"routers_{model_name}_balanced.npz")
    np.savez_compressed(path, **out)
    print("wrote", path)


def main():
    for name in sys.argv[1:] or ["pvt_v2_b0"]:
        make(name)


if __name__ == "__main__":
    main()
