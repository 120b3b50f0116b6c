"""Router weight sets for the benchmark models.

The reference draws every MoE router W_g ~ N(0, 0.02^2) (ref model.py:499-521)
and balances it during training with latency-aware importance / load losses
(ref moe.py:111-189, MoeConfig.lat = (3, 1): the shift expert is 3x cheaper,
so the balanced split sends ~75 % of the tokens to it). A random-init router
splits tokens arbitrarily (0-100 % per layer), which makes the expert mix of a
benchmark an accident of the seed. `load_balanced(model)` returns the routers
trained by the reference's router-only procedure
(tests/golden/make_balanced_routers.py, run against the unmodified reference;
weights committed under data/), which bench.py --router balanced and the
parity tests install with `apply_model`.
"""

from __future__ import annotations

import os

import numpy as np
import torch

DATA = os.path.join(os.path.dirname(os.path.abspath(__file__)), "data")


class RouterSet:
    """Named (d, 2) f32 router matrices, keyed like Network.moe_modules()
    ("s0.b0.attn.q", ..., "s2.b1.mlp"), plus the expert-1 (shift) share each
    reached on its training tokens."""

    def __init__(self, name: str, weights: dict, train_shares: dict):
        self.name = name
        self.weights = weights
        self.train_shares = train_shares

    def apply_model(self, model):
        """Install the routers into a device Network (in place, before its
        first forward)."""
        mods = dict(model.moe_modules())
        missing = sorted(set(self.weights) - set(mods))
        if missing or set(mods) - set(self.weights):
            raise ValueError(f"router set {self.name} does not match the model: {missing}")
        for key, mod in mods.items():
            w = torch.from_numpy(self.weights[key])
            if tuple(mod.wg.value.shape) != tuple(w.shape):
                raise ValueError(f"{key}: router shape {tuple(w.shape)} != {tuple(mod.wg.value.shape)}")
            mod.wg.value.copy_(w.to(mod.wg.value.device))
        return model

    @staticmethod
    def shares(model) -> dict:
        """Shift-expert share of every MoE layer in the model's last forward,
        plus the token-weighted overall share."""
        out, tot, shift = {}, 0, 0
        for key, mod in model.moe_modules():
            e = mod.last_plan.expert_of
            out[key] = round(float(e.mean()), 4)
            tot += e.size
            shift += int(e.sum())
        out["overall"] = round(shift / max(tot, 1), 4)
        return out


def load_balanced(model_name: str) -> RouterSet:
    path = os.path.join(DATA, f"routers_{model_name}_balanced.npz")
    if not os.path.exists(path):
        raise FileNotFoundError(f"no balanced routers for {model_name} ({path}); generate them "
                                "with tests/golden/make_balanced_routers.py")
    with np.load(path) as z:
        weights = {k: z[k].astype(np.float32) for k in z.files if ":" not in k and "." in k}
        shares = {k[len("share:"):]: float(z[k]) for k in z.files if k.startswith("share:")}
    return RouterSet(model_name, weights, shares)
