"""Architecture specs for the benchmark configs (BASELINE.json `configs`).

The reference ships one toy ViT (ref model.py:525-577). The PVT / DeiT models
named by the benchmark are composed from the reference's own layers (Block,
AttentionLayer, Mlp, MoeModule, ShiftLinearLayer, Linear, LayerNorm), with the
public architecture constants pinned here:

- PVTv2-B0: dims 32/64/160/256, heads 1/2/5/8, MLP ratios 8/8/4/4, depths 2/2/2/2
- PVTv2-B2: dims 64/128/320/512, heads 1/2/5/8, ratios 8/8/4/4, depths 3/4/6/3
- PVTv1-Tiny: B2 dims, depths 2/2/2/2, non-overlapping patch embeds 4/2/2/2, pos embeds
- DeiT-Tiny: d 192, 12 blocks, 3 heads, ratio 4, patch 16, cls token → 197 tokens

Deviations from the public models (documented in DESIGN.md §2):
- patch embedding is non-overlapping patchify + Linear (+LN) at every stage;
  PVTv2's overlapping 7×7/3×3 conv embed is not expressible with reference layers;
- attention uses full-resolution K/V (the reference attention has no spatial
  reduction), binary linear attention in all but the last stage, which stays
  softmax MSA with dense projections (PAPER "keep the last stage as MSA",
  ref config exempt_last);
- the PVT MLP has no DWConv (ref SPEC.md:474); the DWConv branch lives on V in
  the linear-attention layers (ref attention.py:170-179), randomised N(0, 0.1)
  at init so it is exercised (the reference zero-initialises it, model.py:546);
- Linear layers carry no bias (ref model.py:96).

A spec is a plain dict; `oracle.nets.build` consumes the same dict.
"""

from __future__ import annotations

import copy

VARIANTS = {
    # name: (attn_linear_mode, mlp_mode) for non-exempt blocks
    "moe": ("moe", "moe"),        # LA + Quant + MoE (both)   — the ShiftAddViT final model
    "shift": ("shift", "shift"),  # LA + Quant + Shift (both)
    "la": ("dense", "dense"),     # LA + Quant only
}


def _block(h, ratio, attn_mode, lin, mlp, exempt=False, binary_order="auto"):
    return {"h": h, "mlp_ratio": float(ratio), "attn_mode": attn_mode,
            "attn_linear_mode": lin, "mlp_mode": mlp, "exempt": exempt,
            "binary_order": binary_order}


def _pyramid(dims, heads, ratios, depths, patches, *, img, classes, seed, variant,
             dw_std, pos, stage_norm_all):
    lin, mlp = VARIANTS[variant]
    stages = []
    last = len(dims) - 1
    for s, (d, h, r, depth, p) in enumerate(zip(dims, heads, ratios, depths, patches)):
        blocks = []
        for _ in range(depth):
            if s == last:   # exempt stage: softmax MSA, dense layers
                blocks.append(_block(h, r, "softmax", "dense", "dense", exempt=True))
            else:
                blocks.append(_block(h, r, "linear-binary", lin, mlp))
        stages.append({"patch": p, "d": d, "pos": pos, "cls_token": False,
                       "embed_norm": True, "stage_norm": stage_norm_all or s == last,
                       "blocks": blocks})
    return {"name": None, "img": img, "channels": 3, "classes": classes, "seed": seed,
            "dw_init": dw_std, "pool": "mean", "p_min": -15, "p_max": 15,
            "stages": stages}


def pvt_v2_b0(img=224, classes=1000, seed=0, variant="moe", dw_std=0.1):
    s = _pyramid([32, 64, 160, 256], [1, 2, 5, 8], [8, 8, 4, 4], [2, 2, 2, 2],
                 [4, 2, 2, 2], img=img, classes=classes, seed=seed, variant=variant,
                 dw_std=dw_std, pos=False, stage_norm_all=True)
    s["name"] = f"pvt_v2_b0-{variant}"
    return s


def pvt_v2_b2(img=224, classes=1000, seed=0, variant="moe", dw_std=0.1):
    s = _pyramid([64, 128, 320, 512], [1, 2, 5, 8], [8, 8, 4, 4], [3, 4, 6, 3],
                 [4, 2, 2, 2], img=img, classes=classes, seed=seed, variant=variant,
                 dw_std=dw_std, pos=False, stage_norm_all=True)
    s["name"] = f"pvt_v2_b2-{variant}"
    return s


def pvt_v1_tiny(img=224, classes=1000, seed=0, variant="moe", dw_std=0.1):
    s = _pyramid([64, 128, 320, 512], [1, 2, 5, 8], [8, 8, 4, 4], [2, 2, 2, 2],
                 [4, 2, 2, 2], img=img, classes=classes, seed=seed, variant=variant,
                 dw_std=dw_std, pos=True, stage_norm_all=False)
    s["name"] = f"pvt_v1_tiny-{variant}"
    return s


def deit_tiny(img=224, classes=1000, seed=0, variant="moe", dw_std=0.1, depth=12):
    """DeiT-T with quadratic binary Hamming attention in all but the last block."""
    lin, mlp = VARIANTS[variant]
    blocks = [_block(3, 4, "linear-binary", lin, mlp, binary_order="quadratic")
              for _ in range(depth - 1)]
    blocks.append(_block(3, 4, "softmax", "dense", "dense", exempt=True))
    return {"name": f"deit_tiny-{variant}", "img": img, "channels": 3, "classes": classes,
            "seed": seed, "dw_init": dw_std, "pool": "cls", "p_min": -15, "p_max": 15,
            "stages": [{"patch": 16, "d": 192, "pos": True, "cls_token": True,
                        "embed_norm": False, "stage_norm": True, "blocks": blocks}]}


def toy_c1(seed=0, blocks=2, d=64, h=4, img=56, patch=4, classes=10, dw_std=0.1,
           attn_linear_mode="shift", mlp_mode="shift"):
    """Config 1: the reference toy stack (ref SURVEY App. C-1) — exactly the
    reference `Model` draw order (pos after patch embed, final LN only). The
    DW kernels (zero in the reference, model.py:546) are drawn afterwards from
    a separate PCG64(seed+1) stream so the main draw order is untouched."""
    return {"name": "toy_c1", "img": img, "channels": 3, "classes": classes, "seed": seed,
            "dw_init": {"std": dw_std, "seed": seed + 1}, "pool": "mean", "p_min": -15, "p_max": 15,
            "stages": [{"patch": patch, "d": d, "pos": True, "cls_token": False,
                        "embed_norm": False, "stage_norm": True,
                        "blocks": [_block(h, 4, "linear-binary", attn_linear_mode, mlp_mode)
                                   for _ in range(blocks)]}]}


BUILDERS = {"pvt_v2_b0": pvt_v2_b0, "pvt_v2_b2": pvt_v2_b2, "pvt_v1_tiny": pvt_v1_tiny,
            "deit_tiny": deit_tiny, "toy_c1": toy_c1}


def clone(spec):
    return copy.deepcopy(spec)
