#!/usr/bin/env python3
"""Generate the golden fixtures that pin the oracle (and, through it, the GPU
path) to the REAL reference package.

Run in the build container only (it imports the unmodified reference from
/root/reference/pkg/src, which does not exist on the GPU box):

    python tests/golden/make_golden.py

Outputs (committed): tests/golden/{kat,toy_c1,toy_c1_moe,pvt_small,deit_small,pvt_b0_full,
    pvt_v1_tiny_full,deit_tiny_full,pvt_v2_b2_full,apply_stage,checkpoint,addlinear}.npz and
    tests/golden/toy_moe.saddckpt (a reference-written checkpoint)

Every model here is composed from the reference's own classes (Linear,
ShiftLinearLayer, MoeModule, Mlp, AttentionLayer, Block, LayerNorm and the
`_make_linear` / `_make_mlp` builders, ref model.py:95-553), following the
spec dicts of paper_2306_06446_b200/specs.py; the toy config uses the
reference `Model` class itself. Layer outputs are captured by wrapping the
layer objects' `forward` methods — the reference code is not modified.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

from shiftadd import attention as A  # noqa: E402  (the reference)
from shiftadd import model as MD  # noqa: E402
from shiftadd import moe as MOE  # noqa: E402
from shiftadd import quantize as Q  # noqa: E402
from shiftadd import tensor as T  # noqa: E402
from shiftadd.tensor import GradPair  # noqa: E402

from paper_2306_06446_b200 import specs  # noqa: E402

F32 = np.float32


def tie_threshold():
    lo, hi = 0, int(np.float32(1e-6).view(np.uint32))
    while lo < hi:
        mid = (lo + hi + 1) // 2
        d = np.array([mid], np.uint32).view(np.float32)
        if np.exp(-d)[0] == np.float32(1.0):
            lo = mid
        else:
            hi = mid - 1
    return np.array([lo], np.uint32).view(np.float32)[0]


def packbits01(bits):
    return np.packbits(np.asarray(bits, np.uint8).ravel(), bitorder="little")


# ---------------------------------------------------------------------------
# known-answer vectors for the primitives


def make_kat():
    out = {}
    g = T.make_rng(2024)
    # quantize_shift: hand values, boundaries near sqrt(2)·2^k, zeros, clamps
    sq2 = np.float32(np.sqrt(2.0))
    hand = np.array([1.0, 0.75, -0.3, 0.0, -0.0, 2.0 ** -20, 2.0 ** 20, -1e-30, 3.0, -0.5,
                     np.nextafter(sq2, F32(0)), np.nextafter(sq2, F32(2)),
                     np.nextafter(sq2 * 4, F32(0)), np.nextafter(sq2 * 4, F32(8)),
                     2.0 ** -15, 2.0 ** -15.5, 2.0 ** 15, 2.0 ** 15.6], np.float32)
    rand = np.concatenate([g.uniform(-4, 4, 600), g.standard_normal(600) * 0.05,
                           np.ldexp(g.uniform(1, 2, 300), g.integers(-20, 20, 300))]).astype(F32)
    w = np.concatenate([hand, rand]).reshape(1, -1)
    lay = Q.quantize_shift(w)
    out["qs_w"], out["qs_s"], out["qs_p"] = w, lay.s, lay.p
    out["qs_rec"] = Q.reconstruct(lay)
    # shift_forward vs a random input (bit-identical to FakeShift by construction)
    x = g.uniform(-1, 1, (37, 48)).astype(F32)
    lay2 = Q.quantize_shift((g.standard_normal((48, 24)) / 7).astype(F32))
    out["sf_x"], out["sf_s"], out["sf_p"] = x, lay2.s, lay2.p
    out["sf_y"] = Q.shift_forward(x, lay2)
    # sign_unit edge cases
    se = np.array([-0.0, 0.0, -1e-45, np.nan, -np.inf, np.inf, -1.0, 1e-45], np.float32)
    out["sign_x"], out["sign_y"] = se, Q.sign_unit(se)
    # binarize per-head + linear core on binary features (dk 16 / 32 / 64)
    for dk, n, H in ((16, 196, 8), (32, 200, 3), (64, 197, 6)):
        qh = g.standard_normal((H, n, dk)).astype(F32)
        kh = g.standard_normal((H, n, dk)).astype(F32)
        vh = g.standard_normal((H, n, dk)).astype(F32)
        qh[0, 3] = -np.abs(qh[0, 3])     # an all-negative query row → zero output
        bq, gq = Q.binarize(qh, "per-head")
        bk, gk = Q.binarize(kh, "per-head")
        qf = (gq * (bq + 1.0) * 0.5).astype(F32)
        kf = (gk * (bk + 1.0) * 0.5).astype(F32)
        o, _ = A.linear_core(qf, kf, vh, A.EPS_NORM)
        pre = f"lc{dk}_"
        out[pre + "q"], out[pre + "k"], out[pre + "v"] = qh, kh, vh
        out[pre + "gq"], out[pre + "gk"], out[pre + "out"] = gq, gk, o
    # dwconv over token grids (5 → 3x3, 196 → 14x14, 197 → 15x15)
    for n in (5, 196, 197):
        v = g.standard_normal((n, 24)).astype(F32)
        k = (g.standard_normal((3, 3, 24)) * 0.1).astype(F32)
        y, side = A._dwconv_tokens(v, k)
        out[f"dw{n}_v"], out[f"dw{n}_k"], out[f"dw{n}_y"] = v, k, y
        out[f"dw{n}_side"] = np.int32(side)
    # softmax core
    qs, ks, vs = (g.standard_normal((8, 49, 32)).astype(F32) for _ in range(3))
    out["sm_q"], out["sm_k"], out["sm_v"] = qs, ks, vs
    out["sm_out"], _ = A.softmax_core(qs, ks, vs)
    # route / dispatch, including crafted near-ties around numpy's exp threshold
    xr = g.standard_normal((2048, 32)).astype(F32)
    wg = (g.standard_normal((32, 2)) * 0.02).astype(F32)
    p, logits = MOE.route(xr, MOE.Router(w_g=wg))
    plan = MOE.dispatch(p, logits)
    out["rt_x"], out["rt_wg"], out["rt_logits"], out["rt_p"] = xr, wg, logits, p
    out["rt_expert"] = plan.expert_of.astype(np.int32)
    out["rt_gate"] = plan.gate_of
    out["rt_perm"] = np.concatenate(plan.index_of).astype(np.int32)
    thr = tie_threshold()
    base = g.standard_normal(64).astype(F32)
    deltas = np.array([0.0, thr, np.nextafter(thr, F32(1)), np.nextafter(thr, F32(0)),
                       2 * thr, 2.0 ** -25, 2.0 ** -24, 1e-7, -thr, -1e-7], np.float32)
    tl = []
    for dlt in deltas:
        for b in base[:6]:
            l0 = np.float32(b)
            l1 = np.float32(l0 + dlt)
            tl.append([l0, l1])
    tl = np.array(tl, np.float32)
    tp = T.softmax(tl, axis=-1)
    tplan = MOE.dispatch(tp, tl)
    out["tie_logits"], out["tie_expert"] = tl, tplan.expert_of.astype(np.int32)
    out["tie_gate"] = tplan.gate_of
    out["tie_threshold"] = np.float32(thr)
    # moe_forward with a dense and a shift expert on shared weights
    wm = (g.standard_normal((32, 40)) / np.sqrt(32)).astype(F32)
    ex = [MD.Linear(wm), MD.ShiftLinearLayer(wm.copy())]
    mod = MD.MoeModule((g.standard_normal((32, 2)) * 0.02).astype(F32), ex, MD.MoeConfig())
    xm = g.standard_normal((333, 32)).astype(F32)
    out["mf_x"], out["mf_w"], out["mf_wg"] = xm, wm, mod.wg.value
    out["mf_y"] = mod.forward(xm)
    out["mf_expert"] = mod.last_plan.expert_of.astype(np.int32)
    # layer norm / gelu on float32
    xl = g.standard_normal((64, 160)).astype(F32) * 3 + 1
    ln = MD.LayerNorm(160, F32)
    out["ln_x"], out["ln_y"] = xl, ln.forward(xl)
    out["gelu_x"] = xl
    out["gelu_y"] = T.gelu(xl)
    return out


# ---------------------------------------------------------------------------
# model compositions from reference classes


class RefNet:
    """Reference layers wired per a spec dict (stage chaining = PVT style)."""

    def __init__(self, spec):
        self.spec = spec
        dt = F32
        qcfg = Q.QuantConfig(p_min=spec["p_min"], p_max=spec["p_max"])
        mcfg = MD.MoeConfig()
        g = T.make_rng(spec["seed"])
        c_in = spec["channels"]
        self.stages = []
        side = spec["img"]
        for st in spec["stages"]:
            d = st["d"]
            side //= st["patch"]
            n = side * side + (1 if st["cls_token"] else 0)
            S = {"pe": MD.Linear(MD._init_linear(g, st["patch"] ** 2 * c_in, d, dt))}
            if st["cls_token"]:
                S["cls"] = (g.standard_normal((1, d)) * 0.02).astype(dt)
            if st["pos"]:
                S["pos"] = (g.standard_normal((n, d)) * 0.02).astype(dt)
            S["blocks"] = []
            for bc in st["blocks"]:
                cfg = MD.BlockConfig(d=d, h=bc["h"], mlp_ratio=bc["mlp_ratio"],
                                     attn_mode=bc["attn_mode"], mlp_mode=bc["mlp_mode"],
                                     attn_linear_mode=bc["attn_linear_mode"],
                                     exempt=bc["exempt"])
                proj = {k: MD._make_linear(cfg.attn_linear_mode, g, d, d, dt, mcfg, qcfg)
                        for k in ("q", "k", "v", "o")}
                dw = None
                if cfg.attn_mode != "softmax":
                    dwi = spec["dw_init"]
                    if isinstance(dwi, (int, float)):
                        dw = GradPair((g.standard_normal((3, 3, d)) * float(dwi)).astype(dt))
                    else:
                        dw = GradPair(np.zeros((3, 3, d), dt))
                mlp = MD._make_mlp(cfg, g, dt, mcfg, qcfg)
                S["blocks"].append(MD.Block(cfg, MD.AttentionLayer(cfg, proj, dw), mlp, dt))
            S["embed_ln"] = MD.LayerNorm(d, dt) if st["embed_norm"] else None
            S["stage_ln"] = MD.LayerNorm(d, dt) if st["stage_norm"] else None
            self.stages.append(S)
            c_in = d
        self.head = MD.Linear(MD._init_linear(g, spec["stages"][-1]["d"], spec["classes"],
                                              dt, scale=0.01))
        dwi = spec["dw_init"]
        if isinstance(dwi, dict):
            g2 = T.make_rng(dwi["seed"])
            for S in self.stages:
                for blk in S["blocks"]:
                    if blk.attn.dw is not None:
                        blk.attn.dw.value[...] = (g2.standard_normal(blk.attn.dw.value.shape)
                                                  * dwi["std"]).astype(dt)

    def weights(self):
        """Arrays in oracle.nets.iter_weights order (names match)."""
        for si, S in enumerate(self.stages):
            yield f"s{si}.pe", S["pe"].w.value
            for key in ("cls", "pos"):
                if key in S:
                    yield f"s{si}.{key}", S[key]
            for bi, blk in enumerate(S["blocks"]):
                pre = f"s{si}.b{bi}"
                for k in ("q", "k", "v", "o"):
                    yield from _ref_layer_weights(f"{pre}.attn.{k}", blk.attn.proj[k])
                if blk.attn.dw is not None:
                    yield f"{pre}.attn.dw", blk.attn.dw.value
                yield from _ref_layer_weights(f"{pre}.mlp", blk.mlp)
        yield "head", self.head.w.value

    def forward(self, images):
        spec = self.spec
        grid = np.asarray(images, dtype=F32) - 0.5
        tok = None
        for si, (st, S) in enumerate(zip(spec["stages"], self.stages)):
            b, hh, ww, c = grid.shape
            p = st["patch"]
            pt = grid.reshape(b, hh // p, p, ww // p, p, c).transpose(0, 1, 3, 2, 4, 5)
            pt = np.ascontiguousarray(pt).reshape(b, (hh // p) * (ww // p), p * p * c)
            n = pt.shape[1]
            tok = S["pe"].forward(pt.reshape(b * n, -1)).reshape(b, n, -1)
            if "cls" in S:
                tok = np.concatenate([np.broadcast_to(S["cls"], (b, 1, st["d"])), tok], axis=1)
            if "pos" in S:
                tok = tok + S["pos"]
            if S["embed_ln"] is not None:
                tok = S["embed_ln"].forward(tok)
            for blk in S["blocks"]:
                tok = blk.forward(tok)
            if S["stage_ln"] is not None:
                tok = S["stage_ln"].forward(tok)
            if si + 1 < len(self.stages):
                sd = int(round(np.sqrt(n)))
                grid = tok.reshape(b, sd, sd, -1)
        pooled = tok[:, 0] if spec["pool"] == "cls" else tok.mean(axis=1)
        return self.head.forward(np.ascontiguousarray(pooled))

    def moe_modules(self):
        for si, S in enumerate(self.stages):
            for bi, blk in enumerate(S["blocks"]):
                pre = f"s{si}.b{bi}"
                for k in ("q", "k", "v", "o"):
                    if isinstance(blk.attn.proj[k], MD.MoeModule):
                        yield f"{pre}.attn.{k}", blk.attn.proj[k]
                if isinstance(blk.mlp, MD.MoeModule):
                    yield f"{pre}.mlp", blk.mlp

    def attn_layers(self):
        for si, S in enumerate(self.stages):
            for bi, blk in enumerate(S["blocks"]):
                yield f"s{si}.b{bi}.attn", blk.attn


def _ref_layer_weights(name, L):
    if isinstance(L, (MD.Linear, MD.ShiftLinearLayer)):
        yield name + ".w", L.w.value
    elif isinstance(L, MD.Mlp):
        yield from _ref_layer_weights(name + ".fc1", L.fc1)
        yield from _ref_layer_weights(name + ".fc2", L.fc2)
    else:
        yield name + ".wg", L.wg.value
        for e, ex in enumerate(L.experts):
            yield from _ref_layer_weights(f"{name}.expert{e}", ex)


def capture(net, images, full=True):
    """Run the reference forward, recording q/k per attention layer and the
    dispatch plan (+ inputs) per MoE layer."""
    rec = {}
    originals = []
    for name, attn in net.attn_layers():
        if attn.cfg.attn_mode != "linear-binary":
            continue
        for key in ("q", "k"):
            lay = attn.proj[key]
            orig = lay.forward

            def wrapped(x, train=False, _o=orig, _n=f"{name}.{key}"):
                y = _o(x, train)
                rec[_n] = y
                return y
            lay.forward = wrapped
            originals.append((lay, orig))
    moe_in = {}
    for name, mod in net.moe_modules():
        orig = mod.forward

        def wrapped(x, train=False, _o=orig, _n=name):
            moe_in[_n] = x
            return _o(x, train)
        mod.forward = wrapped
        originals.append((mod, orig))
    logits = net.forward(images)
    for obj, orig in originals:
        obj.forward = orig
    out = {"logits": logits}
    heads = {}
    for name, attn in net.attn_layers():
        heads[name] = attn.cfg.h
    for key, val in rec.items():
        attn_name = key.rsplit(".", 1)[0]
        h = heads[attn_name]
        B = images.shape[0]
        n = val.shape[0] // B
        d = val.shape[1]
        bits = (~(val < 0)).astype(np.uint8)
        if full:
            out[f"act:{key}"] = val
        out[f"codes:{key}"] = packbits01(bits)
        qh = A.split_heads(val.reshape(B, n, d), h).reshape(B * h, n, d // h)
        _, gam = Q.binarize(qh, "per-head")
        out[f"gamma:{key}"] = gam.reshape(B, h)
    for name, mod in net.moe_modules():
        plan = mod.last_plan
        out[f"route:{name}"] = packbits01(plan.expert_of.astype(np.uint8))
        out[f"gate:{name}"] = plan.gate_of.astype(F32)
        if full:
            out[f"moe_x:{name}"] = moe_in[name]
    return out


def weight_digest(net):
    h = hashlib.sha256()
    for name, arr in net.weights():
        h.update(name.encode())
        h.update(np.ascontiguousarray(arr).tobytes())
    return h.hexdigest()


def make_model_fixture(spec, batch, img_seed, full=True):
    net = RefNet(spec)
    images = T.make_rng(img_seed).uniform(0, 1, (batch, spec["img"], spec["img"], 3)).astype(F32)
    out = capture(net, images, full=full)
    out["images_seed"] = np.int64(img_seed)
    out["batch"] = np.int64(batch)
    out["weight_sha256"] = np.array(weight_digest(net))
    if full:
        out["images"] = images
    return out


def make_toy_via_reference_model():
    """Config 1 through the reference `Model` class itself (+ DW randomised
    from the side stream), to tie the spec format to the reference Model."""
    spec = specs.toy_c1()
    bcs = [MD.BlockConfig(d=64, h=4, mlp_ratio=4.0, attn_mode="linear-binary",
                          mlp_mode="shift", attn_linear_mode="shift") for _ in range(2)]
    m = MD.Model(MD.ModelConfig(blocks=bcs, patch=4, img=56, classes=10, seed=0))
    g2 = T.make_rng(spec["dw_init"]["seed"])
    for blk in m.blocks:
        blk.attn.dw.value[...] = (g2.standard_normal(blk.attn.dw.value.shape) * 0.1).astype(F32)
    images = T.make_rng(1).uniform(0, 1, (8, 56, 56, 3)).astype(F32)
    return m.forward(images)


# full-224 fixtures of BASELINE configs C3 / C4 / C5 (batch 2, codes / routes /
# gates / logits only): name -> (spec builder, batch, image seed)
FULL_224 = {
    "pvt_v1_tiny_full": (specs.pvt_v1_tiny, 2, 21),   # C3: dk = 64, d = 64/128/320/512, pos
    "deit_tiny_full": (specs.deit_tiny, 2, 22),       # C4: 197 tokens, 12 blocks, 15x15 DW grid
    "pvt_v2_b2_full": (specs.pvt_v2_b2, 2, 23),       # C5: depths 3/4/6/3
}


def _ref_model_weights(m):
    """Reference `Model` parameters in paper_2306_06446_b200 Network.named_weights order."""
    yield "s0.pe", m.patch_embed.w.value
    yield "s0.pos", m.pos.value
    for bi, blk in enumerate(m.blocks):
        pre = f"s0.b{bi}"
        for k in ("q", "k", "v", "o"):
            yield from _ref_layer_weights(f"{pre}.attn.{k}", blk.attn.proj[k])
        if blk.attn.dw is not None:
            yield f"{pre}.attn.dw", blk.attn.dw.value
        yield from _ref_layer_weights(f"{pre}.mlp", blk.mlp)
    yield "head", m.head.w.value


def _digest_pairs(pairs):
    h = hashlib.sha256()
    for name, arr in pairs:
        h.update(name.encode())
        h.update(np.ascontiguousarray(arr).tobytes())
    return h.hexdigest()


def make_apply_stage():
    """ref model.py:897-930 on a softmax/dense toy Model (last block exempt):
    logits and weight digests after stage 1 (linear-binary attention) and after
    stage 2 (MoE projections and MLPs, routers from PCG64(77))."""
    bcs = [MD.BlockConfig(d=64, h=4, mlp_ratio=4.0, attn_mode="softmax", mlp_mode="dense",
                          attn_linear_mode="dense", exempt=(i == 2)) for i in range(3)]
    m = MD.Model(MD.ModelConfig(blocks=bcs, patch=4, img=32, classes=10, seed=5))
    images = T.make_rng(9).uniform(0, 1, (3, 32, 32, 3)).astype(F32)
    out = {"images": images, "logits0": m.forward(images),
           "sha0": np.array(_digest_pairs(_ref_model_weights(m)))}
    MD.apply_stage(m, 1)
    out["logits1"] = m.forward(images)
    out["sha1"] = np.array(_digest_pairs(_ref_model_weights(m)))
    MD.apply_stage(m, 2, mlp_target="moe", attn_target="moe")
    out["logits2"] = m.forward(images)
    out["sha2"] = np.array(_digest_pairs(_ref_model_weights(m)))
    for bi, blk in enumerate(m.blocks):
        for k in ("q", "k", "v", "o"):
            if isinstance(blk.attn.proj[k], MD.MoeModule):
                plan = blk.attn.proj[k].last_plan
                out[f"route:s0.b{bi}.attn.{k}"] = plan.expert_of.astype(np.int32)
        if isinstance(blk.mlp, MD.MoeModule):
            out[f"route:s0.b{bi}.mlp"] = blk.mlp.last_plan.expert_of.astype(np.int32)
    return out


def make_addlinear():
    """MatAdd KATs from the reference (ref quantize.py:143-160, 177-185 and
    tests/test_quantize.py:150-171): the hand case, the all-plus-one row sum and
    binarized random layers (reparam_linear(w, "add"))."""
    out = {}
    layer = Q.AddLinear(b=T.tensor([[1.0], [-1.0]]), gamma=1.0)
    out["hand_x"] = T.tensor([[1.0, 2.0]])
    out["hand_b"] = layer.b
    out["hand_y"] = Q.add_matmul(out["hand_x"], layer)
    g = T.make_rng(31)
    for i, (m, k, n) in enumerate(((4, 6, 3), (8, 8, 8), (100, 64, 48), (1000, 96, 80))):
        x = g.uniform(-1, 1, (m, k)).astype(F32)
        if i == 0:
            b, gamma = np.ones((k, n), F32), 1.0
        else:
            rr = Q.reparam_linear(g.uniform(-1, 1, (k, n)).astype(F32), "add")
            b, gamma = rr.layer.b, rr.layer.gamma
            out[f"w{i}"] = rr.shadow
        out[f"x{i}"], out[f"b{i}"], out[f"g{i}"] = x, b.astype(F32), np.array(gamma)
        out[f"y{i}"] = Q.add_matmul(x, Q.AddLinear(b=b, gamma=gamma))
    return out


def make_checkpoint():
    """A SADDCKPT container written by the reference (ref checkpoint.py:64-97)
    for a toy MoE Model whose weights were perturbed away from the init (so a
    loader must really read them), plus the reference forward logits and
    `evaluate` dispatch maps / shares (ref model.py:745-765) over 5 images in
    batches of 3."""
    from shiftadd import checkpoint as CK
    from shiftadd import data as DATA
    bcs = [MD.BlockConfig(d=32, h=2, mlp_ratio=2.0, attn_mode="linear-binary", mlp_mode="moe",
                          attn_linear_mode="moe"),
           MD.BlockConfig(d=32, h=2, mlp_ratio=2.0, attn_mode="linear-binary", mlp_mode="shift",
                          attn_linear_mode="moe")]
    m = MD.Model(MD.ModelConfig(blocks=bcs, patch=4, img=16, classes=5, seed=3))
    g = T.make_rng(11)
    for _, p in m.named_params():
        p.value[...] = (p.value + g.standard_normal(p.value.shape) * 0.05).astype(F32)
    m.post_step()
    CK.save_checkpoint(os.path.join(HERE, "toy_moe.saddckpt"), m, step=42,
                       extra_meta={"note": "golden fixture"})
    images = T.make_rng(12).uniform(0, 1, (5, 16, 16, 3)).astype(F32)
    labels = T.make_rng(13).integers(0, 5, 5).astype(np.int64)
    out = {"images": images, "labels": labels, "logits": m.forward(images)}
    res = MD.evaluate(m, DATA.Dataset(images=images, labels=labels), batch_size=3)
    out["accuracy"] = np.array(res.accuracy)
    for name, arr in res.dispatch_maps.items():
        out["map:" + name] = arr.astype(np.int32)
        out["share:" + name] = np.array(res.expert_shares[name])
    return out


def main():
    only = sys.argv[1:]
    if only:   # e.g. `make_golden.py pvt_v1_tiny_full` regenerates just that fixture
        for name in only:
            if name == "apply_stage":
                np.savez_compressed(os.path.join(HERE, "apply_stage.npz"), **make_apply_stage())
                continue
            if name == "checkpoint":
                np.savez_compressed(os.path.join(HERE, "checkpoint.npz"), **make_checkpoint())
                continue
            if name == "addlinear":
                np.savez_compressed(os.path.join(HERE, "addlinear.npz"), **make_addlinear())
                continue
            fn, b, seed = FULL_224[name]
            np.savez_compressed(os.path.join(HERE, name + ".npz"),
                                **make_model_fixture(fn(), b, seed, full=False))
        return
    np.savez_compressed(os.path.join(HERE, "kat.npz"), **make_kat())
    toy = make_model_fixture(specs.toy_c1(), 8, 1)
    toy["logits_via_Model"] = make_toy_via_reference_model()
    assert np.array_equal(toy["logits_via_Model"], toy["logits"]), "spec composition != Model"
    np.savez_compressed(os.path.join(HERE, "toy_c1.npz"), **toy)
    toy_moe = make_model_fixture(specs.toy_c1(attn_linear_mode="moe", mlp_mode="moe"), 2, 3)
    np.savez_compressed(os.path.join(HERE, "toy_c1_moe.npz"), **toy_moe)
    np.savez_compressed(os.path.join(HERE, "pvt_small.npz"),
                        **make_model_fixture(specs.pvt_v2_b0(img=64, classes=10), 2, 5))
    np.savez_compressed(os.path.join(HERE, "deit_small.npz"),
                        **make_model_fixture(specs.deit_tiny(img=64, classes=10, depth=3), 2, 6))
    np.savez_compressed(os.path.join(HERE, "pvt_b0_full.npz"),
                        **make_model_fixture(specs.pvt_v2_b0(), 1, 7, full=False))
    for name, (fn, b, seed) in FULL_224.items():
        np.savez_compressed(os.path.join(HERE, name + ".npz"),
                            **make_model_fixture(fn(), b, seed, full=False))
    np.savez_compressed(os.path.join(HERE, "apply_stage.npz"), **make_apply_stage())
    np.savez_compressed(os.path.join(HERE, "checkpoint.npz"), **make_checkpoint())
    np.savez_compressed(os.path.join(HERE, "addlinear.npz"), **make_addlinear())
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))


if __name__ == "__main__":
    main()
