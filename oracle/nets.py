"""Forward-only numpy restatement of the reference layers and of the model
compositions the benchmark configs need. Test infrastructure only.

Architecture specs are plain dicts (the product's `ArchSpec.to_dict()` emits
the same format) so this module never imports the product:

    {"img", "channels", "classes", "seed",
     "dw_init": "zeros" | std (main stream, in place) | {"std", "seed"} (side stream),
     "pool": "mean" | "cls", "p_min", "p_max",
     "stages": [{"patch", "d", "pos", "cls_token", "embed_norm", "stage_norm",
                 "blocks": [{"h", "mlp_ratio", "attn_mode", "mlp_mode",
                             "attn_linear_mode", "exempt"}, ...]}, ...]}

The single-stage spec with pos=True, embed_norm=False, stage_norm=True and
dw_init="zeros" is exactly the reference toy `Model` (ref model.py:525-577).
Multi-stage specs chain stages PVT-style: the token grid of stage s is the
"image" patchified by stage s+1.
"""

from __future__ import annotations

import numpy as np

from . import ops

F32 = np.float32


# ---------------------------------------------------------------------------
# parameter construction (draw order = ref model.py:487-553)


def _draw_linear(g, fan_in, fan_out, scale=None):
    """N(0,1)·scale, scale defaults to 1/√fan_in (ref model.py:487-489)."""
    sc = scale if scale is not None else 1.0 / np.sqrt(fan_in)
    return (g.standard_normal((fan_in, fan_out)) * sc).astype(F32)


def _shift_layer(w, spec):
    s, p = ops.shift_quantize(w, spec.get("p_min", ops.P_MIN), spec.get("p_max", ops.P_MAX))
    return {"kind": "shift", "w": w, "s": s, "p": p}


def _linear(mode, g, fan_in, fan_out, spec):
    """One projection in dense / shift / moe form (ref model.py:492-503):
    the weight is drawn first, then (moe only) the router."""
    w = _draw_linear(g, fan_in, fan_out)
    if mode == "dense":
        return {"kind": "dense", "w": w}
    if mode == "shift":
        return _shift_layer(w, spec)
    if mode == "moe":
        wg = _draw_linear(g, fan_in, 2, scale=0.02)
        return {"kind": "moe", "wg": wg,
                "experts": [{"kind": "dense", "w": w}, _shift_layer(w.copy(), spec)]}
    raise ValueError(mode)


def _mlp(bc, d, g, spec):
    """MLP in dense / shift / moe form (ref model.py:506-522); for moe the
    router is drawn BEFORE w1, w2."""
    hidden = int(d * bc["mlp_ratio"])
    mode = bc["mlp_mode"]
    if mode in ("dense", "shift"):
        w1 = _draw_linear(g, d, hidden)
        w2 = _draw_linear(g, hidden, d)
        mk = (lambda w: {"kind": "dense", "w": w}) if mode == "dense" else \
            (lambda w: _shift_layer(w, spec))
        return {"kind": "mlp", "fc1": mk(w1), "fc2": mk(w2)}
    if mode == "moe":
        wg = _draw_linear(g, d, 2, scale=0.02)
        w1 = _draw_linear(g, d, hidden)
        w2 = _draw_linear(g, hidden, d)
        return {"kind": "moe", "wg": wg, "experts": [
            {"kind": "mlp", "fc1": {"kind": "dense", "w": w1}, "fc2": {"kind": "dense", "w": w2}},
            {"kind": "mlp", "fc1": _shift_layer(w1.copy(), spec),
             "fc2": _shift_layer(w2.copy(), spec)}]}
    raise ValueError(mode)


def stage_tokens(spec, si):
    """Token count of stage si (before an optional cls token)."""
    side = spec["img"]
    for st in spec["stages"][: si + 1]:
        side //= st["patch"]
    return side * side


def build(spec: dict) -> dict:
    """All parameters of `spec`, drawn from one PCG64 stream."""
    g = ops.rng(spec["seed"])
    c_in = spec.get("channels", 3)
    net = {"spec": spec, "stages": []}
    for si, st in enumerate(spec["stages"]):
        d = st["d"]
        S = {"pe": _draw_linear(g, st["patch"] * st["patch"] * c_in, d), "blocks": []}
        n = stage_tokens(spec, si) + (1 if st.get("cls_token") else 0)
        if st.get("cls_token"):
            S["cls"] = (g.standard_normal((1, d)) * 0.02).astype(F32)
        if st.get("pos"):
            S["pos"] = (g.standard_normal((n, d)) * 0.02).astype(F32)
        for bc in st["blocks"]:
            B = {"cfg": bc, "d": d}
            B["proj"] = {k: _linear(bc["attn_linear_mode"], g, d, d, spec) for k in "qkvo"}
            if bc["attn_mode"] != "softmax":
                dwi = spec.get("dw_init", "zeros")
                if isinstance(dwi, (int, float)):   # drawn in place from the main stream
                    B["dw"] = (g.standard_normal((3, 3, d)) * float(dwi)).astype(F32)
                else:                               # zeros, maybe filled from a side stream below
                    B["dw"] = np.zeros((3, 3, d), F32)
            else:
                B["dw"] = None
            B["mlp"] = _mlp(bc, d, g, spec)
            S["blocks"].append(B)
        net["stages"].append(S)
        c_in = d
    net["head"] = _draw_linear(g, spec["stages"][-1]["d"], spec["classes"], scale=0.01)
    dwi = spec.get("dw_init", "zeros")
    if isinstance(dwi, dict):   # side stream, block order, after all main draws
        g2 = ops.rng(dwi["seed"])
        for S in net["stages"]:
            for B in S["blocks"]:
                if B["dw"] is not None:
                    B["dw"][...] = (g2.standard_normal(B["dw"].shape) * dwi["std"]).astype(F32)
    return net


def iter_weights(net):
    """(name, array) for every parameter, in a fixed order (for checksums and
    for handing weights to the GPU in tests)."""
    for si, S in enumerate(net["stages"]):
        yield f"s{si}.pe", S["pe"]
        for key in ("cls", "pos"):
            if key in S:
                yield f"s{si}.{key}", S[key]
        for bi, B in enumerate(S["blocks"]):
            pre = f"s{si}.b{bi}"
            for k in "qkvo":
                yield from _iter_layer(f"{pre}.attn.{k}", B["proj"][k])
            if B["dw"] is not None:
                yield f"{pre}.attn.dw", B["dw"]
            yield from _iter_layer(f"{pre}.mlp", B["mlp"])
    yield "head", net["head"]


def _iter_layer(name, L):
    if L["kind"] in ("dense", "shift"):
        yield name + ".w", L["w"]
    elif L["kind"] == "mlp":
        yield from _iter_layer(name + ".fc1", L["fc1"])
        yield from _iter_layer(name + ".fc2", L["fc2"])
    else:
        yield name + ".wg", L["wg"]
        for e, ex in enumerate(L["experts"]):
            yield from _iter_layer(f"{name}.expert{e}", ex)


# ---------------------------------------------------------------------------
# forward


class Trace:
    """Collects per-layer intermediates when passed to `forward`."""

    def __init__(self):
        self.attn = []   # dicts: name, q, k, v, merged
        self.moe = []    # dicts: name, x, expert_of, gate, perm

    def by_name(self, kind):
        return {r["name"]: r for r in getattr(self, kind)}


def linear_fwd(L, x, name="", trace=None):
    kind = L["kind"]
    if kind == "dense":
        return ops.mm(x, L["w"])                                   # ref model.py:104-107
    if kind == "shift":
        return ops.mm(x, ops.shift_weights(L["s"], L["p"], x.dtype))  # ref quantize.py:104-109
    if kind == "mlp":
        return linear_fwd(L["fc2"], ops.gelu_tanh(linear_fwd(L["fc1"], x)))  # ref model.py:204-208
    if kind == "moe":
        return moe_fwd(L, x, name, trace)
    raise ValueError(kind)


def moe_fwd(L, x, name="", trace=None):
    """Route, gather, expert, ×gate, scatter (ref model.py:250-274)."""
    p, _ = ops.router_probs(x, L["wg"])
    expert_of, gate, index_of = ops.dispatch_plan(p)
    if trace is not None:
        trace.moe.append({"name": name, "x": x, "expert_of": expert_of,
                          "gate": gate, "perm": np.concatenate(index_of)})
    out = None
    for e, ex in enumerate(L["experts"]):
        idx = index_of[e]
        if idx.size == 0:
            continue
        y = linear_fwd(ex, x[idx])
        if out is None:
            out = np.zeros((x.shape[0], y.shape[1]), y.dtype)
        out[idx] = y * gate[idx, None]
    return out if out is not None else np.zeros_like(x)


def attention_fwd(B, x, name="", trace=None):
    """Multi-head attention over (batch, n, d) (ref model.py:340-377)."""
    bc = B["cfg"]
    b, n, d = x.shape
    h = bc["h"]
    flat = x.reshape(b * n, d)
    q = linear_fwd(B["proj"]["q"], flat, name + ".q", trace)
    k = linear_fwd(B["proj"]["k"], flat, name + ".k", trace)
    v = linear_fwd(B["proj"]["v"], flat, name + ".v", trace)

    def fold(t):  # ref model.py:330-333
        return ops.heads_split(t.reshape(b, n, d), h).reshape(b * h, n, d // h)

    qh, kh, vh = fold(q), fold(k), fold(v)
    mode = bc["attn_mode"]
    rec = {"name": name, "q": q, "k": k, "v": v} if trace is not None else None
    if mode == "softmax":
        out = ops.softmax_core(qh, kh, vh)
    elif mode == "linear-binary":
        qf, gq = ops.binary_features(qh)
        kf, gk = ops.binary_features(kh)
        out = ops.qkv_linear_core(qf, kf, vh, ops.ATTN_EPS)
        if rec is not None:
            rec.update(gq=gq.reshape(b, h), gk=gk.reshape(b, h),
                       codes_q=ops.pack_codes(qh), codes_k=ops.pack_codes(kh))
    else:
        raise ValueError(f"attention mode {mode!r} is outside the inference hot path")
    merged = ops.heads_merge(out.reshape(b, h, n, d // h)).reshape(b * n, d)  # ref model.py:335-338
    if mode != "softmax" and B["dw"] is not None:                 # ref model.py:367-373
        conv = np.concatenate([ops.dwconv_tokens(v[i * n:(i + 1) * n], B["dw"]) for i in range(b)])
        merged = merged + conv
    if rec is not None:
        rec["merged"] = merged
        trace.attn.append(rec)
    return linear_fwd(B["proj"]["o"], merged, name + ".o", trace).reshape(b, n, d)


def block_fwd(B, x, name="", trace=None):
    """Pre-norm residual block (ref model.py:454-459); LN gain 1, bias 0."""
    b, n, d = x.shape
    one, zero = np.ones(d, F32), np.zeros(d, F32)
    h = x + attention_fwd(B, ops.layer_norm(x, one, zero), name + ".attn", trace)
    flat = ops.layer_norm(h, one, zero).reshape(b * n, d)
    return h + linear_fwd(B["mlp"], flat, name + ".mlp", trace).reshape(b, n, d)


def patchify(grid: np.ndarray, p: int) -> np.ndarray:
    """(B, H, W, C) → (B, (H/p)(W/p), p·p·C), (row, col) × (py, px, c) order
    (ref model.py:557-563)."""
    b, hh, ww, c = grid.shape
    x = grid.reshape(b, hh // p, p, ww // p, p, c).transpose(0, 1, 3, 2, 4, 5)
    return np.ascontiguousarray(x).reshape(b, (hh // p) * (ww // p), p * p * c)


def forward(net: dict, images: np.ndarray, trace: Trace = None) -> np.ndarray:
    """Logits (B, classes) float32 (ref model.py:565-577, chained per stage)."""
    spec = net["spec"]
    grid = np.asarray(images, dtype=F32) - 0.5
    tok = None
    nst = len(net["stages"])
    for si, (st, S) in enumerate(zip(spec["stages"], net["stages"])):
        b = grid.shape[0]
        patches = patchify(grid, st["patch"])
        _, n, pd = patches.shape
        d = st["d"]
        tok = ops.mm(patches.reshape(b * n, pd), S["pe"]).reshape(b, n, d)
        if "cls" in S:
            tok = np.concatenate([np.broadcast_to(S["cls"], (b, 1, d)), tok], axis=1)
        if "pos" in S:
            tok = tok + S["pos"]
        one, zero = np.ones(d, F32), np.zeros(d, F32)
        if st.get("embed_norm"):
            tok = ops.layer_norm(tok, one, zero)
        for bi, B in enumerate(S["blocks"]):
            tok = block_fwd(B, tok, f"s{si}.b{bi}", trace)
        if st.get("stage_norm"):
            tok = ops.layer_norm(tok, one, zero)
        if si + 1 < nst:
            side = int(round(np.sqrt(n)))
            grid = tok.reshape(b, side, side, d)
    pooled = tok[:, 0] if spec.get("pool", "mean") == "cls" else tok.mean(axis=1)
    return ops.mm(np.ascontiguousarray(pooled), net["head"])
