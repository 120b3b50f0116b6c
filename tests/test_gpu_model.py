"""End-to-end parity of the device models against the oracle and the golden
fixtures produced by the real reference.

fp32 contract: logits within 1e-5 of max|logit|; hash codes and
router winners bit-exact at every layer when each layer is fed the oracle's
inputs (teacher forcing), and reported (expected 0) end to end."""

import hashlib

import numpy as np
import pytest
import torch

from oracle import nets, ops
from paper_2306_06446_b200 import specs

pytestmark = pytest.mark.gpu
F32 = np.float32
LOGIT_TOL = 1e-5


# Deep configs (C3 / C4 / C5 at 224²): the tensor-core fp32-parity GEMMs
# accumulate in TMEM fp32, whose error grows with K (scripts/diag_gemm_ulp.py:
# max|err|/rms 2e-6 at K = 32, 7e-5 at K = 2048, profiles/r2_gemm_ulp.txt), so
# over 8-12 blocks an input lying within that error of a sign boundary flips a
# code or a route and the flip cascades downstream. For these the
# end-to-end contract is tier 3: logits within the stated tolerance, top-1
# agreement, and a bounded flip RATE; tier 1 (bit-exact codes, popcounts,
# routes, permutations on the oracle's own inputs) is pinned at the same full
# shapes in test_gpu_configs.py. Shallow fixtures keep tier 2 (1e-5, 0 flips).
# The same cascade is why a single flip can also appear at the benchmark shape
# of PVTv2-B0 on other images (bench.py's gate uses tier 3 for every config).
# Tier 3: (logit tolerance relative to max|logit|, max code-flip rate, max
# route-flip rate), measured worst case DeiT-T 5.5e-4 / 5.5e-5 / 1.8e-4.
TIER3 = (2e-3, 1e-4, 5e-4)
DEEP = {"pvt_v1_tiny_full": TIER3, "pvt_v2_b2_full": TIER3, "deit_tiny_full": TIER3}


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.detach().cpu().numpy()


def rel_err(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))


def digest(named):
    h = hashlib.sha256()
    for name, arr in named:
        h.update(name.encode())
        a = arr.detach().cpu().numpy() if isinstance(arr, torch.Tensor) else arr
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


FIXTURES = {
    "toy_c1": lambda: specs.toy_c1(),
    "toy_c1_moe": lambda: specs.toy_c1(attn_linear_mode="moe", mlp_mode="moe"),
    "pvt_small": lambda: specs.pvt_v2_b0(img=64, classes=10),
    "deit_small": lambda: specs.deit_tiny(img=64, classes=10, depth=3),
    "pvt_b0_full": lambda: specs.pvt_v2_b0(),
    # BASELINE configs C3 / C4 / C5 at full 224 (batch 2)
    "pvt_v1_tiny_full": lambda: specs.pvt_v1_tiny(),
    "deit_tiny_full": lambda: specs.deit_tiny(),
    "pvt_v2_b2_full": lambda: specs.pvt_v2_b2(),
}


def capture_device(model):
    """Wrap the binary core to record the packed q / k codes it is given (the
    fused attention-input kernel and the unfused sign-hash both feed it)."""
    from paper_2306_06446_b200 import attention as A
    recs = {"codes": {}, "plans": {}}
    orig = A.binary_core_codes

    def binary_core_codes(cq, ck, gq, gk, v, batch, heads, dw=None, eps=A.EPS_NORM, order="auto"):
        dk = v.shape[1] // heads
        recs["codes"].setdefault("q", []).append((cq.clone(), dk))
        recs["codes"].setdefault("k", []).append((ck.clone(), dk))
        return orig(cq, ck, gq, gk, v, batch, heads, dw, eps, order)
    A.binary_core_codes = binary_core_codes
    return recs, lambda: setattr(A, "binary_core_codes", orig)


def code_bits(rec):
    """([B, H, n, W] packed words, dk) → the reference's sign bits of the flat
    (B·n, d) projection, packed little-endian (the golden 'codes:' layout)."""
    codes, dk = rec
    c = host(codes).view(np.uint32)
    B, H, n, W = c.shape
    bits = ((c[..., None] >> np.arange(32, dtype=np.uint32)) & 1).astype(np.uint8)   # B,H,n,W,32
    bits = bits.reshape(B, H, n, W * 32)[..., :dk].transpose(0, 2, 1, 3).reshape(-1)
    return np.packbits(bits, bitorder="little")


@pytest.mark.parametrize("name", sorted(FIXTURES))
def test_model_vs_golden(golden, name):
    from paper_2306_06446_b200 import model as MD
    fx = golden(name)
    spec = FIXTURES[name]()
    m = MD.Network(spec)
    assert digest(m.named_weights()) == str(fx["weight_sha256"]), "weights differ from reference"
    b = int(fx["batch"])
    images = fx["images"] if "images" in fx else ops.rng(int(fx["images_seed"])).uniform(
        0, 1, (b, spec["img"], spec["img"], 3)).astype(F32)
    recs, restore = capture_device(m)
    try:
        logits = host(m.forward(dev(images)))
    finally:
        restore()
    # end-to-end code / route agreement (fp32 path), counted per layer first
    per_layer = []
    total = 0
    names = [k[len("codes:"):] for k in fx if k.startswith("codes:")]
    qs = [n for n in names if n.endswith(".q")]
    ks = [n for n in names if n.endswith(".k")]
    assert len(recs["codes"].get("q", [])) == len(qs), "codes of every binary layer recorded"
    for key_list, tag in ((qs, "q"), (ks, "k")):
        for got, key in zip(recs["codes"].get(tag, []), key_list):
            bits = code_bits(got)
            f = int(np.unpackbits(bits ^ fx["codes:" + key]).sum())
            total += bits.size * 8
            if f:
                per_layer.append((key, f))
    flips = sum(f for _, f in per_layer)
    route_flips = 0
    for lname, mod in m.moe_modules():
        bits = np.packbits(mod.last_plan.expert_of.astype(np.uint8), bitorder="little")
        f = int(np.unpackbits(bits ^ fx["route:" + lname]).sum())
        route_flips += f
        if f:
            per_layer.append((lname, f))
    err = rel_err(logits, fx["logits"])
    print(f"{name}: logits rel {err:.2e}, {flips} / {total} code flips, "
          f"{route_flips} route flips, per layer {per_layer}")
    assert np.array_equal(logits.argmax(1), fx["logits"].argmax(1))
    if name in DEEP:
        tol, code_rate, route_rate = DEEP[name]
        routed = sum(mod.last_plan.expert_of.size for _, mod in m.moe_modules())
        assert err < tol
        assert flips <= code_rate * total, f"{flips} / {total} code flips"
        assert route_flips <= route_rate * routed, f"{route_flips} / {routed} route flips"
        return
    assert err < LOGIT_TOL
    assert flips == 0, f"{flips} / {total} code flips"
    assert route_flips == 0, f"{route_flips} route flips"


@pytest.mark.parametrize("name", ["toy_c1_moe", "pvt_small", "deit_small"])
def test_teacher_forced_layers_bit_exact(golden, name):
    """Each MoE layer fed the REFERENCE's captured input must reproduce the
    reference's winners bit-exactly (SURVEY §0.5 tier 1)."""
    from paper_2306_06446_b200 import moe as MOE
    fx = golden(name)
    net = nets.build(FIXTURES[name]())
    m_inputs = {k[len("moe_x:"):]: v for k, v in fx.items() if k.startswith("moe_x:")}
    assert m_inputs
    wg = {}
    for si, S in enumerate(net["stages"]):
        for bi, B in enumerate(S["blocks"]):
            for key in "qkvo":
                L = B["proj"][key]
                if L["kind"] == "moe":
                    wg[f"s{si}.b{bi}.attn.{key}"] = L["wg"]
            if B["mlp"]["kind"] == "moe":
                wg[f"s{si}.b{bi}.mlp"] = B["mlp"]["wg"]
    for lname, x in m_inputs.items():
        plan, _ = MOE.route_plan(dev(x), dev(wg[lname]))
        bits = np.packbits(plan.expert_of.astype(np.uint8), bitorder="little")
        assert np.array_equal(bits, fx["route:" + lname]), lname
        assert rel_err(plan.gate_of, fx["gate:" + lname]) < 1e-6


def test_reference_model_class_api():
    """`Model(ModelConfig)` holds exactly the reference Model's parameters and
    runs the same forward (ref model.py:525-577)."""
    from paper_2306_06446_b200 import model as MD
    bcs = [MD.BlockConfig(d=64, h=4, mlp_ratio=4.0, attn_mode="linear-binary",
                          mlp_mode="shift", attn_linear_mode="shift") for _ in range(2)]
    m = MD.Model(MD.ModelConfig(blocks=bcs, patch=4, img=56, classes=10, seed=0))
    spec = dict(specs.toy_c1())
    spec["dw_init"] = "zeros"
    net = nets.build(spec)
    assert digest(m.named_weights()) == digest(nets.iter_weights(net))
    images = ops.rng(1).uniform(0, 1, (4, 56, 56, 3)).astype(F32)
    assert rel_err(host(m.forward(dev(images))), nets.forward(net, images)) < LOGIT_TOL


def test_pvt_b0_full_batch_properties():
    """PVTv2-B0 at the benchmark batch (256): deterministic, finite, every token
    routed exactly once, per-image logits independent of batching."""
    from paper_2306_06446_b200 import model as MD
    m = MD.pvt_v2_b0()
    g = ops.rng(11)
    images = dev(g.uniform(0, 1, (256, 224, 224, 3)).astype(F32))
    a = m.forward(images)
    b = m.forward(images)
    la, lb = host(a), host(b)
    assert np.isfinite(la).all()
    assert np.array_equal(la, lb), "forward is not deterministic"
    for _, mod in m.moe_modules():
        plan = mod.last_plan
        seen = np.sort(np.concatenate(plan.index_of))
        assert np.array_equal(seen, np.arange(plan.expert_of.size))
    part = host(m.forward(images[:8].contiguous()))
    assert rel_err(part, la[:8]) < 1e-5
    # oracle on two of the images
    net = nets.build(specs.pvt_v2_b0())
    ref = nets.forward(net, host(images[:2]))
    assert rel_err(la[:2], ref) < LOGIT_TOL


BENCH_BATCH = {   # BASELINE.json configs at their benchmark batch per GPU
    "pvt_v1_tiny": 256,   # C3
    "deit_tiny": 512,     # C4
    "pvt_v2_b2": 256,     # C5 (global 2048 over 8 GPUs)
}
# (pvt_v2_b0 at batch 256 is test_pvt_b0_full_batch_properties)


@pytest.mark.parametrize("name", sorted(BENCH_BATCH))
def test_config_full_batch_properties(name):
    """C3 / C4 / C5 at the benchmark batch: deterministic, finite, every token
    routed exactly once, logits independent of batching, and the oracle on two
    of the benchmarked images within the fp32 tolerance."""
    from paper_2306_06446_b200 import model as MD
    spec = specs.BUILDERS[name]()
    m = MD.Network(spec)
    B = BENCH_BATCH[name]
    g = ops.rng(12)
    images = dev(g.uniform(0, 1, (B, 224, 224, 3)).astype(F32))
    la = host(m.forward(images))
    lb = host(m.forward(images))
    assert np.isfinite(la).all()
    assert np.array_equal(la, lb), "forward is not deterministic"
    for _, mod in m.moe_modules():
        plan = mod.last_plan
        seen = np.sort(np.concatenate(plan.index_of))
        assert np.array_equal(seen, np.arange(plan.expert_of.size))
    part = host(m.forward(images[B - 4:].contiguous()))
    assert rel_err(part, la[B - 4:]) < 1e-5
    ref = nets.forward(nets.build(spec), host(images[B - 2:]))
    assert rel_err(la[B - 2:], ref) < DEEP[name + "_full"][0]
    assert np.array_equal(la[B - 2:].argmax(1), ref.argmax(1))


@pytest.mark.parametrize("name", ["toy_c1_moe", "pvt_small", "pvt_b0_full"])
def test_fused_qkv_matches_unfused(golden, name):
    """sa_ln_qkv_hash (LN1 + routers + q/k/v + sign-hash in one kernel) against
    the unfused chain (LN+routers, three MoE projections, two sign-hash calls):
    identical routes and codes, logits within fp32 summation noise."""
    from paper_2306_06446_b200 import model as MD
    fx = golden(name)
    spec = FIXTURES[name]()
    m = MD.Network(spec)
    b = int(fx["batch"])
    images = fx["images"] if "images" in fx else ops.rng(int(fx["images_seed"])).uniform(
        0, 1, (b, spec["img"], spec["img"], 3)).astype(F32)
    x = dev(images)
    old = MD.FUSE_QKV
    try:
        MD.FUSE_QKV = False
        recs0, restore = capture_device(m)
        ref = host(m.forward(x))
        restore()
        plans_ref = [mod.last_plan.expert_of.copy() for _, mod in m.moe_modules()]
        MD.FUSE_QKV = True
        recs1, restore = capture_device(m)
        got = host(m.forward(x))
        restore()
        plans = [mod.last_plan.expert_of.copy() for _, mod in m.moe_modules()]
        idx = [mod.last_plan.index_of for _, mod in m.moe_modules()]
    finally:
        MD.FUSE_QKV = old
    for a, c in zip(plans, plans_ref):
        assert np.array_equal(a, c)
    for e, ix in zip(plans, idx):   # lazily materialised stable partition
        assert np.array_equal(ix[0], np.flatnonzero(e == 0))
        assert np.array_equal(ix[1], np.flatnonzero(e == 1))
    for key in ("q", "k"):
        for (c0, _), (c1, _) in zip(recs0["codes"][key], recs1["codes"][key]):
            assert np.array_equal(host(c0), host(c1))
    assert rel_err(got, ref) < 1e-6
    assert rel_err(got, fx["logits"]) < LOGIT_TOL


@pytest.mark.parametrize("name", ["toy_c1_moe", "pvt_small", "pvt_b0_full"])
def test_fused_wo_ln2_route_bit_identical(golden, name):
    """sa_fused_moe_linear_ln_route (W_O + residual, then LN2 and the MLP
    router in the same kernel's epilogue) reproduces sa_fused_moe_linear +
    sa_ln_route exactly: identical logits and identical routes of every MoE
    layer."""
    from paper_2306_06446_b200 import model as MD
    fx = golden(name)
    spec = FIXTURES[name]()
    m = MD.Network(spec)
    b = min(int(fx["batch"]), 4)
    images = fx["images"][:b] if "images" in fx else ops.rng(int(fx["images_seed"])).uniform(
        0, 1, (b, spec["img"], spec["img"], 3)).astype(F32)
    x = dev(images)
    old = MD.FUSE_LN2
    try:
        MD.FUSE_LN2 = False
        ref = host(m.forward(x))
        plans_ref = [mod.last_plan.expert_of.copy() for _, mod in m.moe_modules()]
        MD.FUSE_LN2 = True
        got = host(m.forward(x))
        plans = [mod.last_plan.expert_of.copy() for _, mod in m.moe_modules()]
        perms = [(mod.last_plan.expert_of.copy(), mod.last_plan.index_of) for _, mod in m.moe_modules()]
    finally:
        MD.FUSE_LN2 = old
    assert np.array_equal(got, ref)
    for a, c in zip(plans, plans_ref):
        assert np.array_equal(a, c)
    for e, ix in perms:   # the lazily built stable partition of the fused routes
        assert np.array_equal(ix[0], np.flatnonzero(e == 0))
        assert np.array_equal(ix[1], np.flatnonzero(e == 1))


@pytest.mark.parametrize("name", ["pvt_small", "pvt_b0_full"])
def test_fused_stage_layernorm_bit_identical(golden, name):
    """sa_tc_moe_mlp_fused_ln (the stage's final LayerNorm in the last block's
    fused MLP, d = 32) reproduces the fused MLP + sa_layernorm exactly."""
    from paper_2306_06446_b200 import model as MD
    fx = golden(name)
    spec = FIXTURES[name]()
    m = MD.Network(spec)
    b = min(int(fx["batch"]), 4)
    images = fx["images"][:b] if "images" in fx else ops.rng(int(fx["images_seed"])).uniform(
        0, 1, (b, spec["img"], spec["img"], 3)).astype(F32)
    x = dev(images)
    old = MD.FUSE_STAGE_LN
    try:
        MD.FUSE_STAGE_LN = False
        ref = host(m.forward(x))
        assert not any(S.blocks[-1].post_ln_applied for S in m.stages)
        MD.FUSE_STAGE_LN = True
        got = host(m.forward(x))
        assert all(S.blocks[-1].post_ln_applied for S in m.stages
                   if S.d in (32, 64) and S.stage_ln is not None)
    finally:
        MD.FUSE_STAGE_LN = old
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("name", ["pvt_small", "pvt_b0_full"])
def test_fused_embed_layernorm_bit_identical(golden, name):
    """sa_tc_patch_embed_ln (embedding LayerNorm in the patch GEMM's epilogue)
    reproduces sa_tc_patch_embed + sa_layernorm exactly: identical logits."""
    from paper_2306_06446_b200 import model as MD
    fx = golden(name)
    spec = FIXTURES[name]()
    m = MD.Network(spec)
    b = min(int(fx["batch"]), 4)
    images = fx["images"][:b] if "images" in fx else ops.rng(int(fx["images_seed"])).uniform(
        0, 1, (b, spec["img"], spec["img"], 3)).astype(F32)
    x = dev(images)
    old = MD.FUSE_EMBED_LN
    try:
        MD.FUSE_EMBED_LN = False
        ref = host(m.forward(x))
        MD.FUSE_EMBED_LN = True
        got = host(m.forward(x))
    finally:
        MD.FUSE_EMBED_LN = old
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("name", ["pvt_small", "pvt_b0_full"])
def test_grouped_qkv_projections_bit_identical(golden, name):
    """sa_tc_moe_linear_grouped (the q/k/v MoE projections of a d = 160 stage in
    one launch) computes each problem exactly as sa_tc_moe_linear."""
    from paper_2306_06446_b200 import model as MD
    fx = golden(name)
    spec = FIXTURES[name]()
    m = MD.Network(spec)
    b = min(int(fx["batch"]), 4)
    images = fx["images"][:b] if "images" in fx else ops.rng(int(fx["images_seed"])).uniform(
        0, 1, (b, spec["img"], spec["img"], 3)).astype(F32)
    x = dev(images)
    old = MD.FUSE_GROUPED_QKV
    try:
        MD.FUSE_GROUPED_QKV = False
        ref = host(m.forward(x))
        MD.FUSE_GROUPED_QKV = True
        got = host(m.forward(x))
    finally:
        MD.FUSE_GROUPED_QKV = old
    assert np.array_equal(got, ref)
    assert rel_err(got, fx["logits"][:b]) < LOGIT_TOL


@pytest.mark.parametrize("name", ["pvt_small", "pvt_b0_full"])
def test_dense_qkv_concat_bit_identical(golden, name):
    """The exempt MSA stage's q/k/v as one GEMM against [W_q | W_k | W_v] and
    the strided softmax core reproduce the three-GEMM path exactly."""
    from paper_2306_06446_b200 import model as MD
    fx = golden(name)
    spec = FIXTURES[name]()
    m = MD.Network(spec)
    b = min(int(fx["batch"]), 4)
    images = fx["images"][:b] if "images" in fx else ops.rng(int(fx["images_seed"])).uniform(
        0, 1, (b, spec["img"], spec["img"], 3)).astype(F32)
    x = dev(images)
    old = MD.FUSE_DENSE_QKV
    try:
        MD.FUSE_DENSE_QKV = False
        ref = host(m.forward(x))
        MD.FUSE_DENSE_QKV = True
        got = host(m.forward(x))
    finally:
        MD.FUSE_DENSE_QKV = old
    assert np.array_equal(got, ref)


def test_apply_stage_matches_reference(golden):
    """`apply_stage` (ref model.py:897-930) on a softmax/dense toy Model: the
    same weights (digest), logits and MoE winners as the reference after
    stage 1 (linear-binary attention, zero DW kernels) and stage 2 (MoE
    projections and MLPs with routers drawn from PCG64(77)); exempt block
    untouched."""
    from paper_2306_06446_b200 import model as MD
    fx = golden("apply_stage")
    bcs = [MD.BlockConfig(d=64, h=4, mlp_ratio=4.0, attn_mode="softmax", mlp_mode="dense",
                          attn_linear_mode="dense", exempt=(i == 2)) for i in range(3)]
    m = MD.Model(MD.ModelConfig(blocks=bcs, patch=4, img=32, classes=10, seed=5))
    x = dev(fx["images"])
    assert digest(m.named_weights()) == str(fx["sha0"])
    assert rel_err(host(m.forward(x)), fx["logits0"]) < LOGIT_TOL
    MD.apply_stage(m, 1)
    assert digest(m.named_weights()) == str(fx["sha1"])
    assert all(b.cfg.attn_mode == ("softmax" if b.cfg.exempt else "linear-binary") for b in m.blocks)
    assert rel_err(host(m.forward(x)), fx["logits1"]) < LOGIT_TOL
    MD.apply_stage(m, 2, mlp_target="moe", attn_target="moe")
    assert digest(m.named_weights()) == str(fx["sha2"])
    assert rel_err(host(m.forward(x)), fx["logits2"]) < LOGIT_TOL
    names = [lname for lname, _ in m.moe_modules()]
    assert names[:2] == ["block0.mlp", "block0.attn.q"]   # the reference's names and order
    for lname, mod in m.moe_modules():   # fixture keys use the s<stage>.b<block> form
        key = "route:" + lname.replace("block", "s0.b", 1)
        assert np.array_equal(mod.last_plan.expert_of, fx[key]), lname
    with pytest.raises(ValueError):
        MD.apply_stage(m, 3)


@pytest.mark.parametrize("B,H,C,patch,d", [(3, 224, 3, 4, 32), (2, 56, 32, 2, 64), (1, 8, 3, 4, 32),
                                           (5, 28, 32, 2, 64), (2, 16, 8, 2, 32)])
def test_embed_ln_kernel_bit_identical_to_gemm_path(B, H, C, patch, d, debug_lib):
    """The dedicated patch-embed + LayerNorm kernel (embed_tc.cu) against the
    GEMM path's LNE epilogue (sa_debug_embed_mode(1)): bit-identical tokens,
    ragged last tiles included, and the oracle's embed + LayerNorm within fp32
    tolerance."""
    import ctypes
    from paper_2306_06446_b200 import _lib
    from paper_2306_06446_b200 import model as MD
    lib = debug_lib
    lib.sa_debug_embed_mode.argtypes = [ctypes.c_int]
    g = ops.rng(B * H + C)
    grid = g.uniform(0, 1, (B, H, H, C)).astype(F32)
    K = patch * patch * C
    w = (g.standard_normal((K, d)) / np.sqrt(K)).astype(F32)
    gain = (1 + 0.1 * g.standard_normal(d)).astype(F32)
    bias = (0.1 * g.standard_normal(d)).astype(F32)
    lay = MD.Linear(w)
    pk, bn, _ = lay.tc_pack()
    side = H // patch
    out = {}
    grid_d, gain_d, bias_d = dev(grid), dev(gain), dev(bias)   # alive until the kernels ran
    for mode in (0, 1):
        y = torch.empty((B * side * side, d), dtype=torch.float32, device="cuda")
        lib.sa_debug_embed_mode(mode)
        try:
            _lib.call("sa_tc_patch_embed_ln", _lib.ptr(grid_d), B, H, H, C, patch, 0.5,
                      _lib.ptr(pk), bn, d, _lib.ptr(gain_d), _lib.ptr(bias_d), 1e-5,
                      _lib.ptr(y), _lib.stream())
            torch.cuda.synchronize()
        finally:
            lib.sa_debug_embed_mode(0)
        out[mode] = host(y)
    assert np.array_equal(out[0], out[1])
    patches = (grid - 0.5).reshape(B, side, patch, side, patch, C).transpose(0, 1, 3, 2, 4, 5)
    tok = ops.mm(patches.reshape(B * side * side, K), w)
    ref = ops.layer_norm(tok, gain, bias)
    assert rel_err(out[0], ref) < 1e-5


@pytest.mark.parametrize("M,d", [(1, 32), (127, 32), (129, 64), (1000, 32), (4097, 64)])
def test_wo_ln2_route_kernel_ragged(M, d):
    """sa_fused_moe_linear_ln_route on ragged row counts equals
    sa_fused_moe_linear followed by sa_ln_route on its output, bit for bit
    (h, LN2(h), the MLP routes and gates)."""
    from paper_2306_06446_b200 import _lib
    from paper_2306_06446_b200 import model as MD
    from paper_2306_06446_b200 import moe as MOE
    g = ops.rng(M + d)
    w = (g.standard_normal((d, d)) / np.sqrt(d)).astype(F32)
    o = MD.MoeModule((g.standard_normal((d, 2)) * 0.5).astype(F32),
                     [MD.Linear(w), MD.ShiftLinearLayer(w.copy())], MD.MoeConfig())
    ln = MD.LayerNorm(d)
    ln.gain.value.copy_(torch.from_numpy((1 + 0.1 * g.standard_normal(d)).astype(F32)))
    ln.bias.value.copy_(torch.from_numpy((0.1 * g.standard_normal(d)).astype(F32)))
    wg2 = dev((g.standard_normal((d, 2)) * 0.5).astype(F32))
    x = dev(g.standard_normal((M, d)).astype(F32))
    res = dev(g.standard_normal((M, d)).astype(F32))
    h_ref = o.forward(x, residual=res)
    y_ref, (plan,) = MOE.ln_route_plans(h_ref, ln.gain.value, ln.bias.value, [wg2])
    e1, g1 = torch.empty(M, dtype=torch.int32, device="cuda"), torch.empty(M, device="cuda")
    h, y2 = torch.empty_like(x), torch.empty_like(x)
    e2, g2 = torch.empty(M, dtype=torch.int32, device="cuda"), torch.empty(M, device="cuda")
    _lib.call("sa_fused_moe_linear_ln_route", _lib.ptr(x), _lib.ptr(o.wg.value),
              _lib.ptr(o.experts[0].tc_pack(d)[0]), _lib.ptr(o.experts[1].tc_pack(d)[0]),
              _lib.ptr(res), MOE.tie_threshold(), M, d, _lib.ptr(e1), _lib.ptr(g1), _lib.ptr(h),
              _lib.ptr(ln.gain.value), _lib.ptr(ln.bias.value), 1e-5, _lib.ptr(wg2), _lib.ptr(y2),
              _lib.ptr(e2), _lib.ptr(g2), _lib.stream())
    assert np.array_equal(host(h), host(h_ref))
    assert np.array_equal(host(y2), host(y_ref))
    assert np.array_equal(host(e2), plan.expert_of)
    assert np.array_equal(host(g2), plan.gate_of)


@pytest.mark.parametrize("M,d,hidden", [(1, 32, 256), (130, 32, 256), (777, 64, 512),
                                        (5000, 32, 512)])
def test_mlp_stage_ln_kernel_ragged(M, d, hidden):
    """sa_tc_moe_mlp_fused_ln on ragged row counts equals the fused MoE MLP
    followed by sa_layernorm, bit for bit."""
    from paper_2306_06446_b200 import model as MD
    from paper_2306_06446_b200 import moe as MOE
    from paper_2306_06446_b200 import tensor as T
    g = ops.rng(M * 3 + d)
    w1 = (g.standard_normal((d, hidden)) / np.sqrt(d)).astype(F32)
    w2 = (g.standard_normal((hidden, d)) / np.sqrt(hidden)).astype(F32)
    mod = MD.MoeModule((g.standard_normal((d, 2)) * 0.5).astype(F32),
                       [MD.Mlp(MD.Linear(w1), MD.Linear(w2)),
                        MD.Mlp(MD.ShiftLinearLayer(w1.copy()), MD.ShiftLinearLayer(w2.copy()))],
                       MD.MoeConfig())
    ln = MD.LayerNorm(d)
    ln.gain.value.copy_(torch.from_numpy((1 + 0.1 * g.standard_normal(d)).astype(F32)))
    ln.bias.value.copy_(torch.from_numpy((0.1 * g.standard_normal(d)).astype(F32)))
    x = dev(g.standard_normal((M, d)).astype(F32))
    res = dev(g.standard_normal((M, d)).astype(F32))
    plan, _ = MOE.route_plan(x, mod.wg.value)
    y = mod.forward(x, plan=plan, residual=res)
    ref, _ = T.layernorm(y, ln.gain.value, ln.bias.value)
    got = mod.forward(x, plan=plan, residual=res, post_ln=ln)
    assert mod.post_ln_applied
    assert np.array_equal(host(got), host(ref))
