"""Pin the numpy oracle to the real reference: every golden vector produced by
tests/golden/make_golden.py (which imports the unmodified reference package)
must be reproduced bit-for-bit by oracle/. CPU only."""

import hashlib

import numpy as np
import pytest

from oracle import nets, ops
from paper_2306_06446_b200 import specs

F32 = np.float32


def test_quantize_shift_kat(golden):
    k = golden("kat")
    s, p = ops.shift_quantize(k["qs_w"])
    assert np.array_equal(s, k["qs_s"]) and np.array_equal(p, k["qs_p"])
    rec = ops.shift_weights(s, p)
    assert np.array_equal(rec.view(np.uint32), k["qs_rec"].view(np.uint32))
    # the reference's own KATs (ref tests/test_quantize.py:15-42)
    s1, p1 = ops.shift_quantize(np.array([[0.75, -0.3, 0.0, -0.0, 1.0]], F32))
    assert s1.tolist() == [[1, -1, 1, 1, 1]] and p1.tolist() == [[0, -2, -15, -15, 0]]


def test_shift_forward_kat(golden):
    k = golden("kat")
    y = ops.mm(k["sf_x"], ops.shift_weights(k["sf_s"], k["sf_p"]))
    assert np.array_equal(y, k["sf_y"])


def test_sign_edge_cases(golden):
    k = golden("kat")
    got = ops.sign_pm1(k["sign_x"])
    assert np.array_equal(got, k["sign_y"])
    assert ops.code_bits(k["sign_x"]).tolist() == [1, 1, 0, 1, 0, 1, 0, 1]


@pytest.mark.parametrize("dk", [16, 32, 64])
def test_binary_linear_core(golden, dk):
    k = golden("kat")
    pre = f"lc{dk}_"
    qf, gq = ops.binary_features(k[pre + "q"])
    kf, gk = ops.binary_features(k[pre + "k"])
    assert np.array_equal(gq, k[pre + "gq"]) and np.array_equal(gk, k[pre + "gk"])
    out = ops.qkv_linear_core(qf, kf, k[pre + "v"])
    assert np.array_equal(out, k[pre + "out"])
    assert np.all(out[0, 3] == 0)


@pytest.mark.parametrize("n", [5, 196, 197])
def test_dwconv_tokens(golden, n):
    k = golden("kat")
    assert ops.token_grid_side(n) == int(k[f"dw{n}_side"])
    assert np.array_equal(ops.dwconv_tokens(k[f"dw{n}_v"], k[f"dw{n}_k"]), k[f"dw{n}_y"])


def test_softmax_core(golden):
    k = golden("kat")
    assert np.array_equal(ops.softmax_core(k["sm_q"], k["sm_k"], k["sm_v"]), k["sm_out"])


def test_route_dispatch(golden):
    k = golden("kat")
    p, logits = ops.router_probs(k["rt_x"], k["rt_wg"])
    assert np.array_equal(logits, k["rt_logits"]) and np.array_equal(p, k["rt_p"])
    e, gate, idx = ops.dispatch_plan(p)
    assert np.array_equal(e, k["rt_expert"])
    assert np.array_equal(gate, k["rt_gate"])
    assert np.array_equal(np.concatenate(idx), k["rt_perm"])


def test_tie_threshold_rule(golden):
    """The 2-expert rule the GPU router implements: expert 1 iff
    f32(l_min - l_max) < -threshold, i.e. iff the deficit exceeds numpy's exp
    threshold."""
    k = golden("kat")
    thr = ops.numpy_exp_tie_threshold()
    assert thr == k["tie_threshold"]
    tl = k["tie_logits"]
    lo = np.minimum(tl[:, 0], tl[:, 1])
    hi = np.maximum(tl[:, 0], tl[:, 1])
    shifted = (lo - hi).astype(F32)
    rule = np.where(tl[:, 1] > tl[:, 0], (-shifted > thr).astype(np.int32), 0)
    assert np.array_equal(rule, k["tie_expert"])
    p = ops.softmax_rows(tl)
    e, gate, _ = ops.dispatch_plan(p)
    assert np.array_equal(e, k["tie_expert"]) and np.array_equal(gate, k["tie_gate"])


def test_moe_forward(golden):
    k = golden("kat")
    w = k["mf_w"]
    s, p = ops.shift_quantize(w)
    L = {"kind": "moe", "wg": k["mf_wg"],
         "experts": [{"kind": "dense", "w": w}, {"kind": "shift", "w": w, "s": s, "p": p}]}
    assert np.array_equal(nets.moe_fwd(L, k["mf_x"]), k["mf_y"])


def test_layernorm_gelu(golden):
    k = golden("kat")
    d = k["ln_x"].shape[1]
    assert np.array_equal(ops.layer_norm(k["ln_x"], np.ones(d, F32), np.zeros(d, F32)), k["ln_y"])
    assert np.array_equal(ops.gelu_tanh(k["gelu_x"]), k["gelu_y"])


def _digest(net):
    h = hashlib.sha256()
    for name, arr in nets.iter_weights(net):
        h.update(name.encode())
        h.update(np.ascontiguousarray(arr).tobytes())
    return h.hexdigest()


MODEL_FIXTURES = {
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


@pytest.mark.parametrize("name", sorted(MODEL_FIXTURES))
def test_model_forward_bit_exact(golden, name):
    fx = golden(name)
    spec = MODEL_FIXTURES[name]()
    net = nets.build(spec)
    assert _digest(net) == str(fx["weight_sha256"]), "weight draw order differs"
    b = int(fx["batch"])
    images = fx["images"] if "images" in fx else ops.rng(int(fx["images_seed"])).uniform(
        0, 1, (b, spec["img"], spec["img"], 3)).astype(F32)
    tr = nets.Trace()
    logits = nets.forward(net, images, tr)
    assert np.array_equal(logits, fx["logits"])
    for rec in tr.moe:
        bits = np.packbits(rec["expert_of"].astype(np.uint8), bitorder="little")
        assert np.array_equal(bits, fx["route:" + rec["name"]]), rec["name"]
        assert np.array_equal(rec["gate"], fx["gate:" + rec["name"]])
    for rec in tr.attn:
        if "codes_q" not in rec:
            continue
        for key in ("q", "k"):
            bits = np.packbits((~(rec[key] < 0)).astype(np.uint8).ravel(), bitorder="little")
            assert np.array_equal(bits, fx[f"codes:{rec['name']}.{key}"])
        assert np.array_equal(rec["gq"], fx[f"gamma:{rec['name']}.q"])


def test_balanced_router_set_matches_model_layout():
    """The committed latency-aware routers cover exactly the MoE layers of
    PVTv2-B0 with (d, 2) f32 matrices, and reached the latency-balanced split
    on their training tokens wherever a bias-free router can split them."""
    from paper_2306_06446_b200 import routers
    rs = routers.load_balanced("pvt_v2_b0")
    net = nets.build(specs.pvt_v2_b0())
    names = {}
    for si, S in enumerate(net["stages"]):
        for bi, B in enumerate(S["blocks"]):
            for key in "qkvo":
                if B["proj"][key]["kind"] == "moe":
                    names[f"s{si}.b{bi}.attn.{key}"] = B["proj"][key]["wg"].shape
            if B["mlp"]["kind"] == "moe":
                names[f"s{si}.b{bi}.mlp"] = B["mlp"]["wg"].shape
    assert set(rs.weights) == set(names)
    for k, shape in names.items():
        assert rs.weights[k].shape == shape and rs.weights[k].dtype == np.float32
    near = [k for k, s in rs.train_shares.items() if abs(s - 0.75) <= 0.10]
    assert len(near) >= len(names) // 2


def test_oracle_add_matmul_golden(golden):
    """MatAdd restatement = the reference's add_matmul bit for bit (ref
    quantize.py:143-160) on its own KATs and binarized random layers."""
    k = golden("addlinear")
    assert np.array_equal(ops.add_matmul(k["hand_x"], k["hand_b"], 1.0), k["hand_y"])
    for i in range(4):
        y = ops.add_matmul(k[f"x{i}"], k[f"b{i}"], float(k[f"g{i}"]))
        assert np.array_equal(y, k[f"y{i}"]), i
