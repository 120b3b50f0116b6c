"""Teacher-forced kernel-boundary parity at the FULL 224² shapes of the
BASELINE configs C3 (PVTv1-Tiny MoE), C4 (DeiT-T, 197 tokens, quadratic
Hamming order) and C5 (PVTv2-B2) — SURVEY §0.5 tier 1.

The oracle runs the whole forward on the host (one image) and records every
binary attention layer's q / k / v / merged output and every MoE layer's
input and plan. Each GPU kernel is then fed the oracle's own fp32 inputs:

* sign-hash (K1): codes bit-exact, gamma within 2e-6;
* popcounts cnt / D of the binary core: integer, bit-exact;
* binary attention + DWConv (K2a linear order, K2b quadratic order) on the
  oracle's codes, gammas and V: within 1e-5 of max|merged|;
* routing + stable partition (K4): winners and permutation bit-exact, gates
  within 1e-6.

End-to-end logits / flip statistics of the same configs are in
test_gpu_model.py (golden fixtures of the real reference)."""

import numpy as np
import pytest
import torch

from oracle import nets, ops
from paper_2306_06446_b200 import specs

pytestmark = pytest.mark.gpu
F32 = np.float32


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.detach().cpu().numpy()


def rel_err(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))


_TRACES = {}


def oracle_trace(name):
    if name not in _TRACES:
        spec = specs.BUILDERS[name]()
        net = nets.build(spec)
        images = ops.rng(31).uniform(0, 1, (1, 224, 224, 3)).astype(F32)
        tr = nets.Trace()
        nets.forward(net, images, tr)
        blocks = {f"s{si}.b{bi}": B for si, S in enumerate(net["stages"])
                  for bi, B in enumerate(S["blocks"])}
        _TRACES[name] = (net, blocks, tr)
    return _TRACES[name]


CONFIGS = ["pvt_v1_tiny", "deit_tiny", "pvt_v2_b2"]


@pytest.mark.parametrize("name", CONFIGS)
def test_sign_hash_and_binary_core_teacher_forced(name):
    from paper_2306_06446_b200 import attention as A
    from paper_2306_06446_b200.quantize import sign_hash
    _, blocks, tr = oracle_trace(name)
    checked = 0
    for rec in tr.attn:
        if "codes_q" not in rec:
            continue
        B = blocks[rec["name"].rsplit(".", 1)[0]]
        h = B["cfg"]["h"]
        d = B["d"]
        n = rec["q"].shape[0]       # batch 1
        dk = d // h
        cq, gq = sign_hash(dev(rec["q"]), h, 1)
        ck, gk = sign_hash(dev(rec["k"]), h, 1)
        assert np.array_equal(host(cq).view(np.uint32).reshape(h, n, -1), rec["codes_q"]), rec["name"]
        assert np.array_equal(host(ck).view(np.uint32).reshape(h, n, -1), rec["codes_k"]), rec["name"]
        assert rel_err(host(gq), rec["gq"]) < 2e-6
        assert rel_err(host(gk), rec["gk"]) < 2e-6
        # integer statistics of the core: cnt_a = sum_j ck_ja, D_i = sum_a cq_ia cnt_a
        cnt, D, _ = A.binary_popcounts(cq, ck, dk)
        bq = ops.code_bits(ops.heads_split(rec["q"].reshape(1, n, d), h).reshape(h, n, dk))
        bk = ops.code_bits(ops.heads_split(rec["k"].reshape(1, n, d), h).reshape(h, n, dk))
        cnt_ref = bk.astype(np.int64).sum(axis=1)
        D_ref = np.einsum("hna,ha->hn", bq.astype(np.int64), cnt_ref)
        assert np.array_equal(host(cnt), cnt_ref)
        assert np.array_equal(host(D), D_ref)
        # the core (+ DWConv on V) fed the oracle's codes, gammas and V
        order = "quadratic" if B["cfg"].get("binary_order") == "quadratic" else "linear"
        dw = dev(B["dw"]) if B["dw"] is not None else None
        merged = A.binary_core_codes(dev(rec["codes_q"].view(np.int32).reshape(1, h, n, -1)),
                                     dev(rec["codes_k"].view(np.int32).reshape(1, h, n, -1)),
                                     dev(rec["gq"]), dev(rec["gk"]), dev(rec["v"]), 1, h, dw,
                                     A.EPS_NORM, order)
        assert rel_err(host(merged), rec["merged"]) < 1e-5, rec["name"]
        checked += 1
    assert checked >= 6


@pytest.mark.parametrize("name", CONFIGS)
def test_routing_teacher_forced(name):
    from paper_2306_06446_b200 import moe as MOE
    net, blocks, tr = oracle_trace(name)
    assert tr.moe
    for rec in tr.moe:
        bname, _, rest = rec["name"].partition(".attn.") if ".attn." in rec["name"] else \
            (rec["name"].rsplit(".", 1)[0], "", "mlp")
        B = blocks[bname]
        L = B["mlp"] if rest == "mlp" else B["proj"][rest]
        plan, _ = MOE.route_plan(dev(rec["x"]), dev(L["wg"]))
        assert np.array_equal(plan.expert_of, rec["expert_of"]), rec["name"]
        assert np.array_equal(np.concatenate(plan.index_of), rec["perm"]), rec["name"]
        assert rel_err(plan.gate_of, rec["gate"]) < 1e-6, rec["name"]


def test_balanced_routers_pvt_b0():
    """PVTv2-B0 with the latency-aware routers (trained by the reference's
    router-only procedure, paper_2306_06446_b200/data): routes bit-exact when
    each MoE layer is fed the oracle's input, logits within tier 3 end to end,
    and the shift expert takes the majority of the tokens."""
    from paper_2306_06446_b200 import model as MD
    from paper_2306_06446_b200 import moe as MOE
    from paper_2306_06446_b200 import routers
    import bench
    rs = routers.load_balanced("pvt_v2_b0")
    spec = specs.pvt_v2_b0()
    m = rs.apply_model(MD.Network(spec))
    net = nets.build(spec)
    bench.apply_router_oracle(rs, net)
    images = ops.rng(41).uniform(0, 1, (2, 224, 224, 3)).astype(F32)
    tr = nets.Trace()
    ref = nets.forward(net, images, tr)
    got = host(m.forward(dev(images)))
    assert rel_err(got, ref) < 2e-3
    assert np.array_equal(got.argmax(1), ref.argmax(1))
    wg = dict(rs.weights)
    for rec in tr.moe:
        plan, _ = MOE.route_plan(dev(rec["x"]), dev(wg[rec["name"]]))
        assert np.array_equal(plan.expert_of, rec["expert_of"]), rec["name"]
    shares = routers.RouterSet.shares(m)
    assert shares["overall"] > 0.6, shares
