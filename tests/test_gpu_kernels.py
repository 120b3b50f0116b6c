"""Kernel-boundary parity on the GPU: every kernel is fed the oracle's own
float32 inputs and compared with the oracle (and the golden vectors pinned to
the real reference).

Bars: bit-exact for codes, popcounts, router winners, permutations and shift
codes; float results within the tolerances written in each test (the reference
accumulates in float64, the kernels in float32)."""

import numpy as np
import pytest
import torch

from oracle import nets, ops

pytestmark = pytest.mark.gpu

F32 = np.float32


def dev(a, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.cuda()


def host(t):
    torch.cuda.synchronize()
    return t.detach().cpu().numpy()


def rel_err(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))


# ---------------------------------------------------------------- K1 sign hash


@pytest.mark.parametrize("B,n,d,h", [(2, 196, 64, 4), (3, 3136, 32, 1), (2, 784, 64, 2),
                                     (2, 196, 160, 5), (2, 197, 192, 3), (1, 5, 32, 2),
                                     (2, 49, 256, 8), (3, 300, 96, 3), (2, 513, 320, 10),
                                     (1, 77, 384, 12), (2, 1000, 160, 5)])
def test_sign_hash_codes_bit_exact(B, n, d, h):
    from paper_2306_06446_b200 import quantize as Q
    g = ops.rng(B * 1000 + n)
    x = g.standard_normal((B * n, d)).astype(F32)
    x[0, :7] = [-0.0, 0.0, -1e-45, np.nan, -np.inf, np.inf, -1e-40]  # edge values
    codes, gamma = Q.sign_hash(dev(x), h, B)
    xh = ops.heads_split(x.reshape(B, n, d), h).reshape(B * h, n, d // h)
    want = ops.pack_codes(xh).view(np.int32).reshape(B, h, n, -1)
    assert np.array_equal(host(codes), want)
    xf = x.copy()
    xf[0, :7] = 0  # gamma comparison on finite values only
    codes2, gamma2 = Q.sign_hash(dev(xf), h, B)
    xh2 = ops.heads_split(xf.reshape(B, n, d), h).reshape(B * h, n, d // h)
    g_ref = ops.per_head_scale(xh2).reshape(B, h)
    assert rel_err(host(gamma2), g_ref) < 2e-6


def test_sign_hash_golden_edge_values(golden):
    from paper_2306_06446_b200 import quantize as Q
    k = golden("kat")
    x = np.zeros((1, 32), F32)
    x[0, :8] = k["sign_x"]
    codes, _ = Q.sign_hash(dev(x), 1, 1)
    bits = [(int(host(codes).reshape(-1)[0]) >> i) & 1 for i in range(8)]
    assert bits == [int(v > 0) for v in k["sign_y"]]


# ------------------------------------------------------- K2a / K2b binary attn


@pytest.mark.parametrize("dk", [16, 32, 64])
@pytest.mark.parametrize("order", ["linear", "quadratic"])
def test_binary_core_matches_golden(golden, dk, order):
    from paper_2306_06446_b200 import attention as A
    k = golden("kat")
    pre = f"lc{dk}_"
    q, kk, v = k[pre + "q"], k[pre + "k"], k[pre + "v"]
    H, n, _ = q.shape
    g = max(1, 32 // dk)          # heads per 'image' so rows are >= 32 channels wide
    nb = H // g

    def flat(t):                  # (H, n, dk) → (nb*n, g*dk), heads as channel blocks
        return dev(ops.heads_merge(t.reshape(nb, g, n, dk)).reshape(nb * n, g * dk))
    out = A.binary_core(flat(q), flat(kk), flat(v), nb, g, None, A.EPS_NORM, order)
    got = ops.heads_split(host(out).reshape(nb, n, g * dk), g).reshape(H, n, dk)
    assert rel_err(got, k[pre + "out"]) < 1e-5
    assert np.all(got[0, 3] == 0)   # all-negative query row → exactly zero


@pytest.mark.parametrize("B,n,d,h", [(2, 196, 64, 4), (2, 3136, 32, 1), (2, 784, 64, 2),
                                     (2, 196, 160, 5)])
def test_linear_binary_attention_with_dwconv(B, n, d, h):
    from paper_2306_06446_b200 import attention as A
    g = ops.rng(7 + n)
    q, kk, v = (g.standard_normal((B * n, d)).astype(F32) for _ in range(3))
    dw = (g.standard_normal((3, 3, d)) * 0.1).astype(F32)
    out = host(A.binary_core(dev(q), dev(kk), dev(v), B, h, dev(dw)))
    # oracle: the reference AttentionLayer core on the same projections
    fold = lambda t: ops.heads_split(t.reshape(B, n, d), h).reshape(B * h, n, d // h)  # noqa
    qf, _ = ops.binary_features(fold(q))
    kf, _ = ops.binary_features(fold(kk))
    o = ops.qkv_linear_core(qf, kf, fold(v))
    merged = ops.heads_merge(o.reshape(B, h, n, d // h)).reshape(B * n, d)
    merged = merged + np.concatenate([ops.dwconv_tokens(v[i * n:(i + 1) * n], dw) for i in range(B)])
    assert rel_err(out, merged) < 2e-5


def test_hamming_matches_linear_order():
    from paper_2306_06446_b200 import attention as A
    g = ops.rng(99)
    B, n, d, h = 2, 197, 192, 3
    q, kk, v = (dev(g.standard_normal((B * n, d)).astype(F32)) for _ in range(3))
    dw = dev((g.standard_normal((3, 3, d)) * 0.1).astype(F32))
    a = host(A.binary_core(q, kk, v, B, h, dw, order="linear"))
    b = host(A.binary_core(q, kk, v, B, h, dw, order="quadratic"))
    assert rel_err(a, b) < 2e-5


@pytest.mark.parametrize("B,n,d,h,with_dw", [(2, 197, 192, 3, True), (3, 197, 192, 3, False),
                                             (2, 49, 64, 2, True), (1, 5, 64, 1, True),
                                             (2, 256, 128, 2, True), (2, 200, 32, 1, True),
                                             (1, 129, 64, 1, True), (2, 17, 192, 3, True)])
def test_tc_hamming_vs_oracle_and_cuda_core(B, n, d, h, with_dw, debug_lib):
    """K2b on the tensor cores (S = Cq Ck^T and S V on tcgen05) against the
    oracle (the same function in K^T V order, associativity) and the CUDA-core
    quadratic kernel; all-negative query rows give exactly the DWConv term."""
    import ctypes
    from paper_2306_06446_b200 import attention as A
    lib = debug_lib
    lib.sa_debug_ham_mode.argtypes = [ctypes.c_int]
    g = ops.rng(23 + n + d)
    q, kk, v = (g.standard_normal((B * n, d)).astype(F32) for _ in range(3))
    q[0, :] = -np.abs(q[0, :]) - 1.0          # one all-negative query row per image 0
    dw = (g.standard_normal((3, 3, d)) * 0.1).astype(F32) if with_dw else None
    args = (dev(q), dev(kk), dev(v), B, h, dev(dw) if with_dw else None, A.EPS_NORM, "quadratic")
    tc = host(A.binary_core(*args))
    try:
        lib.sa_debug_ham_mode(1)
        cc = host(A.binary_core(*args))
    finally:
        lib.sa_debug_ham_mode(0)
    fold = lambda t: ops.heads_split(t.reshape(B, n, d), h).reshape(B * h, n, d // h)  # noqa
    qf, _ = ops.binary_features(fold(q))
    kf, _ = ops.binary_features(fold(kk))
    o = ops.qkv_linear_core(qf, kf, fold(v))
    merged = ops.heads_merge(o.reshape(B, h, n, d // h)).reshape(B * n, d)
    if with_dw:
        merged = merged + np.concatenate([ops.dwconv_tokens(v[i * n:(i + 1) * n], dw)
                                          for i in range(B)])
    assert rel_err(tc, merged) < 2e-5
    assert rel_err(tc, cc) < 2e-5
    if not with_dw:
        assert np.all(tc[0] == 0)


@pytest.mark.parametrize("dk,n", [(32, 300), (64, 197), (16, 196)])
def test_popcounts_bit_exact(dk, n):
    from paper_2306_06446_b200 import attention as A
    from paper_2306_06446_b200 import quantize as Q
    g = ops.rng(dk + n)
    H = 4
    gh = max(1, 32 // dk)             # heads per 'image' (rows >= 32 channels)
    q = g.standard_normal((H * n, dk)).astype(F32)
    kk = g.standard_normal((H * n, dk)).astype(F32)

    def as_images(t):                 # (H*n, dk) head stacks → (H/gh*n, gh*dk) images
        return dev(ops.heads_merge(t.reshape(H // gh, gh, n, dk)).reshape(-1, gh * dk))
    cq, _ = Q.sign_hash(as_images(q), gh, H // gh)
    ck, _ = Q.sign_hash(as_images(kk), gh, H // gh)
    cnt, D, S = A.binary_popcounts(cq, ck, dk, with_scores=True)
    bq = ops.code_bits(q.reshape(H, n, dk)).astype(np.int64)
    bk = ops.code_bits(kk.reshape(H, n, dk)).astype(np.int64)
    cnt_ref = bk.sum(axis=1)
    S_ref = np.einsum("hia,hja->hij", bq, bk)
    assert np.array_equal(host(cnt), cnt_ref)
    assert np.array_equal(host(D), np.einsum("hia,ha->hi", bq, cnt_ref))
    assert np.array_equal(host(S), S_ref)
    # XOR identity popc(a&b) = (popc a + popc b - popc(a^b)) / 2
    x = (bq[:, :, None, :] ^ bk[:, None, :, :]).sum(-1)
    assert np.array_equal(host(S), (bq.sum(-1)[:, :, None] + bk.sum(-1)[:, None, :] - x) // 2)


@pytest.mark.parametrize("n", [5, 196, 197])
def test_dwconv_tokens_golden(golden, n):
    from paper_2306_06446_b200 import attention as A
    k = golden("kat")
    out, side = A._dwconv_tokens(dev(k[f"dw{n}_v"]), dev(k[f"dw{n}_k"]))
    assert side == int(k[f"dw{n}_side"])
    assert rel_err(host(out), k[f"dw{n}_y"]) < 1e-6


# -------------------------------------------------------------- K3 shift linear


def test_quantize_shift_golden_bit_exact(golden):
    from paper_2306_06446_b200 import quantize as Q
    k = golden("kat")
    lay = Q.quantize_shift(dev(k["qs_w"]))
    assert np.array_equal(host(lay.s), k["qs_s"])
    assert np.array_equal(host(lay.p), k["qs_p"])
    rec = host(Q.reconstruct(lay))
    assert np.array_equal(rec.view(np.uint32), k["qs_rec"].view(np.uint32))
    packed = ops.pack_shift_codes(k["qs_s"], k["qs_p"])
    assert np.array_equal(host(lay.packed), packed)


@pytest.mark.parametrize("M,K,N", [(37, 48, 24), (802, 32, 256), (1000, 256, 32), (64, 640, 160)])
@pytest.mark.parametrize("variant", [0, 1])
def test_shift_linear_vs_oracle(M, K, N, variant):
    from paper_2306_06446_b200 import quantize as Q
    g = ops.rng(M + K + N)
    x = g.uniform(-1, 1, (M, K)).astype(F32)
    w = (g.standard_normal((K, N)) / np.sqrt(K)).astype(F32)
    lay = Q.quantize_shift(dev(w))
    y = host(Q.shift_forward(dev(x), lay, variant=variant))
    s, p = ops.shift_quantize(w)
    ref = ops.mm(x, ops.shift_weights(s, p))
    assert rel_err(y, ref) < 2e-6


def test_shift_linear_golden(golden):
    from paper_2306_06446_b200 import quantize as Q
    k = golden("kat")
    lay = Q.ShiftLinear(s=dev(k["sf_s"]), p=dev(k["sf_p"]))
    for variant in (0, 1):
        y = host(Q.shift_forward(dev(k["sf_x"]), lay, variant=variant))
        assert rel_err(y, k["sf_y"]) < 2e-6


def test_shift_variants_agree_with_fakeshift_on_device():
    """Decoded-weight GEMM and literal exponent-add against a dense GEMM on
    s·exp2(P) built by float multiply (ref tests/test_quantize.py:79-85)."""
    from paper_2306_06446_b200 import quantize as Q
    from paper_2306_06446_b200 import tensor as T
    g = ops.rng(5)
    x = dev(g.uniform(-1, 1, (256, 64)).astype(F32))
    lay = Q.quantize_shift(dev(g.uniform(-2, 2, (64, 48)).astype(F32)))
    fake = (lay.s * torch.exp2(lay.p.float())).contiguous()
    dense = host(T.matmul(x, fake))
    assert np.array_equal(host(Q.shift_forward(x, lay, 0)), dense)   # same FFMA core, same order
    assert rel_err(host(Q.shift_forward(x, lay, 1)), dense) < 2e-6


# ------------------------------------------------------------------- K6 GEMM


@pytest.mark.parametrize("M,K,N", [(1, 4, 1), (129, 48, 32), (513, 256, 1000), (300, 640, 10)])
def test_gemm_vs_oracle(M, K, N):
    from paper_2306_06446_b200 import tensor as T
    g = ops.rng(M * 7 + N)
    a = g.standard_normal((M, K)).astype(F32)
    b = g.standard_normal((K, N)).astype(F32)
    assert rel_err(host(T.matmul(dev(a), dev(b))), ops.mm(a, b)) < 2e-6


# ------------------------------------------------------------ K4 router / plan


def test_route_golden_bit_exact(golden):
    from paper_2306_06446_b200 import moe as MOE
    k = golden("kat")
    assert MOE.tie_threshold() == float(k["tie_threshold"])
    plan, logits = MOE.route_plan(dev(k["rt_x"]), dev(k["rt_wg"]), want_logits=True)
    assert np.array_equal(host(logits), k["rt_logits"])
    assert np.array_equal(plan.expert_of, k["rt_expert"])
    assert np.array_equal(np.concatenate(plan.index_of), k["rt_perm"])
    assert rel_err(plan.gate_of, k["rt_gate"]) < 1e-6


def test_dispatch_ties_golden(golden):
    from paper_2306_06446_b200 import moe as MOE
    k = golden("kat")
    plan = MOE.dispatch(None, dev(k["tie_logits"]))
    assert np.array_equal(plan.expert_of, k["tie_expert"])
    assert rel_err(plan.gate_of, k["tie_gate"]) < 1e-6


@pytest.mark.parametrize("M,d", [(100_003, 32), (5000, 256), (1, 64), (70_000, 160),
                                 (20_001, 192), (3000, 96)])
def test_route_partition_vs_oracle(M, d):
    from paper_2306_06446_b200 import moe as MOE
    g = ops.rng(M + d)
    x = g.standard_normal((M, d)).astype(F32)
    wg = (g.standard_normal((d, 2)) * 0.02).astype(F32)
    plan, logits = MOE.route_plan(dev(x), dev(wg), want_logits=True)
    p, lg = ops.router_probs(x, wg)
    e, gate, idx = ops.dispatch_plan(p)
    assert np.array_equal(host(logits), lg)
    assert np.array_equal(plan.expert_of, e)
    assert np.array_equal(np.concatenate(plan.index_of), np.concatenate(idx))
    assert rel_err(plan.gate_of, gate) < 1e-6
    # without logits d >= 96 takes the 8-lanes-per-row kernel: same plan
    plan2, _ = MOE.route_plan(dev(x), dev(wg))
    assert np.array_equal(plan2.expert_of, e)
    assert np.array_equal(np.concatenate(plan2.index_of), np.concatenate(idx))
    assert rel_err(plan2.gate_of, gate) < 1e-6


def test_route_all_to_one_and_empty_expert():
    from paper_2306_06446_b200 import moe as MOE
    x = np.ones((1000, 32), F32)
    wg = np.zeros((32, 2), F32)
    wg[:, 1] = 1.0
    plan, _ = MOE.route_plan(dev(x), dev(wg))
    assert plan.share(1) == 1.0 and plan.index_of[0].size == 0
    wg[:, 1] = 0.0   # exact tie everywhere → expert 0
    plan, _ = MOE.route_plan(dev(x), dev(wg))
    assert plan.share(0) == 1.0 and np.allclose(plan.gate_of, 0.5)


# ----------------------------------------------------------------- K5 experts


def _moe_layers(d, out, hidden=None, seed=3):
    from paper_2306_06446_b200 import model as MD
    g = ops.rng(seed)
    wg = (g.standard_normal((d, 2)) * 0.5).astype(F32)   # spread the routes
    if hidden is None:
        w = (g.standard_normal((d, out)) / np.sqrt(d)).astype(F32)
        mod = MD.MoeModule(wg, [MD.Linear(w), MD.ShiftLinearLayer(w.copy())], MD.MoeConfig())
        s, p = ops.shift_quantize(w)
        L = {"kind": "moe", "wg": wg, "experts": [{"kind": "dense", "w": w},
                                                  {"kind": "shift", "w": w, "s": s, "p": p}]}
    else:
        w1 = (g.standard_normal((d, hidden)) / np.sqrt(d)).astype(F32)
        w2 = (g.standard_normal((hidden, d)) / np.sqrt(hidden)).astype(F32)
        mod = MD.MoeModule(wg, [MD.Mlp(MD.Linear(w1), MD.Linear(w2)),
                                MD.Mlp(MD.ShiftLinearLayer(w1.copy()),
                                       MD.ShiftLinearLayer(w2.copy()))], MD.MoeConfig())
        s1, p1 = ops.shift_quantize(w1)
        s2, p2 = ops.shift_quantize(w2)
        L = {"kind": "moe", "wg": wg, "experts": [
            {"kind": "mlp", "fc1": {"kind": "dense", "w": w1}, "fc2": {"kind": "dense", "w": w2}},
            {"kind": "mlp", "fc1": {"kind": "shift", "w": w1, "s": s1, "p": p1},
             "fc2": {"kind": "shift", "w": w2, "s": s2, "p": p2}}]}
    return mod, L


@pytest.mark.parametrize("M,d,hidden", [(3000, 32, None), (3000, 32, 256), (777, 160, 640),
                                        (4096, 64, 512)])
def test_moe_module_vs_oracle(M, d, hidden):
    mod, L = _moe_layers(d, d, hidden)
    x = ops.rng(M).standard_normal((M, d)).astype(F32)
    res = ops.rng(M + 1).standard_normal((M, d)).astype(F32)
    y = host(mod.forward(dev(x), residual=dev(res)))
    tr = nets.Trace()
    ref = nets.moe_fwd(L, x, "m", tr)
    assert np.array_equal(mod.last_plan.expert_of, tr.moe[0]["expert_of"])
    assert 0.05 < mod.last_plan.share(1) < 0.95
    assert rel_err(y - res, ref) < 1e-5
    assert rel_err(y, res + ref) < 1e-5


@pytest.mark.parametrize("M,d,hidden,scale,force", [
    (5, 32, 256, 1.0, None), (129, 32, 512, 1.0, None), (1000, 64, 256, 1.0, None),
    (3000, 32, 128, 1.0, None), (2000, 32, 256, 8.0, None), (777, 64, 512, 6.0, None),
    (1500, 32, 256, 1.0, 0), (1500, 32, 256, 1.0, 1), (640, 64, 512, 1.0, 1),
    # wide form (d = 128 / 160: hidden chunks of 32, single acc2, streamed weights)
    (5, 160, 640, 1.0, None), (1000, 160, 640, 1.0, None), (777, 160, 640, 6.0, None),
    (1500, 160, 640, 1.0, 0), (1500, 160, 640, 1.0, 1), (3001, 128, 512, 1.0, None),
    (700, 128, 1024, 1.0, None), (2000, 192, 768, 1.0, None), (333, 192, 768, 6.0, None),
    (1200, 192, 768, 1.0, 0), (1200, 192, 768, 1.0, 1)])
def test_fused_moe_mlp_edges(M, d, hidden, scale, force):
    """Fused MoE MLP kernel: ragged and tiny M, resident (d = 32, hidden <= 256)
    and streamed weights, hidden pre-activations spanning the GELU's saturated
    tails (scale), every token on one expert (force) — routes bit-exact and
    y within 1e-5 of the oracle."""
    mod, L = _moe_layers(d, d, hidden, seed=M + d)
    if force is not None:   # positive inputs, router +1 / -1 columns: one expert wins everywhere
        wg = np.zeros((d, 2), F32)
        wg[:, force] = 1.0
        wg[:, 1 - force] = -1.0
        mod.wg.value.copy_(torch.from_numpy(wg))
        L["wg"] = wg
        x = np.abs(ops.rng(M).standard_normal((M, d))).astype(F32) * scale + 0.01
    else:
        x = (ops.rng(M).standard_normal((M, d)) * scale).astype(F32)
    res = ops.rng(M + 1).standard_normal((M, d)).astype(F32)
    y = host(mod.forward(dev(x), residual=dev(res)))
    tr = nets.Trace()
    ref = nets.moe_fwd(L, x, "m", tr)
    assert np.array_equal(mod.last_plan.expert_of, tr.moe[0]["expert_of"])
    if force is not None:
        assert mod.last_plan.share(force) == 1.0
    assert rel_err(y - res, ref) < 1e-5


@pytest.mark.parametrize("d,hidden,shift", [(32, 256, False), (32, 256, True), (64, 512, False),
                                           (64, 512, True), (32, 512, False), (160, 640, False),
                                           (160, 640, True), (128, 1024, False)])
def test_fused_mlp_plain_vs_oracle(d, hidden, shift):
    """Single-expert fused MLP (sa_tc_mlp_fused) for dense and shift layers."""
    from paper_2306_06446_b200 import model as MD
    g = ops.rng(d + hidden)
    M = 2049
    x = (g.standard_normal((M, d)) * 2).astype(F32)
    w1 = (g.standard_normal((d, hidden)) / np.sqrt(d)).astype(F32)
    w2 = (g.standard_normal((hidden, d)) / np.sqrt(hidden)).astype(F32)
    mk = MD.ShiftLinearLayer if shift else MD.Linear
    mlp = MD.Mlp(mk(w1), mk(w2))
    assert MD.fused_mlp_ok(d, hidden)
    y = host(mlp.forward(dev(x)))
    if shift:
        L1 = dict(zip(("kind", "s", "p"), ("shift",) + ops.shift_quantize(w1)))
        L2 = dict(zip(("kind", "s", "p"), ("shift",) + ops.shift_quantize(w2)))
    else:
        L1, L2 = {"kind": "dense", "w": w1}, {"kind": "dense", "w": w2}
    ref = nets.linear_fwd({"kind": "mlp", "fc1": L1, "fc2": L2}, x)
    assert rel_err(y, ref) < 1e-5


def test_moe_golden(golden):
    from paper_2306_06446_b200 import model as MD
    k = golden("kat")
    w = k["mf_w"]
    mod = MD.MoeModule(k["mf_wg"], [MD.Linear(w), MD.ShiftLinearLayer(w.copy())], MD.MoeConfig())
    y = host(mod.forward(dev(k["mf_x"])))
    assert np.array_equal(mod.last_plan.expert_of, k["mf_expert"])
    assert rel_err(y, k["mf_y"]) < 1e-5


# --------------------------------------------------------------------- glue


def test_layernorm_golden(golden):
    from paper_2306_06446_b200 import tensor as T
    k = golden("kat")
    d = k["ln_x"].shape[1]
    y, _ = T.layernorm(dev(k["ln_x"]), dev(np.ones(d, F32)), dev(np.zeros(d, F32)))
    assert rel_err(host(y), k["ln_y"]) < 2e-6


def test_softmax_core_golden(golden):
    from paper_2306_06446_b200 import attention as A
    k = golden("kat")
    out, _ = A.softmax_core(dev(k["sm_q"]), dev(k["sm_k"]), dev(k["sm_v"]))
    assert rel_err(host(out), k["sm_out"]) < 2e-6


@pytest.mark.parametrize("n", [7, 32, 33, 43, 47, 49, 64])
def test_softmax_attn32_bit_identical_to_generic(n, debug_lib):
    """The register-blocked dk=32 softmax kernel computes the generic kernel's
    arithmetic in the same order: bit-identical outputs, and the oracle's
    softmax core within fp32 tolerance."""
    from paper_2306_06446_b200 import _lib
    from paper_2306_06446_b200 import attention as A
    lib = debug_lib
    g = ops.rng(n)
    B, heads, dk = 5, 3, 32
    q, k, v = (g.standard_normal((B * n, heads * dk)).astype(F32) for _ in range(3))
    fast = host(A.softmax_core_flat(dev(q), dev(k), dev(v), B, heads))
    for qb in (2, 8):   # queries per warp iteration: same arithmetic per query
        lib.sa_debug_softmax_qb(qb)
        try:
            assert np.array_equal(host(A.softmax_core_flat(dev(q), dev(k), dev(v), B, heads)), fast)
        finally:
            lib.sa_debug_softmax_qb(4)
    lib.sa_debug_softmax_generic(1)
    try:
        slow = host(A.softmax_core_flat(dev(q), dev(k), dev(v), B, heads))
    finally:
        lib.sa_debug_softmax_generic(0)
    assert np.array_equal(fast, slow)
    for b in range(B):
        for h in range(heads):
            sl = (slice(b * n, (b + 1) * n), slice(h * dk, (h + 1) * dk))
            ref = ops.softmax_core(q[sl][None], k[sl][None], v[sl][None])[0]
            assert rel_err(fast[sl], ref) < 2e-6


@pytest.mark.parametrize("B,n,heads,dk", [(3, 197, 3, 64), (2, 49, 8, 64), (2, 5, 2, 64),
                                          (2, 256, 2, 64), (2, 100, 3, 32), (1, 129, 1, 64),
                                          (2, 200, 5, 32)])
def test_softmax_tc_vs_oracle_and_generic(B, n, heads, dk, debug_lib):
    """Tensor-core softmax core (six-product fp32 split of q k^T and p v) against
    the oracle's softmax core and the CUDA-core generic kernel, on the strided
    q|k|v layout the exempt stage uses."""
    from paper_2306_06446_b200 import attention as A
    from paper_2306_06446_b200 import _lib
    lib = debug_lib
    g = ops.rng(31 + n + dk)
    d = heads * dk
    qkv = (g.standard_normal((B * n, 3 * d)) * 1.5).astype(F32)
    t = dev(qkv)
    out = torch.empty((B * n, d), dtype=torch.float32, device="cuda")

    def run():
        base = _lib.ptr(t)
        _lib.call("sa_softmax_attn_strided", base, base + 4 * d, base + 8 * d, 3 * d,
                  _lib.ptr(out), B, n, d, heads, _lib.stream())
        return host(out).copy()
    tc = run()
    lib.sa_debug_softmax_tc(1)
    try:
        cc = run()
    finally:
        lib.sa_debug_softmax_tc(0)
    q, k, v = qkv[:, :d], qkv[:, d:2 * d], qkv[:, 2 * d:]
    fold = lambda x: ops.heads_split(x.reshape(B, n, d), heads).reshape(B * heads, n, dk)  # noqa
    ref = ops.heads_merge(ops.softmax_core(fold(q), fold(k), fold(v)).reshape(B, heads, n, dk))
    ref = ref.reshape(B * n, d)
    assert rel_err(tc, ref) < 2e-5
    assert rel_err(cc, ref) < 2e-6
    assert rel_err(tc, cc) < 2e-5


def test_mlp_gelu_vs_oracle(golden):
    from paper_2306_06446_b200 import model as MD
    g = ops.rng(1)
    x = g.standard_normal((999, 64)).astype(F32)
    w1 = (g.standard_normal((64, 256)) / 8).astype(F32)
    w2 = (g.standard_normal((256, 64)) / 16).astype(F32)
    for shift in (False, True):
        mk = MD.ShiftLinearLayer if shift else MD.Linear
        mlp = MD.Mlp(mk(w1), mk(w2))
        y = host(mlp.forward(dev(x)))
        L1 = {"kind": "dense", "w": w1} if not shift else dict(zip(("kind", "s", "p"), ("shift",) + ops.shift_quantize(w1)))
        L2 = {"kind": "dense", "w": w2} if not shift else dict(zip(("kind", "s", "p"), ("shift",) + ops.shift_quantize(w2)))
        ref = nets.linear_fwd({"kind": "mlp", "fc1": L1, "fc2": L2}, x)
        assert rel_err(y, ref) < 1e-5


@pytest.mark.parametrize("M,d,nr", [(50_000, 32, 3), (777, 64, 1), (4096, 64, 3),
                                    (50_176, 160, 3), (1001, 160, 1), (333, 256, 2),
                                    (4097, 96, 3)])
def test_ln_route_fused_vs_oracle(M, d, nr):
    """LayerNorm fused with 1..3 routers: y within fp32 tolerance of the
    oracle LN, winners / permutations bit-exact against the oracle router
    evaluated on the device's own y (kernel-boundary parity)."""
    from paper_2306_06446_b200 import moe as MOE
    g = ops.rng(M + d + nr)
    x = (g.standard_normal((M, d)) * 2 + 0.3).astype(F32)
    wgs = [(g.standard_normal((d, 2)) * 0.3).astype(F32) for _ in range(nr)]
    gain = np.ones(d, F32)
    bias = np.zeros(d, F32)
    y, plans = MOE.ln_route_plans(dev(x), dev(gain), dev(bias), [dev(w) for w in wgs])
    yh = host(y)
    assert rel_err(yh, ops.layer_norm(x, gain, bias)) < 2e-6
    for w, plan in zip(wgs, plans):
        p, _ = ops.router_probs(yh, w)
        e, gate, idx = ops.dispatch_plan(p)
        assert np.array_equal(plan.expert_of, e)
        assert np.array_equal(np.concatenate(plan.index_of), np.concatenate(idx))
        assert rel_err(plan.gate_of, gate) < 1e-6


@pytest.mark.parametrize("M,d,nr,ln", [(50_176, 160, 3, True), (1001, 96, 1, True),
                                       (333, 256, 2, True), (70_001, 160, 1, False),
                                       (129, 192, 1, False)])
def test_ln_route_two_rows_per_thread_bit_identical(M, d, nr, ln, debug_lib):
    """The 8-lanes-per-row LN+router kernel with two rows per thread writes the
    one-row-per-thread kernel's y, winners, gates and partitions bit for bit."""
    from paper_2306_06446_b200 import _lib
    from paper_2306_06446_b200 import moe as MOE
    lib = debug_lib
    g = ops.rng(M + 3 * d + nr)
    x = dev((g.standard_normal((M, d)) * 1.3 + 0.1).astype(F32))
    gain = dev((1 + 0.1 * g.standard_normal(d)).astype(F32))
    bias = dev((0.05 * g.standard_normal(d)).astype(F32))
    wgs = [dev((g.standard_normal((d, 2)) * 0.3).astype(F32)) for _ in range(nr)]

    def run():
        if ln:
            y, plans = MOE.ln_route_plans(x, gain, bias, wgs)
            return host(y), plans
        plan, _ = MOE.route_plan(x, wgs[0])
        return None, [plan]
    y2, p2 = run()
    lib.sa_debug_oct_rows(1)
    try:
        y1, p1 = run()
    finally:
        lib.sa_debug_oct_rows(2)
    if ln:
        assert np.array_equal(y1, y2)
    for a, b in zip(p1, p2):
        assert np.array_equal(a.expert_of, b.expert_of)
        assert np.array_equal(a.gate_of, b.gate_of)
        for ia, ib in zip(a.index_of, b.index_of):
            assert np.array_equal(ia, ib)


@pytest.mark.parametrize("M,d,nr", [(50_176, 160, 3), (999, 160, 1), (2000, 256, 2)])
def test_ln_route_wide_matches_unfused(M, d, nr):
    """The warp-per-row LN+router kernel (d = 32k > 64) writes exactly
    sa_layernorm's y, and its winners / gates / partitions equal the unfused
    router's on that y."""
    from paper_2306_06446_b200 import moe as MOE
    from paper_2306_06446_b200 import tensor as T
    g = ops.rng(M * 7 + d)
    x = (g.standard_normal((M, d)) * 1.7 - 0.2).astype(F32)
    gain = (1 + 0.1 * g.standard_normal(d)).astype(F32)
    bias = (0.05 * g.standard_normal(d)).astype(F32)
    wgs = [(g.standard_normal((d, 2)) * 0.3).astype(F32) for _ in range(nr)]
    y, plans = MOE.ln_route_plans(dev(x), dev(gain), dev(bias), [dev(w) for w in wgs])
    y_ref, _ = T.layernorm(dev(x), dev(gain), dev(bias))
    assert np.array_equal(host(y), host(y_ref))
    for w, plan in zip(wgs, plans):
        ref, _ = MOE.route_plan(y_ref, dev(w))
        assert np.array_equal(plan.expert_of, ref.expert_of)
        assert np.array_equal(plan.gate_of, ref.gate_of)
        for a, b in zip(plan.index_of, ref.index_of):
            assert np.array_equal(a, b)


@pytest.mark.parametrize("B,n,d,h,with_dw", [(3, 3136, 32, 1, True), (2, 784, 64, 2, True),
                                             (2, 196, 160, 5, True), (2, 300, 96, 3, True),
                                             (3, 197, 64, 2, False), (1, 5, 32, 1, True),
                                             (2, 49, 256, 8, True), (2, 3136, 64, 1, True),
                                             (2, 784, 128, 2, True), (2, 196, 320, 5, True),
                                             (2, 197, 192, 3, True), (1, 5, 64, 1, True),
                                             (2, 1000, 128, 2, False)])
def test_tc_binary_attention_vs_oracle_and_cuda_core(B, n, d, h, with_dw, debug_lib):
    """The product kernels (dk = 32: CUDA-core single-pass cluster kernel; 64:
    tensor-core cluster kernel) against the oracle, the tensor-core cluster
    kernel at every dk, the streaming tensor-core kernel (debug build) and the
    three-kernel path, on square and non-square token grids with partial last
    rows; the split two-kernel form is bit-identical to the fused CUDA-core one."""
    import ctypes
    from paper_2306_06446_b200 import attention as A
    lib = debug_lib
    lib.sa_debug_attn_mode.argtypes = [ctypes.c_int]
    g = ops.rng(11 + n + d)
    q, kk, v = (g.standard_normal((B * n, d)).astype(F32) for _ in range(3))
    dw = (g.standard_normal((3, 3, d)) * 0.1).astype(F32) if with_dw else None
    args = (dev(q), dev(kk), dev(v), B, h, dev(dw) if with_dw else None)

    def run(mode):
        try:
            lib.sa_debug_attn_mode(mode)
            return host(A.binary_core(*args))
        finally:
            lib.sa_debug_attn_mode(0)
    prod = host(A.binary_core(*args))        # default path (dk 32: CUDA-core fused, 64: tc)
    assert np.array_equal(run(0), prod)
    tc = run(3)                              # the tensor-core cluster kernel at every dk
    prev = run(4)                            # = the product choice
    stream = run(5)                          # the streaming tensor-core kernel
    assert np.array_equal(run(5), stream)    # deterministic
    legacy = run(1)
    fold = lambda t: ops.heads_split(t.reshape(B, n, d), h).reshape(B * h, n, d // h)  # noqa
    qf, _ = ops.binary_features(fold(q))
    kf, _ = ops.binary_features(fold(kk))
    o = ops.qkv_linear_core(qf, kf, fold(v))
    merged = ops.heads_merge(o.reshape(B, h, n, d // h)).reshape(B * n, d)
    if with_dw:
        merged = merged + np.concatenate([ops.dwconv_tokens(v[i * n:(i + 1) * n], dw)
                                          for i in range(B)])
    assert rel_err(tc, merged) < 2e-5
    assert rel_err(legacy, merged) < 2e-5
    assert rel_err(tc, legacy) < 2e-5
    assert rel_err(prod, merged) < 2e-5
    assert rel_err(prod, tc) < 2e-5
    assert np.array_equal(prev, prod)
    if d // h in (32, 64):
        assert rel_err(stream, merged) < 2e-5
        assert rel_err(stream, tc) < 2e-5
    if d // h == 32:
        assert rel_err(prev, legacy) < 2e-6   # CUDA-core fused vs three-kernel path
        assert np.array_equal(run(2), prev)   # split form: same arithmetic
    else:
        assert np.array_equal(prev, tc)
    # all-negative query rows give exactly the DWConv term (zero attention part)
    q2 = q.copy()
    q2[0, :] = -np.abs(q2[0, :]) - 1.0
    out2 = host(A.binary_core(dev(q2), dev(kk), dev(v), B, h, None))
    assert np.all(out2[0] == 0)


@pytest.mark.parametrize("M,d", [(777, 32), (20000, 64), (802816 // 64, 32)])
def test_fused_moe_linear_matches_unfused(M, d):
    """sa_fused_moe_linear (router + both experts + residual in one kernel, the
    W_O path) against route_plan + sa_tc_moe_linear: identical winners, gates
    and outputs (the same split-precision MMA chains), and the oracle."""
    from paper_2306_06446_b200 import model as MD
    mod, L = _moe_layers(d, d, None)
    g = ops.rng(M + d)
    x = g.standard_normal((M, d)).astype(F32)
    res = g.standard_normal((M, d)).astype(F32)
    old = MD.FUSE_O
    try:
        MD.FUSE_O = False
        y0 = host(mod.forward(dev(x), residual=dev(res)))
        e0, g0, i0 = mod.last_plan.expert_of, mod.last_plan.gate_of, mod.last_plan.index_of
        MD.FUSE_O = True
        y1 = host(mod.forward(dev(x), residual=dev(res)))
        e1, g1, i1 = mod.last_plan.expert_of, mod.last_plan.gate_of, mod.last_plan.index_of
    finally:
        MD.FUSE_O = old
    assert np.array_equal(e0, e1) and np.array_equal(g0, g1)
    assert np.array_equal(i0[0], i1[0]) and np.array_equal(i0[1], i1[1])
    assert np.array_equal(y0, y1)
    tr = nets.Trace()
    ref = nets.moe_fwd(L, x, "m", tr)
    assert np.array_equal(e1, tr.moe[0]["expert_of"])
    assert rel_err(y1, res + ref) < 1e-5


@pytest.mark.parametrize("M,d", [(1000, 160), (50_176, 160), (333, 96)])
def test_grouped_moe_linear_matches_per_problem(M, d):
    """sa_tc_moe_linear_grouped (three problems, six row groups in one launch)
    equals three sa_tc_moe_linear calls bit for bit, including empty groups
    (a problem routed entirely to one expert) and ragged M."""
    import ctypes
    from paper_2306_06446_b200 import _lib
    from paper_2306_06446_b200 import model as MD
    g = ops.rng(M + 7 * d)
    x = dev(g.standard_normal((M, d)).astype(F32))
    mods = []
    for r in range(3):
        w = (g.standard_normal((d, d)) / np.sqrt(d)).astype(F32)
        mods.append((MD.Linear(w), MD.ShiftLinearLayer(w.copy())))
    perm = np.zeros((3, M), np.int32)
    counts = np.zeros((3, 2), np.int32)
    gate = (0.5 + 0.5 * g.random((3, M))).astype(F32)
    e = g.integers(0, 2, M)                       # problem 0: a random split
    perm[0] = np.concatenate([np.flatnonzero(e == 0), np.flatnonzero(e == 1)])
    counts[0] = [(e == 0).sum(), (e == 1).sum()]
    perm[1] = np.arange(M)                        # problem 1: all expert 0
    counts[1] = [M, 0]
    perm[2] = g.permutation(M)                    # problem 2: all expert 1
    counts[2] = [0, M]
    perm_d, counts_d, gate_d = dev(perm), dev(counts), dev(gate)
    packs = [(a.tc_pack(), b.tc_pack()) for a, b in mods]
    bn = packs[0][0][1]
    y = torch.empty((3, M, d), dtype=torch.float32, device="cuda")
    dense = (ctypes.c_void_p * 3)(*[_lib.ptr(p[0][0]) for p in packs])
    shift = (ctypes.c_void_p * 3)(*[_lib.ptr(p[1][0]) for p in packs])
    _lib.call("sa_tc_moe_linear_grouped", _lib.ptr(x), _lib.ptr(perm_d), _lib.ptr(counts_d),
              _lib.ptr(gate_d), ctypes.addressof(dense), ctypes.addressof(shift), 3, bn,
              _lib.ptr(y), M, d, d, _lib.stream())
    got = host(y)
    for r in range(3):
        yr = torch.empty((M, d), dtype=torch.float32, device="cuda")
        _lib.call("sa_tc_moe_linear", _lib.ptr(x), _lib.ptr(perm_d[r]), _lib.ptr(counts_d[r]),
                  _lib.ptr(gate_d[r]), _lib.ptr(packs[r][0][0]), _lib.ptr(packs[r][1][0]), bn,
                  _lib.ptr(yr), None, M, d, d, _lib.stream())
        assert np.array_equal(got[r], host(yr)), r


def test_packed_gelu_and_split_bitwise_equal_scalar(debug_lib):
    """gelu_fast2 / split3x2 (packed f32x2 arithmetic) reproduce the scalar
    gelu_fast and bf16 plane split bit for bit over 2^24 patterned inputs
    (range [-16, 16] and arbitrary finite bit patterns)."""
    from paper_2306_06446_b200 import _lib
    lib = debug_lib
    bad = torch.zeros(1, dtype=torch.int64, device="cuda")
    assert lib.sa_debug_gelu_pair_check(ctypes_i64(1 << 24), ctypes_p(bad.data_ptr()), None) == 0
    torch.cuda.synchronize()
    assert int(bad.item()) == 0


def ctypes_i64(v):
    import ctypes
    return ctypes.c_int64(v)


def ctypes_p(v):
    import ctypes
    return ctypes.c_void_p(v)


# ------------------------------------------------------------------ MatAdd


def test_add_matmul_golden_bit_exact(golden):
    """sa_add_linear (signed fp64 accumulation, one gamma multiply) against the
    reference's add_matmul outputs: bit-exact (ref quantize.py:143-160)."""
    from paper_2306_06446_b200 import quantize as Q
    k = golden("addlinear")
    y = host(Q.add_matmul(dev(k["hand_x"]), Q.AddLinear(b=dev(k["hand_b"]), gamma=1.0)))
    assert np.array_equal(y, k["hand_y"])
    for i in range(4):
        layer = Q.AddLinear(b=dev(k[f"b{i}"]), gamma=float(k[f"g{i}"]))
        y = host(Q.add_matmul(dev(k[f"x{i}"]), layer))
        assert np.array_equal(y, k[f"y{i}"]), i


def test_reparam_add_and_project(golden):
    """reparam_linear(w, "add") reproduces the reference's signs (gamma to
    1 ulp: fp64 vs numpy float32 mean) and attention.project dispatches an
    AddLinear to add_matmul (ref attention.py:66-71, quantize.py:177-189)."""
    from paper_2306_06446_b200 import attention as A
    from paper_2306_06446_b200 import quantize as Q
    k = golden("addlinear")
    for i in (1, 2, 3):
        rr = Q.reparam_linear(dev(k[f"w{i}"]), "add")
        assert np.array_equal(host(rr.layer.b), k[f"b{i}"])
        assert abs(rr.layer.gamma - float(k[f"g{i}"])) <= 2 * np.spacing(np.float32(k[f"g{i}"]))
        assert np.array_equal(host(rr.shadow), k[f"w{i}"])
        y = host(A.project(dev(k[f"x{i}"]), rr.layer))
        ref = ops.add_matmul(k[f"x{i}"], host(rr.layer.b), rr.layer.gamma)
        assert np.array_equal(y, ref)
        rec = host(Q.reconstruct_add(rr.layer))
        assert np.array_equal(rec, (rr.layer.gamma * host(rr.layer.b).astype(np.float64)).astype(F32))
    with pytest.raises(ValueError):
        Q.reparam_linear(dev(k["w1"]), "mult")


def test_add_matmul_shapes_and_errors():
    from paper_2306_06446_b200 import quantize as Q
    from paper_2306_06446_b200.tensor import ShapeError
    g = ops.rng(5)
    b = np.where(g.standard_normal((37, 29)) < 0, -1.0, 1.0).astype(F32)
    x = g.standard_normal((131, 37)).astype(F32)
    layer = Q.AddLinear(b=dev(b), gamma=0.37)
    assert np.array_equal(host(Q.add_matmul(dev(x), layer)), ops.add_matmul(x, b, 0.37))
    assert host(Q.add_matmul(dev(x[:0]), layer)).shape == (0, 29)
    with pytest.raises(ShapeError):
        Q.add_matmul(dev(x[:, :36]), layer)
    with pytest.raises(ShapeError):
        Q.add_matmul(dev(x.reshape(-1)), layer)
