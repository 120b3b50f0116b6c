"""tcgen05 tensor-core GEMM path (split-bf16, float32-faithful) against the
oracle's float64-accumulated products, and against the CUDA-core path."""

import numpy as np
import pytest
import torch

from oracle import ops

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


def tc_linear(x, layer, act=0, residual=None):
    from paper_2306_06446_b200 import _lib
    pk, bn, kind = layer.tc_pack()
    M, K = x.shape
    N = layer.out_dim
    y = torch.empty((M, N), dtype=torch.float32, device="cuda")
    _lib.call("sa_tc_linear", _lib.ptr(x), _lib.ptr(pk), kind, bn, _lib.ptr(y), M, K, N,
              _lib.ptr(residual), act, _lib.stream())
    return y


SHAPES = [(1, 32, 32), (129, 48, 32), (1000, 32, 256), (777, 256, 32), (300, 160, 640),
          (256, 1024, 256), (513, 64, 64), (200, 256, 1000), (64, 128, 10), (3000, 640, 160)]


@pytest.mark.parametrize("M,K,N", SHAPES)
@pytest.mark.parametrize("kind", ["dense", "shift"])
def test_tc_linear_vs_oracle(M, K, N, kind):
    from paper_2306_06446_b200 import model as MD
    g = ops.rng(M * 31 + K + N)
    x = g.standard_normal((M, K)).astype(F32)
    w = (g.standard_normal((K, N)) / np.sqrt(K)).astype(F32)
    if kind == "dense":
        layer = MD.Linear(w)
        ref = ops.mm(x, w)
    else:
        layer = MD.ShiftLinearLayer(w)
        s, p = ops.shift_quantize(w)
        ref = ops.mm(x, ops.shift_weights(s, p))
    y = host(tc_linear(dev(x), layer))
    # tensor-core fp32 accumulation truncates (round-toward-zero-like) once per
    # 16-deep MMA step, so the bound grows with K/16 (measured 7.8e-6 at K=1024)
    tol = 5e-6 if K <= 256 else 1.2e-5
    assert rel_err(y, ref) < tol, rel_err(y, ref)


def test_tc_epilogues_gelu_residual():
    from paper_2306_06446_b200 import model as MD
    g = ops.rng(3)
    x = g.standard_normal((515, 64)).astype(F32)
    w = (g.standard_normal((64, 256)) / 8).astype(F32)
    res = g.standard_normal((515, 256)).astype(F32)
    layer = MD.Linear(w)
    y = host(tc_linear(dev(x), layer, act=1, residual=dev(res)))
    ref = res + ops.gelu_tanh(ops.mm(x, w))
    assert rel_err(y, ref) < 5e-6


def test_tc_shift_products_exact_small_k():
    """With K small and exactly representable partial sums, the split-bf16
    shift product must reproduce FakeShift bit-for-bit."""
    from paper_2306_06446_b200 import model as MD
    g = ops.rng(9)
    x = (g.integers(-64, 64, (256, 32)) / 64.0).astype(F32)     # 7-bit values: exact sums
    w = np.ldexp(np.where(g.uniform(size=(32, 32)) < 0.5, -1.0, 1.0),
                 g.integers(-4, 4, (32, 32))).astype(F32)
    layer = MD.ShiftLinearLayer(w)
    y = host(tc_linear(dev(x), layer))
    assert np.array_equal(y, (x.astype(np.float64) @ w.astype(np.float64)).astype(F32))


def test_tc_matches_simt_path():
    from paper_2306_06446_b200 import _lib
    from paper_2306_06446_b200 import model as MD
    g = ops.rng(4)
    x = dev(g.standard_normal((4096, 160)).astype(F32))
    w = (g.standard_normal((160, 640)) / 13).astype(F32)
    for layer in (MD.Linear(w), MD.ShiftLinearLayer(w)):
        a = host(tc_linear(x, layer))
        wt, kind, p_min = layer.weight_arg()
        b = torch.empty_like(torch.from_numpy(a)).cuda()
        _lib.call("sa_linear", _lib.ptr(x), _lib.ptr(wt), kind, _lib.ptr(b), 4096, 160, 640, p_min,
                  None, 0, _lib.stream())
        assert rel_err(a, host(b)) < 5e-6
