"""Numpy restatement of the reference primitives on the inference path.

Test infrastructure (see oracle/__init__.py). Numerics follow the reference
exactly: every matrix product widens both operands to float64, multiplies, and
rounds the result back to the operand dtype (ref tensor.py:68-75, 85-90); all
elementwise work stays in the activation dtype (float32).
"""

from __future__ import annotations

import math

import numpy as np

F32 = np.float32
LN_EPS = 1e-5          # ref tensor.py:22
ATTN_EPS = 1e-6        # ref attention.py:32 (EPS_NORM)
GELU_C = 0.7978845608028654   # ref tensor.py:145
GELU_A = 0.044715             # ref tensor.py:146
P_MIN, P_MAX = -15, 15        # ref quantize.py:27-28


def rng(seed: int) -> np.random.Generator:
    """PCG64 stream (ref tensor.py:33-35)."""
    return np.random.Generator(np.random.PCG64(seed))


# ---------------------------------------------------------------------------
# dense substrate


def mm(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """2-D product with float64 accumulation (ref tensor.py:68-75)."""
    assert a.ndim == 2 and b.ndim == 2 and a.shape[1] == b.shape[0]
    wide = a.astype(np.float64) @ b.astype(np.float64)
    return wide.astype(np.result_type(a.dtype, b.dtype), copy=False)


def bmm(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Stacked product with float64 accumulation (ref tensor.py:85-90)."""
    wide = np.matmul(a.astype(np.float64), b.astype(np.float64))
    return wide.astype(np.result_type(a.dtype, b.dtype), copy=False)


def softmax_rows(x: np.ndarray) -> np.ndarray:
    """Max-shifted softmax over the last axis (ref tensor.py:97-103)."""
    e = np.exp(x - np.max(x, axis=-1, keepdims=True))
    return e / np.sum(e, axis=-1, keepdims=True)


def layer_norm(x, gain, bias, eps=LN_EPS):
    """Biased-variance layer norm over the last axis (ref tensor.py:114-128)."""
    mu = np.mean(x, axis=-1, keepdims=True)
    c = x - mu
    var = np.mean(c * c, axis=-1, keepdims=True)
    return c * (1.0 / np.sqrt(var + eps)) * gain + bias


def gelu_tanh(x):
    """tanh-form GELU with the `x ** 3` power (ref tensor.py:149-152)."""
    return 0.5 * x * (1.0 + np.tanh(GELU_C * (x + GELU_A * x ** 3)))


def dw3x3(grid: np.ndarray, k: np.ndarray) -> np.ndarray:
    """Depthwise 3x3, zero pad 1, float64 taps (ref tensor.py:177-199).

    grid is (h, w, c); k is (3, 3, c)."""
    h, w, c = grid.shape
    pad = np.zeros((h + 2, w + 2, c), np.float64)
    pad[1:h + 1, 1:w + 1] = grid
    k64 = k.astype(np.float64)
    acc = np.zeros((h, w, c), np.float64)
    for r in range(3):
        for s in range(3):
            acc += pad[r:r + h, s:s + w] * k64[r, s]
    return acc.astype(np.result_type(grid.dtype, k.dtype), copy=False)


# ---------------------------------------------------------------------------
# shift / sign quantization


def sign_pm1(x: np.ndarray) -> np.ndarray:
    """+1 unless x < 0 (so -0.0 and NaN give +1) (ref quantize.py:78-80)."""
    return np.where(x < 0, -1.0, 1.0).astype(x.dtype, copy=False)


def code_bits(x: np.ndarray) -> np.ndarray:
    """{0,1} code = (sign_pm1(x)+1)/2 as uint8 (ref model.py:357-358)."""
    return (~(x < 0)).astype(np.uint8)


def shift_quantize(w: np.ndarray, p_min=P_MIN, p_max=P_MAX):
    """(s, P): s = sign_pm1(w); P = clip(rint(log2|w|)) in float64, zeros and
    non-finite logs → p_min (ref quantize.py:83-96)."""
    s = sign_pm1(w)
    with np.errstate(divide="ignore"):
        lg = np.rint(np.log2(np.abs(w.astype(np.float64))))
    lg = np.nan_to_num(lg, nan=p_min, neginf=p_min)
    return s, np.clip(lg, p_min, p_max).astype(np.int32)


def shift_weights(s: np.ndarray, p: np.ndarray, dtype=F32) -> np.ndarray:
    """Exact s·2^P via ldexp (ref quantize.py:99-101)."""
    return np.ldexp(s.astype(dtype), p)


def pack_shift_codes(s: np.ndarray, p: np.ndarray, p_min=P_MIN) -> np.ndarray:
    """Byte layout the GPU consumes: bit7 = (s<0), bits0-4 = P - p_min."""
    return (((s < 0).astype(np.uint8) << 7) | (p - p_min).astype(np.uint8)).astype(np.uint8)


def per_head_scale(xh: np.ndarray) -> np.ndarray:
    """γ = mean|x| over every axis but 0, keepdims (ref quantize.py:134-137)."""
    return np.mean(np.abs(xh), axis=tuple(range(1, xh.ndim)), keepdims=True)


def pack_codes(xh: np.ndarray) -> np.ndarray:
    """Pack the code bits of (H, n, dk) into uint32 words (H, n, ceil(dk/32));
    bit j of word w is channel 32w+j. This is the GPU's code layout."""
    H, n, dk = xh.shape
    words = (dk + 31) // 32
    bits = code_bits(xh).astype(np.uint64)
    out = np.zeros((H, n, words), np.uint32)
    for wi in range(words):
        chunk = bits[..., 32 * wi: min(dk, 32 * wi + 32)]
        sh = np.arange(chunk.shape[-1], dtype=np.uint64)
        out[..., wi] = (chunk << sh).sum(axis=-1).astype(np.uint32)
    return out


# ---------------------------------------------------------------------------
# attention


def heads_split(x: np.ndarray, h: int) -> np.ndarray:
    """(..., n, d) → (..., h, n, d/h); head i owns channels [i·dk,(i+1)·dk)
    (ref attention.py:74-78)."""
    *lead, n, d = x.shape
    return np.swapaxes(x.reshape(*lead, n, h, d // h), -3, -2)


def heads_merge(x: np.ndarray) -> np.ndarray:
    """Inverse of heads_split (ref attention.py:81-85)."""
    x = np.ascontiguousarray(np.swapaxes(x, -3, -2))
    *lead, n, h, dk = x.shape
    return x.reshape(*lead, n, h * dk)


def binary_features(xh: np.ndarray):
    """(features, γ) with features = γ·(sign+1)/2 (ref model.py:355-358,
    quantize.py:123-140 per-head mode)."""
    g = per_head_scale(xh)
    f = (g * (sign_pm1(xh) + 1.0) * 0.5).astype(xh.dtype, copy=False)
    return f, g


def qkv_linear_core(qf, kf, v, eps=ATTN_EPS):
    """Normalized q~(k~ᵀV) on nonnegative features (ref attention.py:113-120)."""
    kv = bmm(np.swapaxes(kf, -1, -2), v)
    z = np.sum(kf, axis=-2)
    num = bmm(qf, kv)
    den = bmm(qf, z[..., None])[..., 0] + eps
    return num / den[..., None]


def softmax_core(q, k, v):
    """Scaled-dot-product core, scale 1/√dk (ref attention.py:92-97)."""
    s = bmm(q, np.swapaxes(k, -1, -2)) / math.sqrt(q.shape[-1])
    return bmm(softmax_rows(s), v)


def token_grid_side(n: int) -> int:
    """ceil(sqrt(n)) (ref attention.py:172-175)."""
    side = math.isqrt(n)
    return side if side * side == n else side + 1


def dwconv_tokens(v: np.ndarray, k: np.ndarray) -> np.ndarray:
    """DW 3x3 over tokens laid row-major on a zero-padded square grid
    (ref attention.py:170-179)."""
    n, d = v.shape
    side = token_grid_side(n)
    grid = np.zeros((side * side, d), v.dtype)
    grid[:n] = v
    return dw3x3(grid.reshape(side, side, d), k).reshape(side * side, d)[:n]


# ---------------------------------------------------------------------------
# mixture of experts


def router_probs(x: np.ndarray, wg: np.ndarray):
    """(p, logits): logits = f32(fp64 x·W_g), p = softmax (ref moe.py:81-84)."""
    logits = mm(x, wg.astype(x.dtype, copy=False))
    return softmax_rows(logits), logits


def dispatch_plan(p: np.ndarray):
    """argmax (lowest index on ties), winning gate, ascending index lists
    (ref moe.py:87-92)."""
    expert_of = np.argmax(p, axis=-1)
    gate_of = p[np.arange(p.shape[0]), expert_of]
    index_of = [np.flatnonzero(expert_of == e) for e in range(p.shape[-1])]
    return expert_of, gate_of, index_of


def numpy_exp_tie_threshold() -> np.float32:
    """Largest f32 d ≥ 0 with np.exp(float32(-d)) == 1 on THIS host's numpy.

    For two experts, argmax(p) picks expert 0 on a logit deficit δ = l1-l0 > 0
    iff exp(-δ) rounds to exactly 1 (then p0 == p1, ref moe.py:89); that
    threshold is a property of numpy's SIMD float32 exp."""
    lo, hi = 0, int(np.float32(1e-6).view(np.uint32))
    while lo < hi:  # binary search over positive f32 bit patterns (monotone)
        mid = (lo + hi + 1) // 2
        d = np.array([mid], np.uint32).view(np.float32)
        if np.exp(-d)[0] == np.float32(1.0):
            lo = mid
        else:
            hi = mid - 1
    return np.array([lo], np.uint32).view(np.float32)[0]


# ---------------------------------------------------------------------------
# MatAdd (AddLinear)


def add_matmul(x: np.ndarray, b: np.ndarray, gamma: float) -> np.ndarray:
    """Signed accumulation of x's columns under b in float64, scaled once by
    gamma, rounded to the input dtype (ref quantize.py:143-160)."""
    x64 = np.asarray(x, dtype=np.float64)
    out = np.empty((x.shape[0], b.shape[1]), dtype=np.float64)
    for j in range(b.shape[1]):
        pos = b[:, j] > 0
        out[:, j] = x64[:, pos].sum(axis=1) - x64[:, ~pos].sum(axis=1)
    out *= gamma
    return out.astype(x.dtype, copy=False)
