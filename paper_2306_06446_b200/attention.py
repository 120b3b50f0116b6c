"""Multi-head attention in softmax form and in binary Q(KV) / (QK)V form on the
device, mirroring the reference `shiftadd.attention` module (ref attention.py).

Binary mode (ref attention.py:155-167, model.py:354-373): Q and K are hashed
to packed {0,1} codes with per-(image, head) mean-|x| scales (K1), the token
mixing runs on the codes with additions only (K2a linear order, K2b quadratic
Hamming order), and the DWConv V-branch is fused into the output pass.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Optional, Union

import torch

from . import _lib
from .quantize import AddLinear, ShiftLinear, add_matmul, shift_forward, sign_hash
from .tensor import ShapeError, matmul, to_device

MODES = ("softmax", "linear", "linear-binary")   # ref attention.py:28
ORDERS = ("auto", "linear", "quadratic")
PHI_EPS = 1e-6
EPS_NORM = 1e-6                                  # ref attention.py:32

Projection = Union[torch.Tensor, ShiftLinear, AddLinear]


@dataclass
class AttentionConfig:
    """ref attention.py:37-54 (+ `order`: which association the binary core uses)."""

    heads: int
    model_dim: int
    mode: str = "softmax"
    eps_norm: float = EPS_NORM
    use_dwconv: bool = True
    order: str = "auto"

    def __post_init__(self):
        if self.model_dim % self.heads != 0:
            raise ShapeError(f"model_dim {self.model_dim} not divisible by heads {self.heads}")
        if self.mode not in MODES:
            raise ValueError(f"unknown attention mode {self.mode!r}")
        if self.order not in ORDERS:
            raise ValueError(f"unknown binary order {self.order!r}")

    @property
    def head_dim(self) -> int:
        return self.model_dim // self.heads


@dataclass
class AttentionWeights:
    """ref attention.py:57-63"""

    wq: Projection
    wk: Projection
    wv: Projection
    wo: Projection
    dw_kernels: Optional[torch.Tensor] = None  # (3, 3, model_dim)


def project(x, w: Projection) -> torch.Tensor:
    """ref attention.py:66-71"""
    if isinstance(w, ShiftLinear):
        return shift_forward(x, w)
    if isinstance(w, AddLinear):
        return add_matmul(x, w)
    return matmul(x, w)


def split_heads(x, heads: int) -> torch.Tensor:
    """(..., n, d) -> (..., heads, n, d/heads) (ref attention.py:74-78)."""
    x = to_device(x)
    *lead, n, d = x.shape
    return x.reshape(*lead, n, heads, d // heads).transpose(-3, -2)


def merge_heads(x) -> torch.Tensor:
    """(..., heads, n, dk) -> (..., n, heads*dk) (ref attention.py:81-85)."""
    x = to_device(x, None).transpose(-3, -2).contiguous()
    *lead, n, h, dk = x.shape
    return x.reshape(*lead, n, h * dk)


def token_grid_side(n: int) -> int:
    s = math.isqrt(n)
    return s if s * s == n else s + 1


# ---------------------------------------------------------------------------
# device cores on flat (batch*n, d) activations


def binary_core(q, k, v, batch: int, heads: int, dw=None, eps: float = EPS_NORM,
                order: str = "auto") -> torch.Tensor:
    """Binary attention on flat projections: hash q/k (K1), then the additive
    core (K2a/K2b) with the DWConv branch fused. Returns merged heads
    (batch*n, d) — the input of W_O (ref model.py:354-373)."""
    M, d = v.shape
    n = M // batch
    cq, gq = sign_hash(q, heads, batch)
    ck, gk = sign_hash(k, heads, batch)
    return binary_core_codes(cq, ck, gq, gk, v, batch, heads, dw, eps, order)


def binary_core_codes(cq, ck, gq, gk, v, batch: int, heads: int, dw=None,
                      eps: float = EPS_NORM, order: str = "auto") -> torch.Tensor:
    M, d = v.shape
    n = M // batch
    out = torch.empty_like(v)
    if order == "quadratic":
        _lib.call("sa_hamming_attn", _lib.ptr(cq), _lib.ptr(ck), _lib.ptr(gq), _lib.ptr(gk),
                  _lib.ptr(v), _lib.ptr(dw), _lib.ptr(out), batch, n, d, heads, float(eps),
                  _lib.stream())
    else:
        ws = _lib.Workspace.get(_lib.load().sa_linear_binary_attn_workspace(batch, n, d, heads),
                                slot=2)
        _lib.call("sa_linear_binary_attn", _lib.ptr(cq), _lib.ptr(ck), _lib.ptr(gq),
                  _lib.ptr(gk), _lib.ptr(v), _lib.ptr(dw), _lib.ptr(out), batch, n, d, heads,
                  float(eps), _lib.ptr(ws), ws.numel(), _lib.stream())
    return out


def softmax_core_flat(q, k, v, batch: int, heads: int) -> torch.Tensor:
    """Softmax attention (ref attention.py:92-97) on flat projections."""
    M, d = v.shape
    out = torch.empty_like(v)
    _lib.call("sa_softmax_attn", _lib.ptr(q), _lib.ptr(k), _lib.ptr(v), _lib.ptr(out), batch,
              M // batch, d, heads, _lib.stream())
    return out


def binary_popcounts(cq, ck, dk: int, with_scores: bool = False):
    """Integer statistics of the binary core: cnt [B*h, dk], D [B*h, n] and
    optionally S [B*h, n, n] = popc(cq_i & ck_j)."""
    B, h, n, _ = cq.shape
    dev = cq.device
    cnt = torch.empty((B * h, dk), dtype=torch.int32, device=dev)
    D = torch.empty((B * h, n), dtype=torch.int32, device=dev)
    S = torch.empty((B * h, n, n), dtype=torch.int32, device=dev) if with_scores else None
    _lib.call("sa_binary_popcounts", _lib.ptr(cq), _lib.ptr(ck), B, n, dk, h, _lib.ptr(cnt),
              _lib.ptr(D), _lib.ptr(S), _lib.stream())
    return cnt, D, S


# ---------------------------------------------------------------------------
# reference-shaped module API (per-head stacks (H, n, dk) / one sequence (n, d))


def softmax_core(q, k, v):
    """(out, cache) on stacked heads (H, n, dk) (ref attention.py:92-97)."""
    q, k, v = to_device(q), to_device(k), to_device(v)
    H, n, dk = q.shape
    flat = lambda t: t.reshape(H * n, dk).contiguous()  # noqa: E731  one 'image' per head
    out = softmax_core_flat(flat(q), flat(k), flat(v), H, 1)
    return out.reshape(H, n, dk), None


def binarize_qk(q, k, cfg: AttentionConfig):
    """Per-head sign codes → {0,1}·gamma features (ref attention.py:155-167).
    q, k are (n, model_dim); returns (qf, kf, (gq, gk)) head-split."""
    q, k = to_device(q), to_device(k)
    from .quantize import unpack_codes
    cq, gq = sign_hash(q, cfg.heads, 1)
    ck, gk = sign_hash(k, cfg.heads, 1)
    dk = cfg.head_dim
    bq = unpack_codes(cq[0], dk).to(torch.float32)
    bk = unpack_codes(ck[0], dk).to(torch.float32)
    gq3 = gq.reshape(cfg.heads, 1, 1)
    gk3 = gk.reshape(cfg.heads, 1, 1)
    return gq3 * bq, gk3 * bk, (gq3, gk3)


def linear_core(qf, kf, v, eps_norm: float):
    """Normalized q~(k~ᵀV) (ref attention.py:113-120) for BINARY features
    (gamma·{0,1}, as produced by `binarize_qk`): codes and per-head scales are
    recovered from the features and the additive K2a core runs on them. The
    relu-feature 'linear' mode is outside the inference hot path."""
    qf, kf, v = to_device(qf), to_device(kf), to_device(v)
    H, n, dk = qf.shape
    if dk not in (16, 32, 64):
        raise ShapeError(f"head dim {dk} unsupported by the device core")
    gq = qf.amax(dim=(1, 2))
    gk = kf.amax(dim=(1, 2))
    if not (torch.all((qf == 0) | (qf == gq[:, None, None]))
            and torch.all((kf == 0) | (kf == gk[:, None, None]))):
        raise ValueError("device linear_core needs binary (gamma·{0,1}) features")
    # re-hash: a feature of 0 must map to code 0 → hash (f - gamma/2)
    cq, _ = sign_hash((qf - 0.5 * gq[:, None, None]).reshape(H * n, dk), 1, H)
    ck, _ = sign_hash((kf - 0.5 * gk[:, None, None]).reshape(H * n, dk), 1, H)
    out = binary_core_codes(cq, ck, gq.contiguous(), gk.contiguous(), v.reshape(H * n, dk).contiguous(),
                            H, 1, None, eps_norm, "linear")
    return out.reshape(H, n, dk), None


def _dwconv_tokens(v, kernels):
    """(out, side): DWConv over the ceil(sqrt(n)) token grid (ref attention.py:170-179)."""
    v = to_device(v)
    kernels = to_device(kernels)
    n, d = v.shape
    out = torch.empty_like(v)
    _lib.call("sa_dwconv_tokens", _lib.ptr(v), _lib.ptr(kernels), _lib.ptr(out), 1, n, d, 0,
              _lib.stream())
    return out, token_grid_side(n)


def softmax_attention(x, w: AttentionWeights, cfg: AttentionConfig) -> torch.Tensor:
    """ref attention.py:198-206 on one sequence (n, d)."""
    x = to_device(x)
    if x.shape[-1] != cfg.model_dim:
        raise ShapeError(f"token dim {x.shape[-1]} != model_dim {cfg.model_dim}")
    q, k, v = project(x, w.wq), project(x, w.wk), project(x, w.wv)
    return project(softmax_core_flat(q, k, v, 1, cfg.heads), w.wo)


def linear_attention(x, w: AttentionWeights, cfg: AttentionConfig) -> torch.Tensor:
    """ref attention.py:209-227 (binary mode) on one sequence (n, d)."""
    if cfg.mode not in ("linear", "linear-binary"):
        raise ValueError(f"linear_attention called with mode {cfg.mode!r}")
    if cfg.mode == "linear":
        raise ValueError("the relu-feature 'linear' mode is outside the inference hot path")
    x = to_device(x)
    if x.shape[-1] != cfg.model_dim:
        raise ShapeError(f"token dim {x.shape[-1]} != model_dim {cfg.model_dim}")
    q, k, v = project(x, w.wq), project(x, w.wk), project(x, w.wv)
    dw = to_device(w.dw_kernels) if (cfg.use_dwconv and w.dw_kernels is not None) else None
    merged = binary_core(q, k, v, 1, cfg.heads, dw, cfg.eps_norm, cfg.order)
    return project(merged, w.wo)


def attention(x, w: AttentionWeights, cfg: AttentionConfig) -> torch.Tensor:
    """ref attention.py:230-234"""
    if cfg.mode == "softmax":
        return softmax_attention(x, w, cfg)
    return linear_attention(x, w, cfg)
