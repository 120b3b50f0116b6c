"""Shift reparameterization and sign binarization on the device, mirroring the
reference `shiftadd.quantize` module (ref quantize.py).

A shift layer stores s ∈ {-1,+1} and integer P ∈ [p_min, p_max]; the device
keeps one packed byte per weight (bit7 = s<0, bits0-4 = P - p_min) which the
kernels expand to exact s·2^P (K3). `binarize` runs the K1 sign-hash kernel.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .tensor import ShapeError, to_device

P_MIN_DEFAULT = -15   # ref quantize.py:27
P_MAX_DEFAULT = 15    # ref quantize.py:28


def check_packable(p_min: int, p_max: int):
    """The device shift code is one byte: bit 7 = sign, bits 0-4 = P - p_min,
    decoded to the f32 exponent field (include/shiftadd_b200.h). Same rule as
    sa_quantize_shift (gemm.cu): ValueError outside it."""
    if p_max - p_min > 31 or p_min < -126 or p_max > 127:
        raise ValueError(f"exponent range [{p_min}, {p_max}] does not fit the 5-bit device "
                         "shift code (need p_max - p_min <= 31, -126 <= p_min, p_max <= 127)")


@dataclass
class QuantConfig:
    """ref quantize.py:31-41"""

    p_min: int = P_MIN_DEFAULT
    p_max: int = P_MAX_DEFAULT
    scale_mode: str = "per-matrix"  # or "per-head"

    def __post_init__(self):
        if self.p_min >= self.p_max:
            raise ValueError(f"p_min {self.p_min} must be below p_max {self.p_max}")
        check_packable(self.p_min, self.p_max)
        if self.scale_mode not in ("per-matrix", "per-head"):
            raise ValueError(f"unknown scale_mode {self.scale_mode!r}")


@dataclass
class ShiftLinear:
    """Sign flips and power-of-two exponents of one linear layer (ref
    quantize.py:44-59), plus the packed device form the kernels read."""

    s: torch.Tensor          # {-1,+1} float32, (in_dim, out_dim)
    p: torch.Tensor          # int32 exponents, same shape
    p_min: int = P_MIN_DEFAULT
    p_max: int = P_MAX_DEFAULT
    packed: torch.Tensor = field(default=None, repr=False)  # uint8, same shape

    def __post_init__(self):
        self.s = to_device(self.s, torch.float32)
        self.p = to_device(self.p, torch.int32)
        if self.s.shape != self.p.shape or self.s.ndim != 2:
            raise ShapeError(f"s/p shapes differ: {tuple(self.s.shape)} vs {tuple(self.p.shape)}")
        check_packable(self.p_min, self.p_max)
        if self.packed is None:
            if int(self.p.min()) < self.p_min or int(self.p.max()) > self.p_max:
                raise ValueError("exponents outside [p_min, p_max]")
            self.packed = (((self.s < 0).to(torch.uint8) << 7)
                           | (self.p - self.p_min).to(torch.uint8)).contiguous()

    @property
    def in_dim(self) -> int:
        return self.s.shape[0]

    @property
    def out_dim(self) -> int:
        return self.s.shape[1]


@dataclass
class AddLinear:
    """Binarized weights plus one trailing scale (ref quantize.py:62-75); the
    device keeps one sign byte per weight (bit 7 = b < 0) for sa_add_linear."""

    b: torch.Tensor          # {-1,+1} float32, (in_dim, out_dim)
    gamma: float
    signs: torch.Tensor = field(default=None, repr=False)  # uint8, same shape

    def __post_init__(self):
        self.b = to_device(self.b, torch.float32)
        if self.b.ndim != 2:
            raise ShapeError(f"AddLinear needs a 2-D sign matrix, got {tuple(self.b.shape)}")
        self.gamma = float(self.gamma)
        if self.signs is None:
            self.signs = ((self.b < 0).to(torch.uint8) << 7).contiguous()

    @property
    def in_dim(self) -> int:
        return self.b.shape[0]

    @property
    def out_dim(self) -> int:
        return self.b.shape[1]


def sign_unit(x) -> torch.Tensor:
    """Sign with sign(0) := +1 (so -0.0 and NaN map to +1) (ref quantize.py:78-80)."""
    x = to_device(x, None)
    one = torch.ones((), dtype=x.dtype, device=x.device)
    return torch.where(x < 0, -one, one)


def quantize_shift(w, cfg: QuantConfig = QuantConfig()) -> ShiftLinear:
    """Round onto the sign·2^P grid on the device (ref quantize.py:83-96): P =
    rint(log2|w|) clamped to [p_min, p_max], zeros → p_min. Exact: P is taken
    from the exponent field plus one comparison against √2 (K3 packing)."""
    w = to_device(w)
    if w.ndim != 2:
        raise ShapeError(f"expected a 2-D weight matrix, got shape {tuple(w.shape)}")
    packed = torch.empty(w.shape, dtype=torch.uint8, device=w.device)
    s = torch.empty(w.shape, dtype=torch.float32, device=w.device)
    p = torch.empty(w.shape, dtype=torch.int32, device=w.device)
    _lib.call("sa_quantize_shift", _lib.ptr(w), w.numel(), cfg.p_min, cfg.p_max,
              _lib.ptr(packed), _lib.ptr(s), _lib.ptr(p), _lib.stream())
    return ShiftLinear(s=s, p=p, p_min=cfg.p_min, p_max=cfg.p_max, packed=packed)


def reconstruct(layer: ShiftLinear, dtype=torch.float32) -> torch.Tensor:
    """Exact s·2^P (ref quantize.py:99-101)."""
    return torch.ldexp(layer.s.to(dtype), layer.p.to(dtype))


def shift_forward(x, layer: ShiftLinear, variant: int = 0) -> torch.Tensor:
    """x @ (s·2^P) (ref quantize.py:104-109). variant 0: decoded weights on the
    GEMM core; variant 1: literal exponent-field add (MatShift)."""
    x = to_device(x)
    if x.shape[-1] != layer.in_dim:
        raise ShapeError(f"input extent {x.shape[-1]} != layer in_dim {layer.in_dim}")
    x2 = x.reshape(-1, layer.in_dim)
    y = torch.empty((x2.shape[0], layer.out_dim), dtype=torch.float32, device=x.device)
    _lib.call("sa_shift_linear", _lib.ptr(x2), _lib.ptr(layer.packed), _lib.ptr(y), x2.shape[0],
              layer.in_dim, layer.out_dim, layer.p_min, int(variant), _lib.stream())
    return y.reshape(*x.shape[:-1], layer.out_dim)


def sign_hash(x, heads: int, batch: int):
    """K1 on a flat (batch*n, d) projection: (codes uint32 [batch, heads, n,
    ceil(dk/32)], gamma float32 [batch, heads])."""
    x = to_device(x)
    if x.ndim != 2 or x.shape[0] % batch:
        raise ShapeError(f"sign_hash expects (batch*n, d), got {tuple(x.shape)}")
    n = x.shape[0] // batch
    d = x.shape[1]
    if d % heads:
        raise ShapeError(f"model_dim {d} not divisible by heads {heads}")
    dk = d // heads
    W = (dk + 31) // 32
    codes = torch.empty((batch, heads, n, W), dtype=torch.int32, device=x.device)
    gamma = torch.empty((batch, heads), dtype=torch.float32, device=x.device)
    ws_n = _lib.load().sa_sign_hash_workspace(batch, n, d, heads)
    ws = _lib.Workspace.get(ws_n)
    _lib.call("sa_sign_hash", _lib.ptr(x), batch, n, d, heads, _lib.ptr(codes), _lib.ptr(gamma),
              _lib.ptr(ws), ws.numel(), _lib.stream())
    return codes, gamma


def unpack_codes(codes: torch.Tensor, dk: int) -> torch.Tensor:
    """[..., W] packed words → [..., dk] {0,1} uint8."""
    shifts = torch.arange(32, device=codes.device, dtype=torch.int32)
    bits = (codes.unsqueeze(-1) >> shifts) & 1
    return bits.reshape(*codes.shape[:-1], -1)[..., :dk].to(torch.uint8)


def binarize(x, scale_mode: str = "per-matrix"):
    """Split x into ±1 sign codes and a mean-|x| scale (ref quantize.py:123-140).

    per-head: x is stacked (heads, ...) and gamma has shape (heads, 1, ..., 1).
    Runs the K1 hash kernel (each leading slice is one 'image' with one head)."""
    x = to_device(x)
    if x.numel() == 0:
        raise ShapeError("cannot binarize an empty array")
    if scale_mode not in ("per-matrix", "per-head"):
        raise ValueError(f"unknown scale_mode {scale_mode!r}")
    lead = x.shape[0] if (scale_mode == "per-head" and x.ndim > 1) else 1
    flat = x.reshape(lead, -1)
    per = flat.shape[1]
    d = 32 if per % 32 == 0 else (16 if per % 16 == 0 else None)
    if d is None:   # ragged groups (weight matrices): device torch reductions, fp64 mean
        b = sign_unit(x).to(torch.float32)
        g = flat.abs().to(torch.float64).mean(dim=1).to(torch.float32)
        if scale_mode == "per-matrix":
            return b, float(g[0])
        return b, g.reshape((lead,) + (1,) * (x.ndim - 1))
    rows = flat.reshape(lead * (per // d), d)
    codes, gamma = sign_hash(rows, heads=1, batch=lead)
    bits = unpack_codes(codes.reshape(-1, 1), d).reshape(x.shape)
    b = bits.to(torch.float32) * 2.0 - 1.0
    if scale_mode == "per-matrix":
        return b, float(gamma.reshape(-1)[0])
    return b, gamma.reshape((lead,) + (1,) * (x.ndim - 1))


def add_matmul(x, layer: AddLinear) -> torch.Tensor:
    """Signed accumulation of x's columns under b, scaled once by gamma (ref
    quantize.py:143-160): sa_add_linear adds / subtracts in fp64 and multiplies
    by gamma once, then rounds to float32 — the reference's arithmetic."""
    x = to_device(x)
    if x.ndim != 2:
        raise ShapeError(f"add_matmul expects a 2-D input, got {tuple(x.shape)}")
    if x.shape[1] != layer.in_dim:
        raise ShapeError(f"input extent {x.shape[1]} != layer in_dim {layer.in_dim}")
    y = torch.empty((x.shape[0], layer.out_dim), dtype=torch.float32, device=x.device)
    _lib.call("sa_add_linear", _lib.ptr(x), _lib.ptr(layer.signs), float(layer.gamma),
              _lib.ptr(y), x.shape[0], layer.in_dim, layer.out_dim, _lib.stream())
    return y


def reconstruct_add(layer: AddLinear, dtype=torch.float32) -> torch.Tensor:
    """gamma·b (ref quantize.py:188-189)."""
    return (layer.gamma * layer.b.to(torch.float64)).to(dtype)


@dataclass
class ReparamResult:
    """ref quantize.py:171-174"""

    layer: object                  # ShiftLinear or AddLinear
    shadow: torch.Tensor           # dense copy of the source weights


def reparam_linear(dense_w, target: str, cfg: QuantConfig = QuantConfig()) -> ReparamResult:
    """Convert a dense matrix into a shift or add layer plus its shadow (ref
    quantize.py:177-185)."""
    w = to_device(dense_w)
    if target == "shift":
        return ReparamResult(layer=quantize_shift(w, cfg), shadow=w.clone())
    if target == "add":
        b, gamma = binarize(w, scale_mode="per-matrix")
        return ReparamResult(layer=AddLinear(b=b, gamma=gamma), shadow=w.clone())
    raise ValueError(f"unknown reparameterization target {target!r}")
