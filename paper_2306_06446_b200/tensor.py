"""Device tensor substrate mirroring the reference `shiftadd.tensor` module
(ref tensor.py) for the inference path.

Activations are float32 CUDA tensors in the reference's flat (tokens,
channels) layout. Products, layer norms and convolutions run in
libshiftadd_b200.so; numpy inputs are accepted and moved to the device once.
Backward passes are out of scope (inference only).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import ShapeError, StateError  # noqa: F401  (re-exported, ref tensor.py:25-30)

DTYPE = np.float32
LAYERNORM_EPS = 1e-5   # ref tensor.py:22


def make_rng(seed: int) -> np.random.Generator:
    """PCG64 stream; weights are drawn on the host exactly like the reference
    (ref tensor.py:33-35) and then moved to the device."""
    return np.random.Generator(np.random.PCG64(seed))


def device() -> torch.device:
    return torch.device("cuda", torch.cuda.current_device())


def to_device(x, dtype=torch.float32) -> torch.Tensor:
    """numpy / torch → contiguous CUDA tensor (one copy at most)."""
    if isinstance(x, torch.Tensor):
        t = x if x.is_cuda else x.to(device(), non_blocking=False)
        if dtype is not None and t.dtype != dtype:
            t = t.to(dtype)
        return t.contiguous()
    arr = np.ascontiguousarray(x)
    t = torch.from_numpy(arr)
    if dtype is not None:
        t = t.to(dtype)
    return t.to(device()).contiguous()


def tensor(data, dtype=torch.float32) -> torch.Tensor:
    """Materialize `data` as a contiguous device tensor (ref tensor.py:38-40)."""
    return to_device(np.asarray(data, dtype=np.float32) if not isinstance(data, torch.Tensor)
                     else data, dtype)


@dataclass
class GradPair:
    """Parameter holder kept for API compatibility (ref tensor.py:43-60). Only
    `value` is used: this package is inference-only, so `grad` stays None."""

    value: torch.Tensor
    grad: object = None


def matmul(a, b) -> torch.Tensor:
    """2-D product (ref tensor.py:68-75) on the device GEMM."""
    a = to_device(a)
    b = to_device(b)
    if a.ndim != 2 or b.ndim != 2:
        raise ShapeError(f"matmul expects 2-D operands, got {tuple(a.shape)} and {tuple(b.shape)}")
    if a.shape[1] != b.shape[0]:
        raise ShapeError(f"inner extents differ: {tuple(a.shape)} x {tuple(b.shape)}")
    M, K = a.shape
    N = b.shape[1]
    c = torch.empty((M, N), dtype=torch.float32, device=a.device)
    _lib.call("sa_gemm", _lib.ptr(a), _lib.ptr(b), _lib.ptr(c), M, K, N, _lib.stream())
    return c


def layernorm(x, gain, bias, eps: float = LAYERNORM_EPS):
    """(y, cache) like the reference (ref tensor.py:114-128); cache is None."""
    x = to_device(x)
    gain, bias = to_device(gain), to_device(bias)
    d = x.shape[-1]
    if gain.shape[-1] != d or bias.shape[-1] != d:
        raise ShapeError(f"last-axis extent {d} does not match affine params")
    y = torch.empty_like(x)
    _lib.call("sa_layernorm", _lib.ptr(x), _lib.ptr(gain), _lib.ptr(bias), _lib.ptr(y),
              x.numel() // d, d, float(eps), _lib.stream())
    return y, None


def dwconv3x3(x, kernels) -> torch.Tensor:
    """Depthwise 3x3, zero padding 1 (ref tensor.py:177-199), on a square
    (side, side, c) or (batch, side, side, c) grid."""
    x = to_device(x)
    kernels = to_device(kernels)
    if kernels.shape[0] != 3 or kernels.shape[1] != 3:
        raise ShapeError(f"kernels must be 3x3xC, got {tuple(kernels.shape)}")
    if x.shape[-1] != kernels.shape[2]:
        raise ShapeError(f"channel mismatch: input {x.shape[-1]}, kernels {kernels.shape[2]}")
    squeeze = x.ndim == 3
    xb = x[None] if squeeze else x
    b, h, w, c = xb.shape
    if h != w:
        raise ShapeError("the device DWConv runs on square token grids")
    out = torch.empty_like(xb)
    _lib.call("sa_dwconv_tokens", _lib.ptr(xb.contiguous()), _lib.ptr(kernels), _lib.ptr(out),
              b, h * w, c, 0, _lib.stream())
    return out[0] if squeeze else out
