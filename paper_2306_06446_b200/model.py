"""Layers, blocks and model builders on the device, mirroring the reference
`shiftadd.model` module (ref model.py) for the inference path.

Every layer keeps the reference's constructor signature, `kind` attribute and
`forward(x, train=False)` entry; forwards take and return CUDA tensors in the
reference's flat (tokens, channels) layout and run in libshiftadd_b200.so.
Each forward also accepts `residual=` so a Block fuses its residual add into
the producing kernel's epilogue. Training (backward, optimizers, balance
losses) is outside the inference hot path; `train=True` raises.

Weights are drawn on the host with the reference's PCG64 order (ref
model.py:487-553) and uploaded once, so `Model(cfg)` holds exactly the
reference `Model(cfg)`'s parameters.
"""

from __future__ import annotations

import os
from dataclasses import asdict, dataclass
from typing import List, Optional

import numpy as np
import torch

from . import _lib
from . import attention as A
from . import moe as MOE
from . import quantize as Q
from . import specs as SPECS
from .tensor import GradPair, ShapeError, StateError, make_rng, to_device

ATTN_MODES = ("softmax", "linear", "linear-binary")   # ref model.py:31
LINEAR_MODES = ("dense", "shift", "moe")              # ref model.py:32


@dataclass
class BlockConfig:
    """ref model.py:35-53 (+ binary_order: linear K^T V or quadratic Hamming)."""

    d: int
    h: int
    mlp_ratio: float = 4.0
    attn_mode: str = "softmax"
    mlp_mode: str = "dense"
    attn_linear_mode: str = "dense"
    exempt: bool = False
    binary_order: str = "auto"

    def __post_init__(self):
        if self.d % self.h != 0:
            raise ShapeError(f"model dim {self.d} not divisible by heads {self.h}")
        if self.attn_mode not in ATTN_MODES:
            raise ValueError(f"unknown attn_mode {self.attn_mode!r}")
        if self.mlp_mode not in LINEAR_MODES:
            raise ValueError(f"unknown mlp_mode {self.mlp_mode!r}")
        if self.attn_linear_mode not in LINEAR_MODES:
            raise ValueError(f"unknown attn_linear_mode {self.attn_linear_mode!r}")
        if self.binary_order not in A.ORDERS:
            raise ValueError(f"unknown binary_order {self.binary_order!r}")


@dataclass
class ModelConfig:
    """ref model.py:56-81"""

    blocks: List[BlockConfig]
    patch: int = 4
    img: int = 16
    classes: int = 5
    seed: int = 0
    channels: int = 3

    def __post_init__(self):
        if self.img % self.patch != 0:
            raise ShapeError(f"image side {self.img} not divisible by patch {self.patch}")

    @property
    def tokens(self) -> int:
        side = self.img // self.patch
        return side * side

    def to_dict(self) -> dict:
        return asdict(self)

    @classmethod
    def from_dict(cls, payload: dict) -> "ModelConfig":
        blocks = [BlockConfig(**b) for b in payload["blocks"]]
        rest = {k: v for k, v in payload.items() if k != "blocks"}
        return cls(blocks=blocks, **rest)


@dataclass
class MoeConfig:
    """ref model.py:84-88"""

    sigma: float = 0.1
    lam: float = 0.01
    lat: tuple = (3.0, 1.0)   # (mult expert, shift expert)


def _no_train(train):
    if train:
        raise NotImplementedError("this package implements the inference path only")


# GEMM engine: "tc" = tcgen05 tensor cores with float32-faithful split-bf16
# operands (default); "simt" = the CUDA-core FFMA path (kept for A/B checks).
GEMM_ENGINE = os.environ.get("SA_GEMM", "tc")


def tc_enabled() -> bool:
    return GEMM_ENGINE == "tc"


# LayerNorm fused with the routers that read its output (d = 32 / 64)
FUSE_LN_ROUTE = os.environ.get("SA_FUSE_LN_ROUTE", "1") == "1"
FUSE_EMBED_LN = os.environ.get("SA_FUSE_EMBED_LN", "1") == "1"
FUSE_GROUPED_QKV = os.environ.get("SA_FUSE_GROUPED_QKV", "1") == "1"
FUSE_DENSE_QKV = os.environ.get("SA_FUSE_DENSE_QKV", "1") == "1"
# fc1 → GELU → fc2 in one tensor-core kernel (d = 32 / 64)
FUSE_MLP = os.environ.get("SA_FUSE_MLP", "1") == "1"
# LN1 + q/k/v routers + both experts of q/k/v + sign-hash in one kernel (d = 32 / 64)
FUSE_QKV = os.environ.get("SA_FUSE_QKV", "1") == "1"


FUSE_O = os.environ.get("SA_FUSE_O", "1") == "1"
# the block's LN2 + MLP router in the W_O kernel's epilogue (sa_fused_moe_linear_ln_route)
FUSE_LN2 = os.environ.get("SA_FUSE_LN2", "1") == "1"
# a stage's final LayerNorm in the last block's fused MLP kernel (d = 32)
FUSE_STAGE_LN = os.environ.get("SA_FUSE_STAGE_LN", "1") == "1"
FUSE_STAGE_LN64 = os.environ.get("SA_FUSE_STAGE_LN64", "1") == "1"


def _fused_o_ok(mod, x2) -> bool:
    return (FUSE_O and tc_enabled() and _dual_expert_linear(mod) and x2.dim() == 2
            and x2.shape[1] == mod.experts[0].in_dim
            and bool(_lib.load().sa_fused_moe_linear_ok(x2.shape[1])))


def _dual_expert_linear(m) -> bool:
    return (isinstance(m, MoeModule) and len(m.experts) == 2 and isinstance(m.experts[0], Linear)
            and isinstance(m.experts[1], ShiftLinearLayer)
            and m.experts[0].in_dim == m.experts[0].out_dim)


def fused_mlp_w1_bn(d: int = 32) -> int:
    """Hidden-chunk width the fused MLP kernel reads W1 packed with at model dim d."""
    return int(_lib.load().sa_tc_fused_mlp_chunk(d))


def fused_mlp_ok(d, hidden) -> bool:
    return tc_enabled() and FUSE_MLP and bool(_lib.load().sa_tc_fused_mlp_ok(d, hidden))


def _pack_weight(w, kind, K, N, p_min, bn=None):
    """Pack a (K, N) weight into the tensor-core shared-memory image (K3/K6)."""
    lib = _lib.load()
    bn = int(lib.sa_tc_tile_n(N)) if bn is None else int(bn)
    out = torch.empty(int(lib.sa_weight_pack_bytes(K, N, kind, bn)), dtype=torch.uint8,
                      device=w.device)
    _lib.call("sa_weight_pack", _lib.ptr(w), kind, K, N, p_min, bn, _lib.ptr(out), _lib.stream())
    return out, bn


def _stream():
    return _lib.stream()


# ---------------------------------------------------------------------------
# layers


class Linear:
    """Dense y = x @ w, no bias (ref model.py:95-123)."""

    kind = "dense"

    def __init__(self, w):
        self.w = GradPair(to_device(w))

    @property
    def in_dim(self):
        return self.w.value.shape[0]

    @property
    def out_dim(self):
        return self.w.value.shape[1]

    def weight_arg(self):
        return self.w.value, _lib.SA_W_DENSE, Q.P_MIN_DEFAULT

    def tc_pack(self, bn=None):
        """(packed planes, bn, kind) for the tensor-core path, built once per bn."""
        cache = self.__dict__.setdefault("_tc", {})
        if bn not in cache:
            pk, b = _pack_weight(self.w.value, _lib.SA_W_DENSE, self.in_dim, self.out_dim, -15, bn)
            cache[bn] = (pk, b, _lib.SA_W_DENSE)
        return cache[bn]

    def forward(self, x, train=False, residual=None, act=0):
        _no_train(train)
        return _linear_call(self, x, residual, act)

    def named_params(self, prefix):
        yield prefix + ".w", self.w

    def extra_blobs(self, prefix):
        return ()

    def post_step(self):
        self._tc = {}   # the packed tensor-core planes follow the (possibly reloaded) weights


class ShiftLinearLayer:
    """Shift layer: forward uses the quantized sign/exponent pair of the dense
    shadow (ref model.py:126-166); the packed codes live on the device."""

    kind = "shift"

    def __init__(self, shadow, quant_cfg: Q.QuantConfig = None):
        self.quant_cfg = quant_cfg or Q.QuantConfig()
        self.w = GradPair(to_device(shadow))
        self.quant = Q.quantize_shift(self.w.value, self.quant_cfg)

    def requantize(self):
        self.quant = Q.quantize_shift(self.w.value, self.quant_cfg)
        self._tc = {}

    def tc_pack(self, bn=None):
        cache = self.__dict__.setdefault("_tc", {})
        if bn not in cache:
            pk, b = _pack_weight(self.quant.packed, _lib.SA_W_SHIFT, self.in_dim, self.out_dim,
                                 self.quant.p_min, bn)
            cache[bn] = (pk, b, _lib.SA_W_SHIFT)
        return cache[bn]

    @property
    def in_dim(self):
        return self.quant.in_dim

    @property
    def out_dim(self):
        return self.quant.out_dim

    def weight_arg(self):
        return self.quant.packed, _lib.SA_W_SHIFT, self.quant.p_min

    def forward(self, x, train=False, residual=None, act=0):
        _no_train(train)
        return _linear_call(self, x, residual, act)

    def named_params(self, prefix):
        yield prefix + ".shadow", self.w

    def extra_blobs(self, prefix):
        yield prefix + ".quant_s", self.quant.s
        yield prefix + ".quant_p", self.quant.p

    def post_step(self):
        self.requantize()


def _linear_call(layer, x, residual, act):
    x = to_device(x)
    lead = x.shape[:-1]
    x2 = x.reshape(-1, x.shape[-1])
    if x2.shape[1] != layer.in_dim:
        raise ShapeError(f"input extent {x2.shape[1]} != layer in_dim {layer.in_dim}")
    y = torch.empty((x2.shape[0], layer.out_dim), dtype=torch.float32, device=x.device)
    res = residual.reshape(y.shape) if residual is not None else None
    if tc_enabled():
        # few row tiles (e.g. the classifier head, M = batch): narrow column
        # tiles so the grid covers more SMs
        small = x2.shape[0] <= 4096 and layer.out_dim > 256
        pk, bn, kind = layer.tc_pack(64) if small else layer.tc_pack()
        _lib.call("sa_tc_linear", _lib.ptr(x2), _lib.ptr(pk), kind, bn, _lib.ptr(y), x2.shape[0],
                  layer.in_dim, layer.out_dim, _lib.ptr(res), int(act), _stream())
        return y.reshape(*lead, layer.out_dim)
    w, kind, p_min = layer.weight_arg()
    _lib.call("sa_linear", _lib.ptr(x2), _lib.ptr(w), kind, _lib.ptr(y), x2.shape[0],
              layer.in_dim, layer.out_dim, p_min, _lib.ptr(res), int(act), _stream())
    return y.reshape(*lead, layer.out_dim)


class LayerNorm:
    """ref model.py:168-193 (eps 1e-5, biased variance)."""

    def __init__(self, dim: int, dtype=np.float32):
        self.gain = GradPair(to_device(np.ones(dim, np.float32)))
        self.bias = GradPair(to_device(np.zeros(dim, np.float32)))

    def forward(self, x, train=False):
        _no_train(train)
        x = to_device(x)
        d = x.shape[-1]
        y = torch.empty_like(x)
        _lib.call("sa_layernorm", _lib.ptr(x), _lib.ptr(self.gain.value), _lib.ptr(self.bias.value),
                  _lib.ptr(y), x.numel() // d, d, 1e-5, _stream())
        return y

    def named_params(self, prefix):
        yield prefix + ".gain", self.gain
        yield prefix + ".bias", self.bias

    def post_step(self):
        pass


class Mlp:
    """fc1 → GELU(tanh) → fc2 (ref model.py:196-228); both linears run in one
    call with the GELU fused into fc1's epilogue."""

    def __init__(self, fc1, fc2):
        self.fc1 = fc1
        self.fc2 = fc2

    def forward(self, x, train=False, residual=None):
        _no_train(train)
        x = to_device(x)
        if not (hasattr(self.fc1, "weight_arg") and hasattr(self.fc2, "weight_arg")):
            # the fused device MLP needs this package's Linear / ShiftLinearLayer
            raise NotImplementedError(f"unsupported MLP layers {type(self.fc1).__name__}, "
                                      f"{type(self.fc2).__name__}")
        lead = x.shape[:-1]
        x2 = x.reshape(-1, x.shape[-1])
        M, d = x2.shape
        hidden = self.fc1.out_dim
        w1, k1, pm1 = self.fc1.weight_arg()
        w2, k2, pm2 = self.fc2.weight_arg()
        if k1 == _lib.SA_W_SHIFT and k2 == _lib.SA_W_SHIFT and pm1 != pm2:
            raise ValueError("fc1/fc2 shift layers must share p_min")
        p_min = pm1 if k1 == _lib.SA_W_SHIFT else pm2
        y = torch.empty((M, self.fc2.out_dim), dtype=torch.float32, device=x.device)
        res = residual.reshape(y.shape) if residual is not None else None
        if fused_mlp_ok(d, hidden) and k1 == k2:
            p1, _, _ = self.fc1.tc_pack(fused_mlp_w1_bn(d))
            p2, _, _ = self.fc2.tc_pack(d)
            _lib.call("sa_tc_mlp_fused", _lib.ptr(x2), _lib.ptr(p1), k1, _lib.ptr(p2), k2,
                      _lib.ptr(y), M, d, hidden, _lib.ptr(res), _stream())
            return y.reshape(*lead, self.fc2.out_dim)
        if tc_enabled():
            p1, bn1, k1 = self.fc1.tc_pack()
            p2, bn2, k2 = self.fc2.tc_pack()
            ws = _lib.Workspace.get(_lib.load().sa_tc_mlp_workspace(M, hidden), slot=3)
            _lib.call("sa_tc_mlp", _lib.ptr(x2), _lib.ptr(p1), k1, bn1, _lib.ptr(p2), k2, bn2,
                      _lib.ptr(y), M, d, hidden, _lib.ptr(res), _lib.ptr(ws), ws.numel(), _stream())
            return y.reshape(*lead, self.fc2.out_dim)
        ws = _lib.Workspace.get(_lib.load().sa_mlp_workspace(M, hidden), slot=3)
        _lib.call("sa_mlp", _lib.ptr(x2), _lib.ptr(w1), k1, _lib.ptr(w2), k2, _lib.ptr(y), M, d,
                  hidden, p_min, _lib.ptr(res), _lib.ptr(ws), ws.numel(), _stream())
        return y.reshape(*lead, self.fc2.out_dim)

    def named_params(self, prefix):
        yield from self.fc1.named_params(prefix + ".fc1")
        yield from self.fc2.named_params(prefix + ".fc2")

    def extra_blobs(self, prefix):
        yield from self.fc1.extra_blobs(prefix + ".fc1")
        yield from self.fc2.extra_blobs(prefix + ".fc2")

    def post_step(self):
        self.fc1.post_step()
        self.fc2.post_step()


def fused_expert_forward(x, experts, plan: MOE.DispatchPlan, residual=None):
    """K5 for the two expert shapes the reference builds (ref model.py:499-502,
    514-521): (Linear, ShiftLinearLayer) and (Mlp(Linear, Linear),
    Mlp(Shift, Shift)). Returns None for any other expert set."""
    return _fused_expert_forward(x, experts, plan, residual)[0]


def _fused_expert_forward(x, experts, plan: MOE.DispatchPlan, residual=None, post_ln=None):
    """(y, post_ln applied): `post_ln` (a LayerNorm) is applied to the output
    in the same kernel when the fused MLP supports it (d = 32 / 64)."""
    if len(experts) != 2:
        return None, False
    e0, e1 = experts
    M = x.shape[0]
    res = residual.reshape(M, -1) if residual is not None else None
    if isinstance(e0, Linear) and isinstance(e1, ShiftLinearLayer):
        K, N = e0.in_dim, e0.out_dim
        if (e1.in_dim, e1.out_dim) != (K, N):
            return None, False
        y = torch.empty((M, N), dtype=torch.float32, device=x.device)
        if tc_enabled():
            pd, bn, _ = e0.tc_pack()
            ps, bn_s, _ = e1.tc_pack()
            assert bn == bn_s
            _lib.call("sa_tc_moe_linear", _lib.ptr(x), _lib.ptr(plan.perm_dev),
                      _lib.ptr(plan.counts_dev), _lib.ptr(plan.gate_dev), _lib.ptr(pd), _lib.ptr(ps),
                      bn, _lib.ptr(y), _lib.ptr(res), M, K, N, _stream())
            return y, False
        _lib.call("sa_moe_linear", _lib.ptr(x), _lib.ptr(plan.perm_dev), _lib.ptr(plan.counts_dev),
                  _lib.ptr(plan.gate_dev), _lib.ptr(e0.w.value), _lib.ptr(e1.quant.packed),
                  e1.quant.p_min, _lib.ptr(y), _lib.ptr(res), M, K, N, _stream())
        return y, False
    if (isinstance(e0, Mlp) and isinstance(e1, Mlp) and isinstance(e0.fc1, Linear)
            and isinstance(e0.fc2, Linear) and isinstance(e1.fc1, ShiftLinearLayer)
            and isinstance(e1.fc2, ShiftLinearLayer)):
        d, hidden = e0.fc1.in_dim, e0.fc1.out_dim
        if e1.fc1.quant.p_min != e1.fc2.quant.p_min:
            return None, False
        y = torch.empty((M, d), dtype=torch.float32, device=x.device)
        if fused_mlp_ok(d, hidden):
            p1d, _, _ = e0.fc1.tc_pack(fused_mlp_w1_bn(d))
            p2d, _, _ = e0.fc2.tc_pack(d)
            p1s, _, _ = e1.fc1.tc_pack(fused_mlp_w1_bn(d))
            p2s, _, _ = e1.fc2.tc_pack(d)
            if post_ln is not None and FUSE_STAGE_LN and (d == 32 or (d == 64 and FUSE_STAGE_LN64)):
                _lib.call("sa_tc_moe_mlp_fused_ln", _lib.ptr(x), _lib.ptr(plan.perm_dev),
                          _lib.ptr(plan.counts_dev), _lib.ptr(plan.gate_dev), _lib.ptr(p1d),
                          _lib.ptr(p2d), _lib.ptr(p1s), _lib.ptr(p2s), _lib.ptr(y), _lib.ptr(res),
                          M, d, hidden, _lib.ptr(post_ln.gain.value), _lib.ptr(post_ln.bias.value),
                          1e-5, _stream())
                return y, True
            _lib.call("sa_tc_moe_mlp_fused", _lib.ptr(x), _lib.ptr(plan.perm_dev),
                      _lib.ptr(plan.counts_dev), _lib.ptr(plan.gate_dev), _lib.ptr(p1d),
                      _lib.ptr(p2d), _lib.ptr(p1s), _lib.ptr(p2s), _lib.ptr(y), _lib.ptr(res),
                      M, d, hidden, _stream())
            return y, False
        if tc_enabled():
            p1d, bn1, _ = e0.fc1.tc_pack()
            p2d, bn2, _ = e0.fc2.tc_pack()
            p1s, _, _ = e1.fc1.tc_pack()
            p2s, _, _ = e1.fc2.tc_pack()
            ws = _lib.Workspace.get(_lib.load().sa_tc_mlp_workspace(M, hidden), slot=3)
            _lib.call("sa_tc_moe_mlp", _lib.ptr(x), _lib.ptr(plan.perm_dev),
                      _lib.ptr(plan.counts_dev), _lib.ptr(plan.gate_dev), _lib.ptr(p1d),
                      _lib.ptr(p2d), _lib.ptr(p1s), _lib.ptr(p2s), bn1, bn2, _lib.ptr(y),
                      _lib.ptr(res), M, d, hidden, _lib.ptr(ws), ws.numel(), _stream())
            return y, False
        ws = _lib.Workspace.get(_lib.load().sa_moe_mlp_workspace(M, hidden), slot=3)
        _lib.call("sa_moe_mlp", _lib.ptr(x), _lib.ptr(plan.perm_dev), _lib.ptr(plan.counts_dev),
                  _lib.ptr(plan.gate_dev), _lib.ptr(e0.fc1.w.value), _lib.ptr(e0.fc2.w.value),
                  _lib.ptr(e1.fc1.quant.packed), _lib.ptr(e1.fc2.quant.packed),
                  e1.fc1.quant.p_min, _lib.ptr(y), _lib.ptr(res), M, d, hidden, _lib.ptr(ws),
                  ws.numel(), _stream())
        return y, False
    return None, False


class MoeModule:
    """Top-1 two-expert mixture (ref model.py:230-314): device routing (K4) and
    one fused launch for both experts (K5). `last_plan` is set on every forward
    and materialises on the host only when read."""

    def __init__(self, w_g, experts: list, moe_cfg: MoeConfig):
        self.wg = GradPair(to_device(w_g))
        self.experts = experts
        self.cfg = moe_cfg
        self.alpha = MOE.latency_coefficients(moe_cfg.lat)
        self.last_plan: Optional[MOE.DispatchPlan] = None

    @property
    def kind(self):
        return "moe"

    @property
    def out_dim(self):
        e = self.experts[0]
        return e.fc2.out_dim if isinstance(e, Mlp) else e.out_dim

    def router(self) -> MOE.Router:
        return MOE.Router(w_g=self.wg.value, sigma=self.cfg.sigma, lam=self.cfg.lam)

    def forward(self, x, train=False, residual=None, plan=None, post_ln=None):
        """`plan` (optional) is a DispatchPlan already computed for x by a fused
        LayerNorm+router pass (Block.forward); otherwise routing runs here.
        `post_ln`: a LayerNorm the fused MLP may apply to the output in the same
        kernel; `self.post_ln_applied` says whether it did."""
        self.post_ln_applied = False
        _no_train(train)
        x = to_device(x)
        lead = x.shape[:-1]
        x2 = x.reshape(-1, x.shape[-1])
        if plan is None and residual is not None and _fused_o_ok(self, x2):
            # route + both experts + residual in one kernel (sa_fused_moe_linear)
            M, d = x2.shape
            expert_of = torch.empty(M, dtype=torch.int32, device=x2.device)
            gate = torch.empty(M, dtype=torch.float32, device=x2.device)
            y = torch.empty_like(x2)
            _lib.call("sa_fused_moe_linear", _lib.ptr(x2), _lib.ptr(self.wg.value),
                      _lib.ptr(self.experts[0].tc_pack(d)[0]), _lib.ptr(self.experts[1].tc_pack(d)[0]),
                      _lib.ptr(residual.reshape(M, d)), MOE.tie_threshold(), M, d,
                      _lib.ptr(expert_of), _lib.ptr(gate), _lib.ptr(y), _stream())
            self.last_plan = MOE.LazyDispatchPlan(expert_of, gate)
            return y.reshape(*lead, d)
        if plan is None:
            plan, _ = MOE.route_plan(x2, self.wg.value)
        self.last_plan = plan
        y, self.post_ln_applied = _fused_expert_forward(x2, self.experts, plan, residual, post_ln)
        if y is None:
            y = MOE.moe_forward(x2, self.experts, plan)
            if residual is not None:
                y = residual.reshape(y.shape) + y
        return y.reshape(*lead, y.shape[-1])

    def named_params(self, prefix):
        yield prefix + ".router.wg", self.wg
        for e, expert in enumerate(self.experts):
            yield from expert.named_params(f"{prefix}.expert{e}")

    def extra_blobs(self, prefix):
        for e, expert in enumerate(self.experts):
            yield from expert.extra_blobs(f"{prefix}.expert{e}")

    def post_step(self):
        for expert in self.experts:
            expert.post_step()


class AttentionLayer:
    """Multi-head attention over (batch, tokens, dim) (ref model.py:316-444)."""

    def __init__(self, block_cfg: BlockConfig, projections: dict, dw_kernels: Optional[GradPair]):
        self.cfg = block_cfg
        self.proj = projections
        self.dw = dw_kernels
        if self.dw is not None and not isinstance(self.dw.value, torch.Tensor):
            self.dw = GradPair(to_device(self.dw.value))

    @property
    def heads(self):
        return self.cfg.h

    def forward(self, x, train=False, residual=None, plans=None):
        _no_train(train)
        x = to_device(x)
        batch, n, d = x.shape
        flat = x.reshape(batch * n, d)
        if plans is None and self.cfg.attn_mode == "softmax" and self._dense_qkv_ok():
            # exempt MSA stage: one GEMM against [W_q | W_k | W_v], strided core
            y = self._qkv_cat_linear().forward(flat)
            merged = torch.empty_like(flat)
            _lib.call("sa_softmax_attn_strided", _lib.ptr(y), y.data_ptr() + 4 * d,
                      y.data_ptr() + 8 * d, 3 * d, _lib.ptr(merged), batch, n, d, self.heads,
                      _stream())
            res = residual.reshape(batch * n, d) if residual is not None else None
            return self.proj["o"].forward(merged, residual=res).reshape(batch, n, d)
        if plans is not None and self._grouped_qkv_ok(flat, plans):
            q, k, v = self._grouped_qkv(flat, plans)
        elif plans is not None:   # q/k/v routed by the fused LN1+router pass
            q = self.proj["q"].forward(flat, plan=plans[0])
            k = self.proj["k"].forward(flat, plan=plans[1])
            v = self.proj["v"].forward(flat, plan=plans[2])
        else:
            q = self.proj["q"].forward(flat)
            k = self.proj["k"].forward(flat)
            v = self.proj["v"].forward(flat)
        mode = self.cfg.attn_mode
        if mode == "softmax":
            merged = A.softmax_core_flat(q, k, v, batch, self.heads)
        elif mode == "linear-binary":
            dw = self.dw.value if self.dw is not None else None
            order = "linear" if self.cfg.binary_order == "auto" else self.cfg.binary_order
            merged = A.binary_core(q, k, v, batch, self.heads, dw, A.EPS_NORM, order)
        else:
            raise ValueError("the relu-feature 'linear' mode is outside the inference hot path")
        res = residual.reshape(batch * n, d) if residual is not None else None
        y = self.proj["o"].forward(merged, residual=res)
        return y.reshape(batch, n, d)

    def _dense_qkv_ok(self) -> bool:
        projs = [self.proj[k] for k in ("q", "k", "v")]
        return (FUSE_DENSE_QKV and tc_enabled() and all(type(p) is Linear for p in projs)
                and len({(p.in_dim, p.out_dim) for p in projs}) == 1)

    def _qkv_cat_linear(self):
        """[W_q | W_k | W_v] as one Linear (built once; column tiles of the
        concatenation are the separate projections' tiles, bit for bit)."""
        if getattr(self, "_qkv_cat", None) is None:
            w = torch.cat([self.proj[k].w.value for k in ("q", "k", "v")], dim=1).contiguous()
            self._qkv_cat = Linear(w)
        return self._qkv_cat

    def _grouped_qkv_ok(self, flat, plans) -> bool:
        """One grouped launch for q/k/v: tensor-core path, (Linear, Shift) experts
        of one shape, and plans stacked in one device buffer (sa_ln_route)."""
        if not (FUSE_GROUPED_QKV and tc_enabled() and len(plans) == 3):
            return False
        projs = [self.proj[k] for k in ("q", "k", "v")]
        if not all(isinstance(p, MoeModule) and _dual_expert_linear(p) for p in projs):
            return False
        M = flat.shape[0]
        for attr, stride in (("perm_dev", M * 4), ("gate_dev", M * 4), ("counts_dev", 8)):
            base = getattr(plans[0], attr)
            if base is None or not base.is_contiguous():
                return False
            for r in (1, 2):
                t = getattr(plans[r], attr)
                if t is None or t.data_ptr() != base.data_ptr() + r * stride:
                    return False
        return True

    def _grouped_qkv(self, flat, plans):
        """sa_tc_moe_linear_grouped: the three MoE projections in one launch."""
        import ctypes
        M, d = flat.shape
        projs = [self.proj[k] for k in ("q", "k", "v")]
        N = projs[0].experts[0].out_dim
        y = torch.empty((3, M, N), dtype=torch.float32, device=flat.device)
        dense = (ctypes.c_void_p * 3)(*[_lib.ptr(p.experts[0].tc_pack()[0]) for p in projs])
        shift = (ctypes.c_void_p * 3)(*[_lib.ptr(p.experts[1].tc_pack()[0]) for p in projs])
        bn = projs[0].experts[0].tc_pack()[1]
        _lib.call("sa_tc_moe_linear_grouped", _lib.ptr(flat), _lib.ptr(plans[0].perm_dev),
                  _lib.ptr(plans[0].counts_dev), _lib.ptr(plans[0].gate_dev),
                  ctypes.addressof(dense), ctypes.addressof(shift), 3, bn, _lib.ptr(y), M, d, N,
                  _stream())
        for p, plan in zip(projs, plans):
            p.last_plan = plan
        return y[0], y[1], y[2]

    def named_params(self, prefix):
        for key in ("q", "k", "v", "o"):
            yield from self.proj[key].named_params(f"{prefix}.{key}")
        if self.dw is not None:
            yield prefix + ".dw", self.dw

    def extra_blobs(self, prefix):
        for key in ("q", "k", "v", "o"):
            yield from self.proj[key].extra_blobs(f"{prefix}.{key}")

    def post_step(self):
        for key in ("q", "k", "v", "o"):
            self.proj[key].post_step()
        self._qkv_cat = None   # weights may have changed


class Block:
    """Pre-norm residual block (ref model.py:446-480); both residual adds are
    fused into the epilogues of W_O and fc2."""

    def __init__(self, cfg: BlockConfig, attn: AttentionLayer, mlp, dtype=np.float32):
        self.cfg = cfg
        self.ln1 = LayerNorm(cfg.d, dtype)
        self.ln2 = LayerNorm(cfg.d, dtype)
        self.attn = attn
        self.mlp = mlp

    def forward(self, x, train=False, post_ln=None):
        """`post_ln`: the stage's final LayerNorm, applied to this block's output
        inside the MLP kernel when it supports it (`self.post_ln_applied`)."""
        _no_train(train)
        self.post_ln_applied = False
        x = to_device(x)
        batch, n, d = x.shape
        x2 = x.reshape(batch * n, d)
        fuse = FUSE_LN_ROUTE and d % 32 == 0 and d <= 256
        qkv = [self.attn.proj[k] for k in ("q", "k", "v")]
        pre = None   # (LN2(h), MLP plan) from the W_O epilogue
        if self._fused_qkv_ok(d, n, qkv):
            h, pre = self._fused_attention(x2, batch, n, d, qkv)
            h = h.reshape(batch, n, d)
        elif fuse and all(isinstance(p, MoeModule) for p in qkv):
            y, plans = MOE.ln_route_plans(x2, self.ln1.gain.value, self.ln1.bias.value,
                                          [p.wg.value for p in qkv])
            h = self.attn.forward(y.reshape(batch, n, d), residual=x, plans=plans)
        else:
            h = self.attn.forward(self.ln1.forward(x), residual=x)
        h2 = h.reshape(batch * n, d)
        if pre is not None:
            y = self.mlp.forward(pre[0], residual=h2, plan=pre[1], post_ln=post_ln)
            self.post_ln_applied = self.mlp.post_ln_applied
        elif fuse and isinstance(self.mlp, MoeModule):
            flat, (plan,) = MOE.ln_route_plans(h2, self.ln2.gain.value, self.ln2.bias.value,
                                               [self.mlp.wg.value])
            y = self.mlp.forward(flat, residual=h2, plan=plan, post_ln=post_ln)
            self.post_ln_applied = self.mlp.post_ln_applied
        else:
            flat = self.ln2.forward(h).reshape(batch * n, d)
            y = self.mlp.forward(flat, residual=h2)
        return y.reshape(batch, n, d)

    def _fused_qkv_ok(self, d, n, qkv) -> bool:
        cfg = self.cfg
        return (FUSE_QKV and tc_enabled() and cfg.attn_mode == "linear-binary"
                and cfg.binary_order in ("auto", "linear") and d == 32 * cfg.h
                and all(_dual_expert_linear(p) for p in qkv)
                and bool(_lib.load().sa_ln_qkv_hash_ok(d, n)))

    def _fused_attention(self, x2, batch, n, d, qkv):
        """sa_ln_qkv_hash (LN1 + routers + q/k/v + sign-hash) → binary core →
        W_O with the residual; the q/k/v plans are set lazily (their stable
        partitions are only computed if read)."""
        M = batch * n
        H = self.cfg.h
        dev = x2.device
        expert_of = torch.empty((3, M), dtype=torch.int32, device=dev)
        gate = torch.empty((3, M), dtype=torch.float32, device=dev)
        cq = torch.empty((batch, H, n, 1), dtype=torch.int32, device=dev)
        ck = torch.empty_like(cq)
        gq = torch.empty((batch, H), dtype=torch.float32, device=dev)
        gk = torch.empty_like(gq)
        v = torch.empty((M, d), dtype=torch.float32, device=dev)
        ws = _lib.Workspace.get(_lib.load().sa_ln_qkv_hash_workspace(batch, n, d), slot=4)
        packs = []
        for proj in qkv:
            packs.append(_lib.ptr(proj.experts[0].tc_pack(d)[0]))
            packs.append(_lib.ptr(proj.experts[1].tc_pack(d)[0]))
        _lib.call("sa_ln_qkv_hash", _lib.ptr(x2), _lib.ptr(self.ln1.gain.value),
                  _lib.ptr(self.ln1.bias.value), 1e-5, *[_lib.ptr(p.wg.value) for p in qkv], *packs,
                  MOE.tie_threshold(), batch, n, d, _lib.ptr(expert_of), _lib.ptr(gate),
                  _lib.ptr(cq), _lib.ptr(ck), _lib.ptr(gq), _lib.ptr(gk), _lib.ptr(v),
                  _lib.ptr(ws), ws.numel(), _stream())
        for r, proj in enumerate(qkv):
            proj.last_plan = MOE.LazyDispatchPlan(expert_of[r], gate[r])
        dw = self.attn.dw.value if self.attn.dw is not None else None
        merged = A.binary_core_codes(cq, ck, gq, gk, v, batch, H, dw, A.EPS_NORM, "linear")
        o = self.attn.proj["o"]
        if FUSE_LN2 and FUSE_LN_ROUTE and isinstance(self.mlp, MoeModule) and _fused_o_ok(o, merged):
            # W_O + residual, then LN2 and the MLP router on the result, in one kernel
            expert_of = torch.empty(M, dtype=torch.int32, device=dev)
            gate_o = torch.empty(M, dtype=torch.float32, device=dev)
            h = torch.empty_like(x2)
            y2 = torch.empty_like(x2)
            expert_of2 = torch.empty(M, dtype=torch.int32, device=dev)
            gate2 = torch.empty(M, dtype=torch.float32, device=dev)
            _lib.call("sa_fused_moe_linear_ln_route", _lib.ptr(merged), _lib.ptr(o.wg.value),
                      _lib.ptr(o.experts[0].tc_pack(d)[0]), _lib.ptr(o.experts[1].tc_pack(d)[0]),
                      _lib.ptr(x2), MOE.tie_threshold(), M, d, _lib.ptr(expert_of),
                      _lib.ptr(gate_o), _lib.ptr(h), _lib.ptr(self.ln2.gain.value),
                      _lib.ptr(self.ln2.bias.value), 1e-5, _lib.ptr(self.mlp.wg.value),
                      _lib.ptr(y2), _lib.ptr(expert_of2), _lib.ptr(gate2), _stream())
            o.last_plan = MOE.LazyDispatchPlan(expert_of, gate_o)
            return h, (y2, MOE.LazyDispatchPlan(expert_of2, gate2))
        return o.forward(merged, residual=x2), None

    def named_params(self, prefix):
        yield from self.ln1.named_params(prefix + ".ln1")
        yield from self.attn.named_params(prefix + ".attn")
        yield from self.ln2.named_params(prefix + ".ln2")
        yield from self.mlp.named_params(prefix + ".mlp")

    def extra_blobs(self, prefix):
        yield from self.attn.extra_blobs(prefix + ".attn")
        yield from self.mlp.extra_blobs(prefix + ".mlp")

    def post_step(self):
        self.attn.post_step()
        self.mlp.post_step()


# ---------------------------------------------------------------------------
# builders (draw order = ref model.py:487-522)


def _init_linear(rng, fan_in, fan_out, dtype=np.float32, scale=None):
    """N(0,1)·scale, default 1/√fan_in (ref model.py:487-489). Host numpy."""
    scale = scale if scale is not None else 1.0 / np.sqrt(fan_in)
    return (rng.standard_normal((fan_in, fan_out)) * scale).astype(dtype)


def _make_linear(mode, rng, fan_in, fan_out, dtype, moe_cfg, quant_cfg):
    """ref model.py:492-503"""
    w = _init_linear(rng, fan_in, fan_out, dtype)
    if mode == "dense":
        return Linear(w)
    if mode == "shift":
        return ShiftLinearLayer(w, quant_cfg)
    if mode == "moe":
        wg = _init_linear(rng, fan_in, 2, dtype, scale=0.02)
        return MoeModule(wg, [Linear(w), ShiftLinearLayer(w.copy(), quant_cfg)], moe_cfg)
    raise ValueError(f"unknown linear mode {mode!r}")


def _make_mlp(cfg: BlockConfig, rng, dtype, moe_cfg, quant_cfg):
    """ref model.py:506-522 (moe: router drawn before w1, w2)."""
    hidden = int(cfg.d * cfg.mlp_ratio)
    if cfg.mlp_mode == "dense":
        return Mlp(Linear(_init_linear(rng, cfg.d, hidden, dtype)),
                   Linear(_init_linear(rng, hidden, cfg.d, dtype)))
    if cfg.mlp_mode == "shift":
        return Mlp(ShiftLinearLayer(_init_linear(rng, cfg.d, hidden, dtype), quant_cfg),
                   ShiftLinearLayer(_init_linear(rng, hidden, cfg.d, dtype), quant_cfg))
    if cfg.mlp_mode == "moe":
        wg = _init_linear(rng, cfg.d, 2, dtype, scale=0.02)
        w1 = _init_linear(rng, cfg.d, hidden, dtype)
        w2 = _init_linear(rng, hidden, cfg.d, dtype)
        return MoeModule(wg, [Mlp(Linear(w1), Linear(w2)),
                              Mlp(ShiftLinearLayer(w1.copy(), quant_cfg),
                                  ShiftLinearLayer(w2.copy(), quant_cfg))], moe_cfg)
    raise ValueError(f"unknown mlp_mode {cfg.mlp_mode!r}")


class Stage:
    """Patch embedding (+cls, +pos, +LN) → blocks → optional stage LN."""

    def __init__(self, spec_stage, c_in, n_tokens, rng, dtype, moe_cfg, quant_cfg, dw_init):
        st = spec_stage
        self.patch = st["patch"]
        self.d = d = st["d"]
        self.n = n_tokens
        self.patch_embed = Linear(_init_linear(rng, self.patch * self.patch * c_in, d, dtype))
        self.cls = None
        self.pos = None
        rows = n_tokens + (1 if st.get("cls_token") else 0)
        if st.get("cls_token"):
            self.cls = GradPair(to_device((rng.standard_normal((1, d)) * 0.02).astype(dtype)))
        if st.get("pos"):
            self.pos = GradPair(to_device((rng.standard_normal((rows, d)) * 0.02).astype(dtype)))
        self.rows = rows
        self.blocks = []
        for bc in st["blocks"]:
            cfg = BlockConfig(d=d, h=bc["h"], mlp_ratio=bc["mlp_ratio"], attn_mode=bc["attn_mode"],
                              mlp_mode=bc["mlp_mode"], attn_linear_mode=bc["attn_linear_mode"],
                              exempt=bc.get("exempt", False),
                              binary_order=bc.get("binary_order", "auto"))
            proj = {k: _make_linear(cfg.attn_linear_mode, rng, d, d, dtype, moe_cfg, quant_cfg)
                    for k in ("q", "k", "v", "o")}
            dw = None
            if cfg.attn_mode != "softmax":
                if isinstance(dw_init, (int, float)):
                    dw = GradPair(to_device((rng.standard_normal((3, 3, d)) * float(dw_init))
                                            .astype(dtype)))
                else:
                    dw = GradPair(to_device(np.zeros((3, 3, d), dtype)))
            mlp = _make_mlp(cfg, rng, dtype, moe_cfg, quant_cfg)
            self.blocks.append(Block(cfg, AttentionLayer(cfg, proj, dw), mlp, dtype))
        self.embed_ln = LayerNorm(d, dtype) if st.get("embed_norm") else None
        self.stage_ln = LayerNorm(d, dtype) if st.get("stage_norm") else None


class Network:
    """A ShiftAddViT built from an architecture spec (see specs.py): the
    reference toy `Model` (one stage) or a PVT / DeiT composition (several
    stages chained through their token grids). `forward(images NHWC) →
    logits (B, classes)` like `Model.forward` (ref model.py:565-577)."""

    def __init__(self, spec: dict, dtype=np.float32, moe_cfg: MoeConfig = None,
                 quant_cfg: Q.QuantConfig = None):
        self.spec = spec
        self.dtype = dtype
        self.moe_cfg = moe_cfg or MoeConfig()
        self.quant_cfg = quant_cfg or Q.QuantConfig(p_min=spec.get("p_min", -15),
                                                    p_max=spec.get("p_max", 15))
        rng = make_rng(spec["seed"])
        c_in = spec.get("channels", 3)
        side = spec["img"]
        self.stages = []
        for st in spec["stages"]:
            if side % st["patch"]:
                raise ShapeError(f"side {side} not divisible by patch {st['patch']}")
            side //= st["patch"]
            self.stages.append(Stage(st, c_in, side * side, rng, dtype, self.moe_cfg,
                                     self.quant_cfg, spec.get("dw_init", "zeros")))
            c_in = st["d"]
        self.head = Linear(_init_linear(rng, spec["stages"][-1]["d"], spec["classes"], dtype,
                                        scale=0.01))
        dwi = spec.get("dw_init", "zeros")
        if isinstance(dwi, dict):   # side stream after all main draws (specs.toy_c1)
            g2 = make_rng(dwi["seed"])
            for S in self.stages:
                for blk in S.blocks:
                    if blk.attn.dw is not None:
                        vals = (g2.standard_normal(tuple(blk.attn.dw.value.shape)) * dwi["std"])
                        blk.attn.dw.value.copy_(torch.from_numpy(vals.astype(dtype)))
        self.pool_mode = 1 if spec.get("pool", "mean") == "cls" else 0

    # -- introspection ---------------------------------------------------
    @property
    def blocks(self):
        return [b for S in self.stages for b in S.blocks]

    def moe_modules(self):
        for si, S in enumerate(self.stages):
            for bi, blk in enumerate(S.blocks):
                pre = f"s{si}.b{bi}"
                for key in ("q", "k", "v", "o"):
                    if isinstance(blk.attn.proj[key], MoeModule):
                        yield f"{pre}.attn.{key}", blk.attn.proj[key]
                if isinstance(blk.mlp, MoeModule):
                    yield f"{pre}.mlp", blk.mlp

    def named_params(self):
        """(name, GradPair) of every parameter (ref Model.named_params,
        model.py:592-598, generalised to several stages: prefix s<i>.)."""
        for si, S in enumerate(self.stages):
            pre = f"s{si}"
            yield f"{pre}.patch_embed.w", S.patch_embed.w
            if S.cls is not None:
                yield f"{pre}.cls", S.cls
            if S.pos is not None:
                yield f"{pre}.pos", S.pos
            if S.embed_ln is not None:
                yield from S.embed_ln.named_params(f"{pre}.embed_ln")
            for bi, blk in enumerate(S.blocks):
                yield from blk.named_params(f"{pre}.block{bi}")
            if S.stage_ln is not None:
                yield from S.stage_ln.named_params(f"{pre}.final_ln")
        yield "head.w", self.head.w

    def extra_blobs(self):
        """Shift-layer sign / exponent blobs (ref model.py:600-602)."""
        for si, S in enumerate(self.stages):
            for bi, blk in enumerate(S.blocks):
                yield from blk.extra_blobs(f"s{si}.block{bi}")

    def post_step(self):
        """Re-derive every layer's device state from its (re)loaded values:
        shift codes from the shadows, packed tensor-core planes (ref
        model.py:604-606)."""
        for S in self.stages:
            S.patch_embed.post_step()
            for blk in S.blocks:
                blk.post_step()
        self.head.post_step()

    def named_weights(self):
        """(name, device tensor) in oracle.nets.iter_weights order."""
        for si, S in enumerate(self.stages):
            yield f"s{si}.pe", S.patch_embed.w.value
            if S.cls is not None:
                yield f"s{si}.cls", S.cls.value
            if S.pos is not None:
                yield f"s{si}.pos", S.pos.value
            for bi, blk in enumerate(S.blocks):
                pre = f"s{si}.b{bi}"
                for key in ("q", "k", "v", "o"):
                    yield from _layer_weights(f"{pre}.attn.{key}", blk.attn.proj[key])
                if blk.attn.dw is not None:
                    yield f"{pre}.attn.dw", blk.attn.dw.value
                yield from _layer_weights(f"{pre}.mlp", blk.mlp)
        yield "head", self.head.w.value

    # -- forward -----------------------------------------------------------
    def forward(self, images, train=False) -> torch.Tensor:
        _no_train(train)
        x = to_device(images)
        if x.ndim != 4:
            raise ShapeError(f"images must be (B, H, W, C), got {tuple(x.shape)}")
        B, H, W, C = x.shape
        grid = x
        sub = 0.5                                   # ref model.py:566
        tok = None
        for S in self.stages:
            tok = torch.empty((B * S.rows, S.d), dtype=torch.float32, device=x.device)
            fused_ln = False
            if tc_enabled():
                pk, bn, _ = S.patch_embed.tc_pack()
                fused_ln = (FUSE_EMBED_LN and S.embed_ln is not None and bool(
                    _lib.load().sa_tc_patch_embed_ln_ok(S.d, S.cls is not None, S.pos is not None)))
                if fused_ln:   # embed + LayerNorm in one kernel (LN in the GEMM epilogue)
                    _lib.call("sa_tc_patch_embed_ln", _lib.ptr(grid), B, H, W, C, S.patch, sub,
                              _lib.ptr(pk), bn, S.d, _lib.ptr(S.embed_ln.gain.value),
                              _lib.ptr(S.embed_ln.bias.value), 1e-5, _lib.ptr(tok),
                              _stream())
                else:
                    _lib.call("sa_tc_patch_embed", _lib.ptr(grid), B, H, W, C, S.patch, sub,
                              _lib.ptr(pk), bn, S.d,
                              _lib.ptr(S.cls.value if S.cls is not None else None),
                              _lib.ptr(S.pos.value if S.pos is not None else None), _lib.ptr(tok),
                              _stream())
            else:
                _lib.call("sa_patch_embed", _lib.ptr(grid), B, H, W, C, S.patch, sub,
                          _lib.ptr(S.patch_embed.w.value), S.d,
                          _lib.ptr(S.cls.value if S.cls is not None else None),
                          _lib.ptr(S.pos.value if S.pos is not None else None), _lib.ptr(tok),
                          _stream())
            if S.embed_ln is not None and not fused_ln:
                tok = S.embed_ln.forward(tok)
            t3 = tok.reshape(B, S.rows, S.d)
            for i, blk in enumerate(S.blocks):
                last = i == len(S.blocks) - 1
                t3 = blk.forward(t3, post_ln=S.stage_ln if last else None)
            tok = t3.reshape(B * S.rows, S.d)
            if S.stage_ln is not None and not (S.blocks and S.blocks[-1].post_ln_applied):
                tok = S.stage_ln.forward(tok)
            side = H // S.patch
            grid, H, W, C, sub = tok, side, side, S.d, 0.0
        last = self.stages[-1]
        pooled = torch.empty((B, last.d), dtype=torch.float32, device=x.device)
        _lib.call("sa_pool", _lib.ptr(tok), _lib.ptr(pooled), B, last.rows, last.d,
                  self.pool_mode, _stream())
        return self.head.forward(pooled)

    __call__ = forward


def _layer_weights(name, L):
    if isinstance(L, (Linear, ShiftLinearLayer)):
        yield name + ".w", L.w.value
    elif isinstance(L, Mlp):
        yield from _layer_weights(name + ".fc1", L.fc1)
        yield from _layer_weights(name + ".fc2", L.fc2)
    else:
        yield name + ".wg", L.wg.value
        for e, ex in enumerate(L.experts):
            yield from _layer_weights(f"{name}.expert{e}", ex)


def _model_cfg_to_spec(cfg: ModelConfig, quant_cfg) -> dict:
    d0 = cfg.blocks[0].d
    if any(b.d != d0 for b in cfg.blocks):
        raise ShapeError("all blocks of the toy Model share one width")
    qc = quant_cfg or Q.QuantConfig()
    return {"name": "Model", "img": cfg.img, "channels": cfg.channels, "classes": cfg.classes,
            "seed": cfg.seed, "dw_init": "zeros", "pool": "mean", "p_min": qc.p_min,
            "p_max": qc.p_max,
            "stages": [{"patch": cfg.patch, "d": d0, "pos": True, "cls_token": False,
                        "embed_norm": False, "stage_norm": True,
                        "blocks": [dict(h=b.h, mlp_ratio=b.mlp_ratio, attn_mode=b.attn_mode,
                                        mlp_mode=b.mlp_mode, attn_linear_mode=b.attn_linear_mode,
                                        exempt=b.exempt, binary_order=b.binary_order)
                                   for b in cfg.blocks]}]}


class Model(Network):
    """The reference toy ViT (ref model.py:525-577): patch embed, learned
    positions, blocks, final LN, mean pool, head — same constructor and the
    same PCG64 parameters as the reference `Model(cfg)`."""

    def __init__(self, cfg: ModelConfig, dtype=np.float32, moe_cfg: MoeConfig = None,
                 quant_cfg: Q.QuantConfig = None):
        self.cfg = cfg
        super().__init__(_model_cfg_to_spec(cfg, quant_cfg), dtype, moe_cfg, quant_cfg)

    def named_params(self):
        """The reference Model's parameter names (ref model.py:592-598)."""
        S = self.stages[0]
        yield "patch_embed.w", S.patch_embed.w
        yield "pos", S.pos
        for i, blk in enumerate(S.blocks):
            yield from blk.named_params(f"block{i}")
        yield from S.stage_ln.named_params("final_ln")
        yield "head.w", self.head.w

    def extra_blobs(self):
        for i, blk in enumerate(self.stages[0].blocks):
            yield from blk.extra_blobs(f"block{i}")

    def moe_modules(self):
        """ref model.py:608-615 (names and order)."""
        for i, blk in enumerate(self.stages[0].blocks):
            if isinstance(blk.mlp, MoeModule):
                yield f"block{i}.mlp", blk.mlp
            for key in ("q", "k", "v", "o"):
                if isinstance(blk.attn.proj[key], MoeModule):
                    yield f"block{i}.attn.{key}", blk.attn.proj[key]

    @property
    def patch_embed(self):
        return self.stages[0].patch_embed

    @property
    def pos(self):
        return self.stages[0].pos

    @property
    def final_ln(self):
        return self.stages[0].stage_ln


@dataclass
class EvalResult:
    """ref model.py:738-742"""

    accuracy: float
    expert_shares: dict
    dispatch_maps: dict        # layer -> (N, tokens) winning expert per token


def evaluate(model: Network, dataset, batch_size: int = 64) -> EvalResult:
    """Accuracy, per-layer expert shares and dispatch maps over a dataset
    (anything with `.images` (N, H, W, C) and `.labels` (N,)) (ref
    model.py:745-765): the forward runs on the device batch by batch; each MoE
    layer's winning experts come from its last DispatchPlan (one D2H copy per
    layer and batch)."""
    images, labels = dataset.images, np.asarray(dataset.labels)
    n = labels.shape[0]
    correct = 0
    names = [name for name, _ in model.moe_modules()]
    maps = {name: [] for name in names}
    for start in range(0, n, batch_size):
        batch = images[start:start + batch_size]
        logits = model.forward(batch).cpu().numpy()
        correct += int((np.argmax(logits, axis=1) == labels[start:start + batch_size]).sum())
        b = logits.shape[0]
        for name, module in model.moe_modules():
            maps[name].append(module.last_plan.expert_of.reshape(b, -1))
    dispatch_maps = {name: np.concatenate(chunks, axis=0) for name, chunks in maps.items() if chunks}
    shares = {}
    for name, arr in dispatch_maps.items():
        counts = np.bincount(arr.ravel(), minlength=2).astype(np.float64)
        shares[name] = (counts / counts.sum()).tolist()
    return EvalResult(accuracy=correct / n, expert_shares=shares, dispatch_maps=dispatch_maps)


def write_dispatch_map(result: EvalResult, layer: str, out_dir) -> str:
    """The reference's dispatch-map export (ref cli.py:233-265,
    docs/formats.md "dispatch_<layer>.csv"): one row per image, `image,
    token0..tokenN-1` with the winning expert (0 = mult, 1 = shift), plus
    dispatch_summary.json with the aggregate shares. Returns the CSV path."""
    import csv
    import json
    if layer not in result.dispatch_maps:
        raise KeyError(f"no MoE layer named {layer!r}; available: {sorted(result.dispatch_maps)}")
    dmap = result.dispatch_maps[layer]
    os.makedirs(out_dir, exist_ok=True)
    grid_csv = os.path.join(out_dir, f"dispatch_{layer.replace('.', '_')}.csv")
    with open(grid_csv, "w", newline="") as fh:
        writer = csv.writer(fh)
        writer.writerow(["image"] + [f"token{t}" for t in range(dmap.shape[1])])
        for i in range(dmap.shape[0]):
            writer.writerow([i] + dmap[i].tolist())
    summary = {"layer": layer, "expert_shares": result.expert_shares,
               "tokens_per_image": int(dmap.shape[1]), "images": int(dmap.shape[0]),
               "accuracy": result.accuracy}
    with open(os.path.join(out_dir, "dispatch_summary.json"), "w") as fh:
        fh.write(json.dumps(summary, indent=2, sort_keys=True) + "\n")
    return grid_csv


def build_model(spec: dict, **kw) -> Network:
    return Network(spec, **kw)


def pvt_v2_b0(**kw) -> Network:
    return Network(SPECS.pvt_v2_b0(**kw))


def pvt_v2_b2(**kw) -> Network:
    return Network(SPECS.pvt_v2_b2(**kw))


def pvt_v1_tiny(**kw) -> Network:
    return Network(SPECS.pvt_v1_tiny(**kw))


def deit_tiny(**kw) -> Network:
    return Network(SPECS.deit_tiny(**kw))


def apply_stage(model: Network, stage: int, mlp_target: str = "shift",
                attn_target: str = "shift", reparam_seed: int = 77) -> Network:
    """Stage-1/2 conversion (ref model.py:897-930): stage 1 switches non-exempt
    attention to linear-binary (zero DW kernels if absent); stage 2 converts
    projections / MLPs to shift or moe, preserving weights, with routers drawn
    from PCG64(reparam_seed) in the reference's order."""
    if stage not in (1, 2):
        raise ValueError(f"stage must be 1 or 2, got {stage}")
    rng = make_rng(reparam_seed)
    blocks = model.blocks
    if stage == 2 and any(b.cfg.attn_mode == "softmax" and not b.cfg.exempt for b in blocks):
        raise ValueError("stage 2 requires a stage-1 model (linear attention)")
    for block in blocks:
        if block.cfg.exempt:
            continue
        if stage == 1:
            block.cfg.attn_mode = "linear-binary"
            block.attn.cfg = block.cfg
            if block.attn.dw is None:
                block.attn.dw = GradPair(to_device(np.zeros((3, 3, block.cfg.d), np.float32)))
        else:
            block.cfg.attn_linear_mode = attn_target
            block.cfg.mlp_mode = mlp_target
            block.attn.cfg = block.cfg
            for key in ("q", "k", "v", "o"):
                block.attn.proj[key] = _convert_linear(block.attn.proj[key], attn_target, rng,
                                                       model.moe_cfg, model.quant_cfg)
            block.mlp = _convert_mlp(block.mlp, mlp_target, rng, model.moe_cfg, model.quant_cfg)
    return model


def _convert_linear(layer, target, rng, moe_cfg, quant_cfg):
    """ref model.py:772-783"""
    if isinstance(layer, MoeModule) or target == "dense":
        return layer
    w = layer.w.value.clone()
    if target == "shift":
        return ShiftLinearLayer(w, quant_cfg)
    if target == "moe":
        wg = (rng.standard_normal((w.shape[0], 2)) * 0.02).astype(np.float32)
        return MoeModule(wg, [Linear(w.clone()), ShiftLinearLayer(w.clone(), quant_cfg)], moe_cfg)
    raise ValueError(f"unknown conversion target {target!r}")


def _convert_mlp(mlp, target, rng, moe_cfg, quant_cfg):
    """ref model.py:786-799"""
    if isinstance(mlp, MoeModule) or target == "dense":
        return mlp
    w1 = mlp.fc1.w.value.clone()
    w2 = mlp.fc2.w.value.clone()
    if target == "shift":
        return Mlp(ShiftLinearLayer(w1, quant_cfg), ShiftLinearLayer(w2, quant_cfg))
    if target == "moe":
        wg = (rng.standard_normal((w1.shape[0], 2)) * 0.02).astype(np.float32)
        return MoeModule(wg, [Mlp(Linear(w1.clone()), Linear(w2.clone())),
                              Mlp(ShiftLinearLayer(w1.clone(), quant_cfg),
                                  ShiftLinearLayer(w2.clone(), quant_cfg))], moe_cfg)
    raise ValueError(f"unknown conversion target {target!r}")


__all__ = ["BlockConfig", "ModelConfig", "MoeConfig", "Linear", "ShiftLinearLayer", "LayerNorm",
           "Mlp", "MoeModule", "AttentionLayer", "Block", "Network", "Model", "build_model",
           "pvt_v2_b0", "pvt_v2_b2", "pvt_v1_tiny", "deit_tiny", "apply_stage", "StateError"]
