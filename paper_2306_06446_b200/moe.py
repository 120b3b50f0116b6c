"""Top-1 two-expert routing on the device, mirroring the reference
`shiftadd.moe` module (ref moe.py) for inference.

Routing semantics are bit-exact with the reference (K4): logits are float32
roundings of fp64 dot products, the winner is argmax of the float32 softmax
with ties to expert 0 — for two experts that is the logit argmax except inside
numpy's exp tie band, whose width is measured on this host at import
(`tie_threshold`) — and the dispatch plan is the stable partition of tokens.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from . import _lib
from .tensor import ShapeError, to_device


def numpy_exp_tie_threshold() -> np.float32:
    """Largest float32 d >= 0 with numpy's float32 exp(-d) == 1 on this host
    (4.1063238e-08 with numpy 2.3 / AVX512). For two experts
    the reference's argmax(p) (ref moe.py:89) picks expert 0 on a logit deficit
    δ > 0 exactly when exp(-δ) rounds to 1 (p0 == p1)."""
    lo, hi = 0, int(np.float32(1e-6).view(np.uint32))
    while lo < hi:
        mid = (lo + hi + 1) // 2
        d = np.array([mid], np.uint32).view(np.float32)
        if np.exp(-d)[0] == np.float32(1.0):
            lo = mid
        else:
            hi = mid - 1
    return np.array([lo], np.uint32).view(np.float32)[0]


_TIE = None


def tie_threshold() -> float:
    global _TIE
    if _TIE is None:
        _TIE = float(numpy_exp_tie_threshold())
    return _TIE


@dataclass
class Router:
    """ref moe.py:45-61"""

    w_g: torch.Tensor            # (d, num_experts)
    sigma: float = 0.1
    lam: float = 0.01

    def __post_init__(self):
        self.w_g = to_device(self.w_g)
        if self.w_g.ndim != 2 or self.w_g.shape[1] < 2:
            raise ShapeError(f"router needs a (d, E>=2) gating matrix, got {tuple(self.w_g.shape)}")
        if self.sigma <= 0:
            raise ValueError("sigma must be positive")
        if self.lam < 0:
            raise ValueError("lambda must be nonnegative")

    @property
    def num_experts(self) -> int:
        return self.w_g.shape[1]


# Bumped by runtime.GraphedForward on every replay: a replay rewrites the
# device buffers of the plans created at capture time, so host copies pulled
# before it (and partitions built outside the graph) are stale.
_generation = [0]


def bump_generation():
    _generation[0] += 1


class DispatchPlan:
    """Winning expert, gate and per-expert token lists (ref moe.py:64-71).

    Kept on the device as expert_of / gate / counts / perm; the reference's
    numpy views (`expert_of`, `gate_of`, `index_of`) are materialised lazily on
    first access (one D2H copy), so the forward never syncs the host."""

    def __init__(self, expert_of_dev, gate_dev, counts_dev, perm_dev):
        self.expert_of_dev = expert_of_dev
        self.gate_dev = gate_dev
        self.counts_dev = counts_dev
        self.perm_dev = perm_dev
        self._host = None
        self._host_gen = -1

    def _pull(self):
        if self._host is None or self._host_gen != _generation[0]:
            self._host_gen = _generation[0]
            e = self.expert_of_dev.cpu().numpy().astype(np.int64)
            g = self.gate_dev.cpu().numpy()
            c = self.counts_dev.cpu().numpy()
            p = self.perm_dev.cpu().numpy().astype(np.int64)
            self._host = (e, g, [p[: c[0]], p[c[0]: c[0] + c[1]]])
        return self._host

    @property
    def expert_of(self) -> np.ndarray:
        return self._pull()[0]

    @property
    def gate_of(self) -> np.ndarray:
        return self._pull()[1]

    @property
    def index_of(self) -> list:
        return self._pull()[2]

    def share(self, expert: int) -> float:
        e = self.expert_of
        return float(self.index_of[expert].size) / max(e.size, 1)


class LazyDispatchPlan(DispatchPlan):
    """A plan whose winners / gates were produced on the device by a fused
    kernel (sa_ln_qkv_hash); the stable partition (counts, perm) is computed
    by sa_moe_partition on first use, on the then-current stream."""

    def __init__(self, expert_of_dev, gate_dev):
        self._in_graph = False
        self._part_gen = -1
        super().__init__(expert_of_dev, gate_dev, None, None)

    def _partition(self):
        # a partition enqueued while a graph was being captured is re-run by
        # every replay; one built outside a graph is rebuilt after a replay
        stale = not self._in_graph and self._part_gen != _generation[0]
        if self._counts is None or stale:
            self._in_graph = torch.cuda.is_current_stream_capturing()
            self._part_gen = _generation[0]
            M = self.expert_of_dev.shape[0]
            dev = self.expert_of_dev.device
            counts = torch.empty(2, dtype=torch.int32, device=dev)
            perm = torch.empty(M, dtype=torch.int32, device=dev)
            nbytes = int(_lib.load().sa_moe_partition_workspace(M))
            ws = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=dev)
            _lib.call("sa_moe_partition", _lib.ptr(self.expert_of_dev), M, _lib.ptr(counts),
                      _lib.ptr(perm), _lib.ptr(ws), ws.numel(), _lib.stream())
            self._counts, self._perm = counts, perm

    @property
    def counts_dev(self):
        self._partition()
        return self._counts

    @counts_dev.setter
    def counts_dev(self, v):
        self._counts = v

    @property
    def perm_dev(self):
        self._partition()
        return self._perm

    @perm_dev.setter
    def perm_dev(self, v):
        self._perm = v


def _check_two(router: Router):
    if router.num_experts != 2:
        raise ShapeError("the device router implements the two-expert (mult, shift) mixture")


def route_plan(x: torch.Tensor, w_g: torch.Tensor, want_logits=False):
    """Fused K4: logits → winner/gate → stable partition. Returns
    (DispatchPlan, logits-or-None). No host synchronisation."""
    M, d = x.shape
    dev = x.device
    expert_of = torch.empty(M, dtype=torch.int32, device=dev)
    gate = torch.empty(M, dtype=torch.float32, device=dev)
    counts = torch.empty(2, dtype=torch.int32, device=dev)
    perm = torch.empty(M, dtype=torch.int32, device=dev)
    logits = torch.empty((M, 2), dtype=torch.float32, device=dev) if want_logits else None
    ws = _lib.Workspace.get(_lib.load().sa_moe_route_workspace(M), slot=1)
    _lib.call("sa_moe_route", _lib.ptr(x), _lib.ptr(w_g), M, d, tie_threshold(),
              _lib.ptr(logits), _lib.ptr(expert_of), _lib.ptr(gate), _lib.ptr(counts),
              _lib.ptr(perm), _lib.ptr(ws), ws.numel(), _lib.stream())
    return DispatchPlan(expert_of, gate, counts, perm), logits


def ln_route_plans(x: torch.Tensor, gain, bias, w_gs, eps: float = 1e-5):
    """LayerNorm of x fused with 1..3 routers on its output (d = 32k <= 256).
    Returns (y, [DispatchPlan per router]); the plans are views of stacked
    device buffers, no host synchronisation."""
    M, d = x.shape
    nr = len(w_gs)
    dev = x.device
    y = torch.empty_like(x)
    expert_of = torch.empty((nr, M), dtype=torch.int32, device=dev)
    gate = torch.empty((nr, M), dtype=torch.float32, device=dev)
    counts = torch.empty((nr, 2), dtype=torch.int32, device=dev)
    perm = torch.empty((nr, M), dtype=torch.int32, device=dev)
    ws = _lib.Workspace.get(_lib.load().sa_ln_route_workspace(M, nr), slot=1)
    wp = [_lib.ptr(w) for w in w_gs] + [None] * (3 - nr)
    _lib.call("sa_ln_route", _lib.ptr(x), _lib.ptr(gain), _lib.ptr(bias), _lib.ptr(y), M, d,
              float(eps), nr, wp[0], wp[1], wp[2], tie_threshold(), _lib.ptr(expert_of),
              _lib.ptr(gate), _lib.ptr(counts), _lib.ptr(perm), _lib.ptr(ws), ws.numel(),
              _lib.stream())
    return y, [DispatchPlan(expert_of[r], gate[r], counts[r], perm[r]) for r in range(nr)]


def route(x, router: Router):
    """(p, logits): p = softmax(x @ W_g) rowwise (ref moe.py:81-84)."""
    x = to_device(x)
    _check_two(router)
    _, logits = route_plan(x, router.w_g.contiguous(), want_logits=True)
    return softmax2(logits), logits


def softmax2(logits: torch.Tensor) -> torch.Tensor:
    """Row softmax of (M, 2) f32 logits in the reference's operation order
    (max-shift, exp, sum, divide; ref tensor.py:97-103) and with the router
    kernel's arithmetic (moe.cu `decide`): a deficit inside numpy's exp tie
    band gives exactly 1, as numpy's f32 exp does, so argmax(p) and p[winner]
    equal the device plan's winner and gate bit for bit."""
    sh = logits - logits.max(dim=1, keepdim=True).values
    e = torch.where(sh >= -tie_threshold(), torch.ones_like(sh), torch.exp(sh))
    return e / (e[:, :1] + e[:, 1:])


def dispatch(p, logits) -> DispatchPlan:
    """Argmax expert with ties to the lower index, winning gate, ascending
    index lists (ref moe.py:87-92). The winner is decided from the logits with
    the numpy tie rule, which equals argmax(p) of the reference bit-for-bit."""
    logits = to_device(logits)
    if logits.ndim != 2 or logits.shape[1] != 2:
        raise ShapeError("the device dispatch implements the two-expert mixture")
    M = logits.shape[0]
    dev = logits.device
    expert_of = torch.empty(M, dtype=torch.int32, device=dev)
    gate = torch.empty(M, dtype=torch.float32, device=dev)
    counts = torch.empty(2, dtype=torch.int32, device=dev)
    perm = torch.empty(M, dtype=torch.int32, device=dev)
    ws = _lib.Workspace.get(_lib.load().sa_moe_route_workspace(M), slot=1)
    _lib.call("sa_moe_dispatch", _lib.ptr(logits), M, tie_threshold(), _lib.ptr(expert_of),
              _lib.ptr(gate), _lib.ptr(counts), _lib.ptr(perm), _lib.ptr(ws), ws.numel(),
              _lib.stream())
    return DispatchPlan(expert_of, gate, counts, perm)


def moe_forward(x, experts: Sequence, plan: DispatchPlan) -> torch.Tensor:
    """Gather tokens per expert, process, scale by the gate, scatter back
    (ref moe.py:95-108). A (dense, shift) expert pair of the package's own
    layer types runs as ONE fused device launch (K5); other duck-typed experts
    go through gather → expert.forward → scatter."""
    from .model import fused_expert_forward  # local import: model imports moe
    x = to_device(x)
    y = fused_expert_forward(x, experts, plan)
    if y is not None:
        return y
    out = None
    counts = plan.counts_dev.cpu()
    c0 = int(counts[0])
    for e, expert in enumerate(experts):
        idx = plan.perm_dev[:c0] if e == 0 else plan.perm_dev[c0:]
        if idx.numel() == 0:
            continue
        idx = idx.long()
        ye = to_device(expert.forward(x[idx]))
        if out is None:
            out = torch.zeros((x.shape[0], ye.shape[1]), dtype=ye.dtype, device=x.device)
        elif ye.shape[1] != out.shape[1]:
            raise ShapeError("experts disagree on output dim")
        out[idx] = ye * plan.gate_dev[idx, None]
    return out if out is not None else x.clone()


def latency_coefficients(lat: Sequence[float]) -> np.ndarray:
    """α_i = lat_i / Σ lat (ref moe.py:74-78)."""
    lat = np.asarray(lat, dtype=np.float64)
    if np.any(lat <= 0):
        raise ValueError("latencies must be positive")
    return lat / lat.sum()
