"""Batch sharding for multi-GPU inference.

Inference shards by image: every hot op is per token or per (image, head)
(ref model.py:355-356, attention.py:115-116, model.py:368-372), so rank r of N
runs the contiguous images [r·B/N, (r+1)·B/N) with replicated weights and the
only collective is one gather of the logits after the forward. One process per
GPU (torchrun), NCCL over NVLink on the GPU box, gloo for the CPU tests.
"""

from __future__ import annotations

import os

import torch
import torch.distributed as dist


def world() -> tuple[int, int, int]:
    """(rank, local_rank, world_size) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")),
            int(os.environ.get("WORLD_SIZE", "1")))


def shard_bounds(global_batch: int, rank: int, world_size: int) -> tuple[int, int]:
    """Contiguous image range of `rank`; the first B % N ranks take one extra."""
    if global_batch < 0 or world_size <= 0 or not 0 <= rank < world_size:
        raise ValueError("bad shard request")
    base, rem = divmod(global_batch, world_size)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def gather_logits(logits: torch.Tensor, global_batch: int, group=None) -> torch.Tensor:
    """All-gather every rank's (b_r, classes) logits into (global_batch, classes)
    in rank order (the path's single collective). Works for uneven shards."""
    if not dist.is_available() or not dist.is_initialized():
        return logits
    ws = dist.get_world_size(group)
    sizes = [shard_bounds(global_batch, r, ws) for r in range(ws)]
    width = max(hi - lo for lo, hi in sizes)
    classes = logits.shape[1]
    # NCCL gathers device tensors over NVLink; gloo (CPU tests, or several
    # ranks sharing one GPU) gathers host copies
    dev = logits.device if _backend(group) == "nccl" else torch.device("cpu")
    padded = torch.zeros((width, classes), dtype=logits.dtype, device=dev)
    padded[: logits.shape[0]] = logits.to(dev)
    out = [torch.empty_like(padded) for _ in range(ws)]
    dist.all_gather(out, padded, group=group)
    return torch.cat([o[: hi - lo] for o, (lo, hi) in zip(out, sizes)], dim=0)


def _backend(group=None) -> str:
    return str(dist.get_backend(group)).lower()


def max_over_ranks(value: float, group=None) -> float:
    """Max of a host float over all ranks (device-timed step times)."""
    if not dist.is_available() or not dist.is_initialized():
        return float(value)
    dev = torch.device("cuda", torch.cuda.current_device()) if _backend(group) == "nccl" \
        else torch.device("cpu")
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
