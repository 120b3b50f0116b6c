"""Inference runtime helpers: per-op device timing (CUDA events on the
launching stream) and CUDA-graph capture of a whole forward.

`OpTimer` hooks the C-ABI dispatcher (`_lib.call`) and brackets every
library call with a pair of CUDA events on the current stream, so the
roofline numbers in bench.py are device durations of the hot-path kernels
measured inside a real forward, not microbenchmarks.
"""

from __future__ import annotations

import contextlib
from collections import defaultdict

import torch

from . import _lib
from . import moe as MOE


class OpTimer:
    """Accumulates device time and call counts per C-ABI entry point."""

    def __init__(self):
        self.events = []          # (name, start, end, meta)
        self._orig = None

    @contextlib.contextmanager
    def record(self):
        orig = _lib.call
        self._orig = orig

        def timed_call(name, *args):
            s = torch.cuda.Event(enable_timing=True)
            e = torch.cuda.Event(enable_timing=True)
            s.record()
            orig(name, *args)
            e.record()
            self.events.append((name, s, e, args))
        _lib.call = timed_call
        try:
            yield self
        finally:
            _lib.call = orig

    def summary(self, key=None):
        """Per-op totals; `key(name, args)` may split an entry point into rows
        (e.g. one per model dim when the shapes run different kernels)."""
        torch.cuda.synchronize()
        out = defaultdict(lambda: {"calls": 0, "ms": 0.0, "args": []})
        for name, s, e, args in self.events:
            r = out[key(name, args) if key else name]
            r["calls"] += 1
            r["ms"] += s.elapsed_time(e)
            r["args"].append(args)
        return dict(out)


class GraphedForward:
    """Capture `model.forward` on a static input buffer into one CUDA graph
    (MoE shapes are resolved on the device, so the graph is reusable across
    inputs). Call with a device tensor of the captured shape."""

    def __init__(self, model, example: torch.Tensor, warmup: int = 2):
        self.model = model
        self.static_in = example.clone()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(warmup):
                self.model.forward(self.static_in)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.static_out = self.model.forward(self.static_in)
        torch.cuda.synchronize()
        # the graph holds raw pointers into the library workspaces: pin them
        # for the graph's lifetime (Workspace also never frees retired ones)
        self._workspaces = _lib.Workspace.live()

    def replay(self):
        MOE.bump_generation()   # host copies of the plans are stale after this
        self.graph.replay()

    def __call__(self, images: torch.Tensor = None) -> torch.Tensor:
        if images is not None and images.data_ptr() != self.static_in.data_ptr():
            self.static_in.copy_(images, non_blocking=True)
        self.replay()
        return self.static_out


class PipelinedForward:
    """Serving loop with host↔device copies overlapped with compute: two
    captured forwards on two device input buffers, a host→device copy stream,
    a compute stream and a device→host stream. Batch i is uploaded while batch
    i-1 is computed and batch i-2's logits are read back; replays stay
    serialised on the compute stream (the library's workspaces are shared)."""

    def __init__(self, model, example: torch.Tensor):
        self.fwd = [GraphedForward(model, example), GraphedForward(model, example)]
        self.h2d = torch.cuda.Stream()
        self.comp = torch.cuda.Stream()
        self.d2h = torch.cuda.Stream()
        self.in_ready = [torch.cuda.Event(), torch.cuda.Event()]
        self.done = [torch.cuda.Event(), torch.cuda.Event()]
        self.read = [torch.cuda.Event(), torch.cuda.Event()]
        for e in self.done + self.read:
            e.record(torch.cuda.current_stream())

    def run(self, host_batches, host_outs):
        """host_batches: pinned host image tensors; host_outs: pinned host
        logits buffers (len >= 2, reused round robin). Returns the number of
        batches issued; completion is on the d2h stream (self.d2h)."""
        for i, hb in enumerate(host_batches):
            k = i & 1
            f = self.fwd[k]
            with torch.cuda.stream(self.h2d):
                self.h2d.wait_event(self.done[k])          # buffer k no longer read
                f.static_in.copy_(hb, non_blocking=True)
                self.in_ready[k].record(self.h2d)
            with torch.cuda.stream(self.comp):
                self.comp.wait_event(self.in_ready[k])
                self.comp.wait_event(self.read[k])         # logits k already read back
                f.replay()
                self.done[k].record(self.comp)
            with torch.cuda.stream(self.d2h):
                self.d2h.wait_event(self.done[k])
                host_outs[i % len(host_outs)].copy_(f.static_out, non_blocking=True)
                self.read[k].record(self.d2h)
        return len(host_batches)
