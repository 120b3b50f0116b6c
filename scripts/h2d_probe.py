#!/usr/bin/env python3
"""Host-to-device copy bandwidth of one C2 image batch (154 MB, pinned) with
1, 2 and 4 copy streams: the e2e line's input leg (diagnostic)."""
import torch
n = 256*224*224*3
h = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
ss = [torch.cuda.Stream() for _ in range(4)]
for ns in (1, 2, 4):
    ts = []
    for rep in range(5):
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record()
        cur = torch.cuda.current_stream()
        chunk = n // ns
        for i in range(ns):
            ss[i].wait_stream(cur)
            with torch.cuda.stream(ss[i]):
                d[i*chunk:(i+1)*chunk].copy_(h[i*chunk:(i+1)*chunk], non_blocking=True)
        for i in range(ns):
            cur.wait_stream(ss[i])
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = sorted(ts)[2]
    print(f"{ns} streams: {ms:.3f} ms, {n*4/ms/1e6:.1f} GB/s")
