#!/usr/bin/env python3
"""ShiftAddViT-PVTv2-B0 inference throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

One step = one full forward of the ShiftAddViT PVTv2-B0 (LA + Quant + MoE
both, last stage MSA; specs.pvt_v2_b0) over a batch of 256 synthetic 224×224
images per GPU (weak scaling), followed by the only collective of the path:
an all-gather of the logits. Prints ONE JSON line on rank 0.

- value: device-timed (CUDA events, barrier + synchronize both sides, max over
  ranks) with the images already resident in HBM; each step reads a 154 MB
  input (> the 126 MB L2), so no extra L2 flush is needed;
- e2e: the same forward through the public API with the images copied from
  pinned host memory and the logits read back every step;
- roofline: the dominant library kernel, timed with CUDA events around its
  calls inside the forward, against MEASURED_PEAKS.json;
- cpu_baseline: the numpy oracle (restatement of the reference, oracle/) on a
  bounded sample of the same workload on this host's cores.
`--impl reference` times only that CPU reference (rank 0), same metric/config.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "ShiftAddViT-PVTv2-B0 images/sec"
UNIT = "images/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=256, help="images per GPU")
    ap.add_argument("--variant", default="moe")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--skip-kernels", action="store_true", help="no standalone kernel timings")
    return ap.parse_args()


def config_dict(args, world):
    return {"workload": f"pvt_v2_b0-{args.variant} forward, 224x224, batch {args.batch}/GPU",
            "model": "ShiftAddViT-PVTv2-B0 (LA+Quant+MoE both, last stage MSA)",
            "global_batch": args.batch * world, "img": 224, "parallelism": f"dp{world}",
            "l2": "inputs larger than L2 (154 MB/step)", "precision": "fp32 parity mode"}


# ---------------------------------------------------------------- CPU baseline


def cpu_reference(spec, images_per_step, seconds, max_steps=None):
    """Oracle forward on a bounded sample; returns (img/s, images, seconds, cores)."""
    from oracle import nets, ops
    net = nets.build(spec)
    g = ops.rng(1234)
    imgs = g.uniform(0, 1, (images_per_step, 224, 224, 3)).astype(np.float32)
    nets.forward(net, imgs[:1])   # warm-up (BLAS init)
    done, t0 = 0, time.perf_counter()
    steps = 0
    while True:
        nets.forward(net, imgs)
        done += images_per_step
        steps += 1
        el = time.perf_counter() - t0
        if (max_steps is None and el >= seconds) or (max_steps is not None and steps >= max_steps):
            break
    cores = len(os.sched_getaffinity(0))
    return done / el, done, el, cores


# ---------------------------------------------------------------- clocks


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        # NVML polls in microseconds, so the ~100 ms timed region gets many
        # samples; nvidia-smi (one subprocess per sample) is the fallback.
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            bits = (pynvml.nvmlClocksThrottleReasonHwSlowdown,
                    pynvml.nvmlClocksThrottleReasonHwThermalSlowdown,
                    pynvml.nvmlClocksThrottleReasonSwThermalSlowdown,
                    pynvml.nvmlClocksThrottleReasonSwPowerCap)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            while not self._stop.is_set():
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                r = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                self.rows.append([str(sm), str(mx)] +
                                 ["Active" if r & b else "Not Active" for b in bits])
                self._stop.wait(0.005)
            return
        except Exception:
            pass
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}",
                                      f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([c.strip() for c in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=6)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > i + 2 and r[i + 2].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ---------------------------------------------------------------- roofline


def op_bytes(name, args):
    """Algorithmic HBM bytes of one C-ABI call (SURVEY §8d, fp32 activations)."""
    A = 4
    if name == "sa_sign_hash":
        _, B, n, d, h = args[:5]
        return B * n * d * A + B * n * d // 8
    if name in ("sa_linear_binary_attn", "sa_hamming_attn"):
        B, n, d = args[7], args[8], args[9]
        return 2 * B * n * d // 8 + 2 * B * n * d * A + (B * n * d * A if args[5] else 0) * 0
    if name == "sa_linear":
        M, K, N = args[4], args[5], args[6]
        kind = args[2]
        wbytes = K * N * (1 if kind == 1 else 4)
        return M * K * A + M * N * A + wbytes + (M * N * A if args[8] else 0)
    if name == "sa_moe_linear":
        M, K, N = args[9], args[10], args[11]
        return M * K * A + M * N * A + K * N * 5 + (M * N * A if args[8] else 0) + M * 8
    if name == "sa_moe_mlp":
        M, d, hidden = args[11], args[12], args[13]
        return 2 * M * d * A + 2 * d * hidden * 5 + (M * d * A if args[10] else 0) + M * 8
    if name == "sa_mlp":
        M, d, hidden = args[6], args[7], args[8]
        return 2 * M * d * A + (M * d * A if args[10] else 0)
    if name == "sa_moe_route":
        M, d = args[2], args[3]
        return M * d * A + M * 12
    if name == "sa_layernorm":
        M, d = args[4], args[5]
        return 2 * M * d * A
    if name in ("sa_patch_embed", "sa_tc_patch_embed", "sa_tc_patch_embed_ln"):
        B, H, W, C, p = args[1:6]
        d = args[8] if name == "sa_patch_embed" else args[9]
        n = (H // p) * (W // p)
        return B * H * W * C * A + B * n * d * A
    if name == "sa_tc_linear":
        kind, M, K, N, res = args[2], args[5], args[6], args[7], args[8]
        return M * K * A + M * N * A + K * N * (2 if kind == 1 else 6) + (M * N * A if res else 0)
    if name == "sa_tc_moe_linear":
        M, K, N, res = args[9], args[10], args[11], args[8]
        return M * K * A + M * N * A + K * N * 8 + (M * N * A if res else 0) + M * 8
    if name in ("sa_tc_moe_mlp_fused", "sa_tc_moe_mlp"):
        if name == "sa_tc_moe_mlp_fused":
            res, M, d, hidden = args[9], args[10], args[11], args[12]
        else:
            res, M, d, hidden = args[11], args[12], args[13], args[14]
        return 2 * M * d * A + (M * d * A if res else 0) + M * 8 + 2 * d * hidden * 8
    if name in ("sa_tc_mlp_fused", "sa_tc_mlp"):
        if name == "sa_tc_mlp_fused":
            M, d, hidden, res = args[6], args[7], args[8], args[9]
        else:
            M, d, hidden, res = args[8], args[9], args[10], args[11]
        return 2 * M * d * A + (M * d * A if res else 0) + 2 * d * hidden * 6
    if name == "sa_ln_route":
        M, d, nr = args[4], args[5], args[7]
        return 2 * M * d * A + nr * M * 12
    if name == "sa_softmax_attn":
        B, n, d = args[4], args[5], args[6]
        return 4 * B * n * d * A
    if name == "sa_softmax_attn_strided":
        B, n, d = args[5], args[6], args[7]
        return 4 * B * n * d * A
    if name == "sa_tc_moe_linear_grouped":
        nprob, M, K, N = args[6], args[9], args[10], args[11]
        return nprob * (M * K * A + M * N * A + K * N * 8 + M * 12)
    if name == "sa_ln_qkv_hash":
        # x in, v out, q/k codes, three (expert, gate) dispatch arrays
        B, n, d = args[14], args[15], args[16]
        M = B * n
        return 2 * M * d * A + 2 * M * d // 8 + 3 * M * 8
    if name == "sa_fused_moe_linear":
        # x, residual in; y out; (expert, gate) dispatch array
        M, d = args[6], args[7]
        return 3 * M * d * A + M * 8
    if name == "sa_pool":
        B, n, d = args[2], args[3], args[4]
        return B * n * d * A
    return None


def kernel_microbench(torch, hbm_peak, iters=20):
    """Standalone timings of the hot-path kernels at the PVTv2-B0 stage-1 shape
    (B=256, n=3136, d=32; hidden 256): K1 sign-hash, K2a binary attention,
    K3 shift-Linear (tensor-core variant 0 and literal exponent-add variant 1),
    K4 route, K5 fused MoE MLP. CUDA events on the launching stream; every
    kernel streams >= 100 MB of fp32 activations (the 126 MB L2 cannot hold a
    launch's working set across launches, except K2a's 3 MB of codes); each
    timing is the mean of `iters` back-to-back launches after one warm-up,
    enqueued behind a device sleep so short ops are not host-bound."""
    import numpy as np
    from paper_2306_06446_b200 import _lib, attention as A, model as MD, moe as MOE
    from paper_2306_06446_b200 import quantize as Q
    B, n, d, hidden = 256, 3136, 32, 256
    M = B * n
    g = np.random.Generator(np.random.PCG64(7))
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    x = dev(g.standard_normal((M, d)).astype(np.float32))
    v = dev(g.standard_normal((M, d)).astype(np.float32))
    dw = dev((g.standard_normal((3, 3, d)) * 0.1).astype(np.float32))
    w1 = (g.standard_normal((d, hidden)) / np.sqrt(d)).astype(np.float32)
    w2 = (g.standard_normal((hidden, d)) / np.sqrt(hidden)).astype(np.float32)
    wg = (g.standard_normal((d, 2)) * 0.3).astype(np.float32)

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        # the iterations are enqueued while the device sleeps, so the events
        # time the kernels, not the host-side launch path of short ops
        torch.cuda._sleep(int(4e7))
        s.record()
        for _ in range(iters):
            fn()
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e) / iters

    rows = []

    def add(kernel, shape, ms, nbytes, bound="hbm", flops=None):
        ach = nbytes / 1e9 / (ms / 1e3)
        r = {"kernel": kernel, "shape": shape, "ms": ms, "bytes": nbytes, "bound": bound,
             "achieved_gbs": ach, "frac_hbm": ach / hbm_peak}
        if flops:
            r["gops"] = flops / 1e9 / (ms / 1e3)
        rows.append(r)

    cq, gq = Q.sign_hash(x, 1, B)
    ck, gk = Q.sign_hash(v, 1, B)
    add("K1 sign_hash", f"({M},{d}) h=1", timed(lambda: Q.sign_hash(x, 1, B)), M * d * 4 + M * d // 8)
    add("K2a linear_binary_attn (+dwconv)", f"B={B} n={n} d={d} h=1",
        timed(lambda: A.binary_core_codes(cq, ck, gq, gk, v, B, 1, dw, A.EPS_NORM, "linear")),
        2 * M * d // 8 + 2 * M * d * 4)
    lay = MD.ShiftLinearLayer(w1)
    y = torch.empty((M, hidden), dtype=torch.float32, device="cuda")
    pk, bn, kind = lay.tc_pack()

    def k3():
        _lib.call("sa_tc_linear", _lib.ptr(x), _lib.ptr(pk), kind, bn, _lib.ptr(y), M, d, hidden,
                  None, 0, _lib.stream())
    add("K3 shift_linear (tcgen05, variant 0)", f"({M},{d})x({d},{hidden})", timed(k3),
        M * d * 4 + M * hidden * 4 + d * hidden)
    xs = x[: M // 16].contiguous()
    ys = torch.empty((M // 16, hidden), dtype=torch.float32, device="cuda")

    def k3b():
        _lib.call("sa_shift_linear", _lib.ptr(xs), _lib.ptr(lay.quant.packed), _lib.ptr(ys),
                  M // 16, d, hidden, -15, 1, _lib.stream())
    ms_b = timed(k3b)
    add("K3 shift_linear (literal exponent-add, variant 1)", f"({M // 16},{d})x({d},{hidden})",
        ms_b, (M // 16) * (d + hidden) * 4 + d * hidden, bound="alu",
        flops=(M // 16) * d * hidden)
    wg_d = dev(wg)   # uploaded once: a per-call pageable copy would sync the host
    add("K4 moe_route (+stable partition)", f"({M},{d})",
        timed(lambda: MOE.route_plan(x, wg_d)), M * d * 4 + M * 12)
    mod = MD.MoeModule(wg, [MD.Mlp(MD.Linear(w1), MD.Linear(w2)),
                            MD.Mlp(MD.ShiftLinearLayer(w1.copy()),
                                   MD.ShiftLinearLayer(w2.copy()))], MD.MoeConfig())
    plan, _ = MOE.route_plan(x, mod.wg.value)
    add("K5 fused MoE MLP (mult+shift experts)", f"({M},{d}) hidden {hidden}",
        timed(lambda: mod.forward(x, plan=plan, residual=v)), 3 * M * d * 4 + M * 8)
    return rows


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    from paper_2306_06446_b200 import specs
    spec = specs.pvt_v2_b0(variant=args.variant)

    if args.impl == "reference":
        if rank != 0:
            return
        per_step = 4
        t0 = time.perf_counter()
        ips, done, el, cores = cpu_reference(spec, per_step, 0, max_steps=max(args.steps, 1))
        line = {"metric": METRIC, "value": ips, "unit": UNIT, "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * el / max(args.steps, 1),
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic uniform(0,1) 224x224x3 images, PCG64 random-init weights",
                "config": config_dict(args, world), "impl": "reference",
                "cpu_baseline": {"value": ips, "unit": UNIT, "cores": cores, "kind": "port",
                                 "sample": f"{args.steps} steps x {per_step} images, numpy oracle "
                                           f"(oracle/nets.py) with all host BLAS threads"},
                "e2e": {"value": ips, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
                "wall_s": time.perf_counter() - t0}
        print(json.dumps(line), flush=True)
        return

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2306_06446_b200 import _lib
    from paper_2306_06446_b200 import model as MD
    from paper_2306_06446_b200.runtime import GraphedForward, OpTimer

    B = args.batch
    m = MD.Network(spec)
    g = np.random.Generator(np.random.PCG64(4242 + rank))
    host_imgs = torch.from_numpy(g.uniform(0, 1, (B, 224, 224, 3)).astype(np.float32)).pin_memory()
    images = host_imgs.cuda()
    gathered = torch.empty((world * B, spec["classes"]), dtype=torch.float32, device="cuda")

    def barrier():
        if world > 1:
            dist.barrier()

    fwd = m.forward if args.no_graph else GraphedForward(m, images)

    def step(inp):
        logits = fwd(inp)
        if world > 1:
            dist.all_gather_into_tensor(gathered, logits)
        return logits

    for _ in range(args.warmup):
        step(images)
    torch.cuda.synchronize()

    # ---- device-timed region (inputs resident) ----
    launches0 = _lib.launch_count()
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        s_ev, e_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s_ev.record()
        for _ in range(args.steps):
            step(images)
        e_ev.record()
        torch.cuda.synchronize()
    barrier()
    ms = s_ev.elapsed_time(e_ev) / args.steps
    launches = _lib.launch_count() - launches0
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = world * B / (ms / 1000.0)

    # launches per forward (eager count: graphs replay the same kernels)
    c0 = _lib.launch_count()
    m.forward(images)
    torch.cuda.synchronize()
    per_fwd = _lib.launch_count() - c0
    gpu_launches = per_fwd * args.steps if not args.no_graph else launches

    # ---- e2e: pinned host images in, logits out, every step ----
    # Serving pipeline (runtime.PipelinedForward): every step uploads its batch
    # from pinned host memory and reads its logits back; uploads / read-backs
    # overlap the neighbouring steps' compute on separate streams. Timed from
    # the first upload to the last read-back (events on the copy streams).
    from paper_2306_06446_b200.runtime import PipelinedForward
    outs = [torch.empty((B, spec["classes"]), dtype=torch.float32).pin_memory() for _ in range(2)]
    if world == 1 and not args.no_graph:
        pipe = PipelinedForward(m, images)
        pipe.run([host_imgs] * max(args.warmup, 2), outs)
        torch.cuda.synchronize()
        s2 = torch.cuda.Event(enable_timing=True)
        e2 = torch.cuda.Event(enable_timing=True)
        s2.record(pipe.h2d)
        pipe.run([host_imgs] * args.steps, outs)
        e2.record(pipe.d2h)
        torch.cuda.synchronize()
        ms2 = s2.elapsed_time(e2) / args.steps
        e2e_mode = "pipelined (H2D / compute / D2H on three streams, two captured forwards)"
    else:
        barrier()
        torch.cuda.synchronize()
        s2, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s2.record()
        for _ in range(args.steps):
            dev_in = host_imgs.to("cuda", non_blocking=True)
            logits = step(dev_in)
            outs[0].copy_(logits, non_blocking=True)
        e2.record()
        torch.cuda.synchronize()
        barrier()
        ms2 = s2.elapsed_time(e2) / args.steps
        e2e_mode = "serial (copy, forward, read-back per step)"
    if world > 1:
        t = torch.tensor([ms2], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms2 = float(t.item())
    e2e = {"value": world * B / (ms2 / 1000.0), "unit": UNIT,
           "h2d_bytes_per_step": host_imgs.numel() * 4, "d2h_bytes_per_step": outs[0].numel() * 4,
           "ms_per_step": ms2, "mode": e2e_mode}

    # ---- per-op device time inside eager forwards (roofline) ----
    timer = OpTimer()
    for _ in range(3):
        torch.cuda.synchronize()
        # the forward is enqueued while the device sleeps: the events time the
        # kernels, not host-side launch gaps
        torch.cuda._sleep(int(3e8))
        with timer.record():
            m.forward(images)
    summ = timer.summary()
    peaks = {}
    pk_path = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(pk_path):
        peaks = json.load(open(pk_path))
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "measured" if "hbm_gbs" in peaks else "fallback"
    ops_rows = []
    for name, r in summ.items():
        nbytes = [op_bytes(name, a) for a in r["args"]]
        total_b = sum(b for b in nbytes if b) if all(b is not None for b in nbytes) else None
        ach = (total_b / 1e9) / (r["ms"] / 1e3) if total_b else None
        ops_rows.append({"op": name, "calls_per_fwd": r["calls"] // 3, "ms_per_fwd": r["ms"] / 3,
                         "bytes_per_fwd": (total_b / 3) if total_b else None,
                         "achieved_gbs": ach, "frac_hbm": (ach / hbm_peak) if ach else None})
    ops_rows.sort(key=lambda r: -r["ms_per_fwd"])
    dom = next(r for r in ops_rows if r["achieved_gbs"] is not None)
    traffic = None
    tr_path = os.path.join(REPO, "profiles", "ncu_traffic.json")
    if os.path.exists(tr_path):   # DRAM bytes per call of the op from the committed ncu capture
        tr = json.load(open(tr_path)).get(dom["op"])
        traffic = tr["dram_bytes_per_call"] if isinstance(tr, dict) else tr
    roofline = {"bound": "hbm", "kernel": dom["op"], "achieved": dom["achieved_gbs"],
                "peak": hbm_peak, "unit": "GB/s", "frac": dom["frac_hbm"],
                "traffic": traffic, "peak_source": peak_src,
                "per_launch_bytes": dom["bytes_per_fwd"] / max(dom["calls_per_fwd"], 1),
                "ms_per_fwd": dom["ms_per_fwd"],
                "timing": "CUDA events around each library call inside 3 eager forwards, each enqueued behind a device sleep"}
    kernels = None if args.skip_kernels else kernel_microbench(torch, hbm_peak)

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32",
            "data": "synthetic uniform(0,1) 224x224x3 images, PCG64 random-init weights",
            "config": config_dict(args, world), "e2e": e2e, "gpu_launches": int(gpu_launches),
            "launches_per_forward": int(per_fwd), "cuda_graph": not args.no_graph,
            "roofline": roofline, "clocks": clk.summary(), "ops": ops_rows[:14],
            "kernels": kernels}

    if rank == 0 and world == 1 and not args.skip_cpu:
        ips, done, el, cores = cpu_reference(spec, 4, args.cpu_seconds)
        line["cpu_baseline"] = {"value": ips, "unit": UNIT, "cores": cores, "kind": "port",
                                "sample": f"{done} images (batches of 4) in {el:.1f}s, numpy oracle "
                                          "with all host BLAS threads"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
