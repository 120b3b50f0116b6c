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

UNIT = "images/s"

# BASELINE.json configs benched here: name -> (builder, images per GPU (None =
# global batch split over the ranks), global batch, metric, model description)
CONFIGS = {
    "c2": ("pvt_v2_b0", 256, None, "ShiftAddViT-PVTv2-B0 images/sec",
           "ShiftAddViT-PVTv2-B0 (LA+Quant+MoE both, last stage MSA)"),
    "c3": ("pvt_v1_tiny", 256, None, "ShiftAddViT-PVTv1-Tiny-MoE images/sec",
           "ShiftAddViT-PVTv1-Tiny (LA+Quant+MoE both, MoE MLP, last stage MSA)"),
    "c4": ("deit_tiny", 512, None, "ShiftAddViT-DeiT-T images/sec",
           "ShiftAddViT-DeiT-T (quadratic binary Hamming attention, 197 tokens, 12 blocks)"),
    "c5": ("pvt_v2_b2", None, 2048, "ShiftAddViT-PVTv2-B2 images/sec",
           "ShiftAddViT-PVTv2-B2 (LA+Quant+MoE both, last stage MSA), global batch 2048"),
}
# parity gate tolerance: tier 3 of tests/test_gpu_model.py for every config
# (full-size forwards on arbitrary images: an fp32-accumulation difference can
# flip a hash code or a route near its boundary and the flip cascades; the
# measured values are reported in the line): (logit tol relative to max|logit|,
# max code-flip rate, max route-flip rate)
GATE = {c: (2e-3, 1e-4, 5e-4) for c in ("c2", "c3", "c4", "c5")}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS),
                    help="BASELINE.json config (c2 = the headline PVTv2-B0 metric)")
    ap.add_argument("--batch", type=int, default=None, help="images per GPU (default: config's)")
    ap.add_argument("--router", default="random", choices=["random", "balanced"],
                    help="MoE router weights: random init (reference draw order) or the "
                         "latency-aware routers trained by the reference procedure")
    ap.add_argument("--backend", default=os.environ.get("SA_DIST_BACKEND", "nccl"),
                    help="torch.distributed backend (gloo: several ranks sharing one GPU)")
    ap.add_argument("--skip-parity", action="store_true", help="no parity gate (debug only)")
    ap.add_argument("--variant", default="moe")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--skip-kernels", action="store_true", help="no standalone kernel timings")
    return ap.parse_args()


def batch_per_gpu(args, world):
    per, glob = CONFIGS[args.config][1], CONFIGS[args.config][2]
    if args.batch is not None:
        return args.batch
    return per if per is not None else glob // world


def config_dict(args, world, cpu_sample=None):
    name, _, glob, _, model = CONFIGS[args.config]
    b = batch_per_gpu(args, world)
    d = {"workload": f"{name}-{args.variant} forward, 224x224, batch {b}/GPU",
         "model": model, "config": args.config, "global_batch": b * world, "img": 224,
         "parallelism": f"dp{world}", "router": args.router,
         "l2": f"inputs larger than L2 ({b * 224 * 224 * 3 * 4 / 1e6:.0f} MB/step)",
         "precision": "fp32 parity mode"}
    if cpu_sample is not None:   # the reference arm runs a bounded sample per step
        d["workload"] = f"{name}-{args.variant} forward, 224x224, {cpu_sample} images per step (CPU)"
        d["cpu_images_per_step"] = cpu_sample
    return d


def scaling(args):
    return "strong" if CONFIGS[args.config][1] is None and args.batch is None else "weak"


# ---------------------------------------------------------------- CPU baseline


def cpu_reference(spec, images_per_step, seconds, max_steps=None, router=None):
    """Oracle forward on a bounded sample; returns (img/s, images, seconds, cores)."""
    from oracle import nets, ops
    net = nets.build(spec)
    if router is not None:
        apply_router_oracle(router, net)
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


def apply_router_oracle(router, net):
    """Install a RouterSet (paper_2306_06446_b200.routers) into an oracle net
    dict (oracle/nets.py layout) so the checker runs the same routers."""
    for si, S in enumerate(net["stages"]):
        for bi, B in enumerate(S["blocks"]):
            for key in "qkvo":
                L = B["proj"][key]
                if L["kind"] == "moe":
                    L["wg"] = router.weights[f"s{si}.b{bi}.attn.{key}"]
            if B["mlp"]["kind"] == "moe":
                B["mlp"]["wg"] = router.weights[f"s{si}.b{bi}.mlp"]


def cpu_host_info(spec, router=None):
    """CPU model, BLAS library / thread count, and the reference CLI's pinned
    single-thread figure (ref cli.py:347-355: BLAS limited to one thread) on
    one image."""
    from oracle import nets, ops
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    info = {"cpu_model": model, "cores": len(os.sched_getaffinity(0))}
    try:
        from threadpoolctl import threadpool_info, threadpool_limits
        blas = [p for p in threadpool_info() if p.get("user_api") == "blas"]
        if blas:
            info["blas"] = f"{blas[0].get('internal_api')} {blas[0].get('version')}"
            info["blas_threads"] = blas[0].get("num_threads")
        net = nets.build(spec)
        if router is not None:
            apply_router_oracle(router, net)
        img = ops.rng(99).uniform(0, 1, (1, 224, 224, 3)).astype(np.float32)
        with threadpool_limits(limits=1, user_api="blas"):
            nets.forward(net, img)
            t0 = time.perf_counter()
            nets.forward(net, img)
            el = time.perf_counter() - t0
        info["one_thread"] = {"value": 1.0 / el, "unit": UNIT, "sample": "1 image, BLAS pinned to 1 thread"}
    except Exception as e:   # pragma: no cover - informational only
        info["one_thread"] = {"error": str(e)[:200]}
    return info


def parity_gate(m, spec, images, logits_full, tol):
    """Bench correctness gate (pattern of ref cli.py:141-172: check, then time):
    the oracle (test infrastructure, oracle/) on two of the benchmarked images
    against the device forward of the same two images — logits, top-1, every
    layer's hash codes and MoE winners — plus batch invariance against the
    full-batch logits the timed forward produced. Returns the report dict."""
    import torch
    from oracle import nets
    from paper_2306_06446_b200 import attention as A
    logit_tol, code_rate, route_rate = tol
    imgs2 = images[:2].contiguous()
    host2 = imgs2.cpu().numpy()
    tr = nets.Trace()
    net = nets.build(spec)
    if getattr(m, "_balanced_router", None) is not None:
        apply_router_oracle(m._balanced_router, net)
    t0 = time.perf_counter()
    ref = nets.forward(net, host2, tr)
    oracle_s = time.perf_counter() - t0
    got_codes = []
    orig = A.binary_core_codes

    def capture(cq, ck, *a, **k):
        got_codes.append((cq.clone(), ck.clone()))
        return orig(cq, ck, *a, **k)
    A.binary_core_codes = capture
    try:
        dev2 = m.forward(imgs2)
        torch.cuda.synchronize()
    finally:
        A.binary_core_codes = orig
    got = dev2.cpu().numpy()
    recs = [r for r in tr.attn if "codes_q" in r]
    code_flips = code_total = 0
    for (cq, ck), r in zip(got_codes, recs):
        for dev_c, ref_c in ((cq, r["codes_q"]), (ck, r["codes_k"])):
            a = dev_c.cpu().numpy().view(np.uint32).reshape(ref_c.shape)
            code_flips += int(np.unpackbits((a ^ ref_c).view(np.uint8)).sum())
            heads = ref_c.shape[0] // 2              # codes are (2 images * h, n, words)
            code_total += ref_c.shape[0] * ref_c.shape[1] * (r["q"].shape[1] // heads)
    route_flips = routed = 0
    ref_routes = {r["name"]: r["expert_of"] for r in tr.moe}
    for name, mod in m.moe_modules():
        e = mod.last_plan.expert_of
        route_flips += int((e != ref_routes[name]).sum())
        routed += e.size
    err = float(np.max(np.abs(got.astype(np.float64) - ref)) / np.max(np.abs(ref)))
    full2 = logits_full[:2].cpu().numpy()
    batch_err = float(np.max(np.abs(full2.astype(np.float64) - got)) / np.max(np.abs(got)))
    ok = (err < logit_tol and np.array_equal(got.argmax(1), ref.argmax(1))
          and len(got_codes) == len(recs) and code_flips <= code_rate * max(code_total, 1)
          and route_flips <= route_rate * max(routed, 1) and batch_err == 0.0)
    return {"ok": bool(ok), "images": 2, "logits_rel_err": err, "logit_tol": logit_tol,
            "top1_agree": bool(np.array_equal(got.argmax(1), ref.argmax(1))),
            "code_flips": code_flips, "codes": code_total, "route_flips": route_flips,
            "routes": routed, "batch_invariance_rel_err": batch_err,
            "oracle_seconds": oracle_s,
            "checker": "oracle/ (numpy restatement pinned to the reference's golden vectors)"}


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

    def _nvml(self):
        # NVML is initialised before the timed region starts (its first init
        # can take longer than a short timed region)
        if getattr(self, "_h", None) is None:
            import pynvml
            pynvml.nvmlInit()
            self._pynvml = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self._mx = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        return self._pynvml, self._h

    def _sample(self):
        pynvml, h = self._nvml()
        bits = (pynvml.nvmlClocksThrottleReasonHwSlowdown,
                pynvml.nvmlClocksThrottleReasonHwThermalSlowdown,
                pynvml.nvmlClocksThrottleReasonSwThermalSlowdown,
                pynvml.nvmlClocksThrottleReasonSwPowerCap)
        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
        r = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
        self.rows.append([str(sm), str(self._mx)] + ["Active" if r & b else "Not Active" for b in bits])

    def _run(self):
        # NVML polls in microseconds, so the timed region gets many samples;
        # nvidia-smi (one subprocess per sample) is the fallback.
        try:
            while not self._stop.is_set():
                self._sample()
                self._stop.wait(0.002)
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
        try:
            self._nvml()
        except Exception:
            pass
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=6)
        if not self.rows:   # a timed region shorter than one polling interval
            try:
                self._sample()
            except Exception:
                pass

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        rows = [r for r in self.rows if len(r) >= 6]   # nvidia-smi errors are single fields
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        self.rows = rows
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
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
    if name in ("sa_tc_moe_mlp_fused", "sa_tc_moe_mlp", "sa_tc_moe_mlp_fused_ln"):
        if name in ("sa_tc_moe_mlp_fused", "sa_tc_moe_mlp_fused_ln"):
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
    if name == "sa_fused_moe_linear_ln_route":
        # x, residual in; h and LN2(h) out; two (expert, gate) dispatch arrays
        M, d = args[6], args[7]
        return 4 * M * d * A + 2 * M * 8
    if name == "sa_pool":
        B, n, d = args[2], args[3], args[4]
        return B * n * d * A
    return None


def op_key(name, args):
    """Row of the per-op table: the fused MoE MLP runs two kernels — the
    narrow form (d = 32 / 64, HBM-bound) and the wide form (d = 128 / 160,
    tensor-bound) — so its calls are split by model dim."""
    if name == "sa_tc_moe_mlp_fused":
        return f"{name}[d={args[11]}]"
    return name


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


def load_router(args, spec_name):
    """The latency-aware routers (--router balanced) or None."""
    if args.router != "balanced":
        return None
    from paper_2306_06446_b200 import routers
    return routers.load_balanced(spec_name)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    from paper_2306_06446_b200 import specs
    if os.environ.get("SA_LIB"):   # A/B runs of a library variant (scripts/build_variant.py)
        from paper_2306_06446_b200 import _lib
        _lib.LIB_PATH = os.environ["SA_LIB"]
    spec_name, _, _, METRIC, _ = CONFIGS[args.config]
    spec = specs.BUILDERS[spec_name](variant=args.variant)
    router = load_router(args, spec_name)

    if args.impl == "reference":
        if rank != 0:
            return
        per_step = 4
        t0 = time.perf_counter()
        ips, done, el, cores = cpu_reference(spec, per_step, 0, max_steps=max(args.steps, 1),
                                             router=router)
        host = cpu_host_info(spec, router)
        line = {"metric": METRIC, "value": ips, "unit": UNIT, "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * el / max(args.steps, 1),
                "higher_is_better": True, "scaling": scaling(args), "vs_baseline": None, "dtype": "f32",
                "data": "synthetic uniform(0,1) 224x224x3 images, PCG64 random-init weights",
                "config": config_dict(args, world, cpu_sample=per_step), "impl": "reference",
                "cpu_baseline": {"value": ips, "unit": UNIT, "cores": cores, "kind": "port",
                                 "sample": f"{args.steps} steps x {per_step} images, numpy oracle "
                                           f"(oracle/nets.py) with all host BLAS threads",
                                 **{k: v for k, v in host.items() if k != "cores"}},
                "e2e": {"value": ips, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
                "wall_s": time.perf_counter() - t0}
        print(json.dumps(line), flush=True)
        return

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local % torch.cuda.device_count())   # gloo: ranks may share a GPU
    if world > 1:
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(args.backend)
    from paper_2306_06446_b200 import _lib
    from paper_2306_06446_b200 import dist as D
    from paper_2306_06446_b200 import model as MD
    from paper_2306_06446_b200.runtime import GraphedForward, OpTimer

    B = batch_per_gpu(args, world)
    m = MD.Network(spec)
    if router is not None:
        router.apply_model(m)
        m._balanced_router = router
    g = np.random.Generator(np.random.PCG64(4242 + rank))
    host_imgs = torch.from_numpy(g.uniform(0, 1, (B, 224, 224, 3)).astype(np.float32)).pin_memory()
    images = host_imgs.cuda()

    def barrier():
        if world > 1:
            dist.barrier()

    fwd = m.forward if args.no_graph else GraphedForward(m, images)

    def step(inp):
        logits = fwd(inp)
        if world > 1:   # the path's single collective (dist.gather_logits)
            D.gather_logits(logits, world * B)
        return logits

    for _ in range(args.warmup):
        out = step(images)
    torch.cuda.synchronize()

    # ---- parity gate before timing (ref cli.py:141-172): rank 0 checks two
    # of its benchmarked images against the oracle ----
    parity = None
    if rank == 0 and not args.skip_parity:
        parity = parity_gate(m, spec, images, out, GATE[args.config])
        if not parity["ok"]:
            print(json.dumps({"metric": METRIC, "error": "parity gate failed", "parity": parity}),
                  flush=True)
            sys.exit(1)
    barrier()

    # ---- device-timed region (inputs resident) ----
    launches0 = _lib.launch_count()
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(torch.cuda.current_device()) as clk:
        s_ev, e_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s_ev.record()
        for _ in range(args.steps):
            step(images)
        e_ev.record()
        torch.cuda.synchronize()
    barrier()
    ms = s_ev.elapsed_time(e_ev) / args.steps
    launches = _lib.launch_count() - launches0
    ms = D.max_over_ranks(ms)
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
    ms2 = D.max_over_ranks(ms2)
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
    summ = timer.summary(op_key)
    peaks = {}
    pk_path = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(pk_path):
        peaks = json.load(open(pk_path))
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "measured" if "hbm_gbs" in peaks else "fallback"
    ops_rows = []
    for name, r in summ.items():
        nbytes = [op_bytes(name.split("[")[0], a) for a in r["args"]]
        total_b = sum(b for b in nbytes if b) if all(b is not None for b in nbytes) else None
        ach = (total_b / 1e9) / (r["ms"] / 1e3) if total_b else None
        ops_rows.append({"op": name, "calls_per_fwd": r["calls"] // 3, "ms_per_fwd": r["ms"] / 3,
                         "bytes_per_fwd": (total_b / 3) if total_b else None,
                         "achieved_gbs": ach, "frac_hbm": (ach / hbm_peak) if ach else None})
    ops_rows.sort(key=lambda r: -r["ms_per_fwd"])
    dom = next(r for r in ops_rows if r["achieved_gbs"] is not None)
    traffic = None
    tr_path = os.path.join(REPO, "profiles", "ncu_traffic.json")
    if os.path.exists(tr_path) and args.config == "c2" and B == 256:   # capture's own shape   # DRAM bytes per call of the op from the committed ncu capture
        tr = json.load(open(tr_path)).get(dom["op"])
        traffic = tr["dram_bytes_per_call"] if isinstance(tr, dict) else tr
    roofline = {"bound": "hbm", "kernel": dom["op"], "achieved": dom["achieved_gbs"],
                "peak": hbm_peak, "unit": "GB/s", "frac": dom["frac_hbm"],
                "traffic": traffic, "peak_source": peak_src,
                "per_launch_bytes": dom["bytes_per_fwd"] / max(dom["calls_per_fwd"], 1),
                "ms_per_fwd": dom["ms_per_fwd"],
                "timing": "CUDA events around each library call inside 3 eager forwards, each enqueued behind a device sleep"}
    kernels = None if (args.skip_kernels or args.config != "c2") else kernel_microbench(torch, hbm_peak)

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": scaling(args),
            "vs_baseline": None, "dtype": "f32",
            "data": "synthetic uniform(0,1) 224x224x3 images, PCG64 random-init weights",
            "config": config_dict(args, world), "e2e": e2e, "gpu_launches": int(gpu_launches),
            "launches_per_forward": int(per_fwd), "cuda_graph": not args.no_graph,
            "roofline": roofline, "clocks": clk.summary(), "ops": ops_rows[:14],
            "kernels": kernels, "parity": parity}
    if router is not None:
        line["expert_shares"] = router.shares(m)

    if rank == 0 and world == 1 and not args.skip_cpu:
        ips, done, el, cores = cpu_reference(spec, 4, args.cpu_seconds, router=router)
        host = cpu_host_info(spec, router)
        line["cpu_baseline"] = {"value": ips, "unit": UNIT, "cores": cores, "kind": "port",
                                "sample": f"{done} images (batches of 4) in {el:.1f}s, numpy oracle "
                                          "with all host BLAS threads",
                                **{k: v for k, v in host.items() if k != "cores"}}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
