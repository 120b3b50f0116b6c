"""Teacher-forced per-block parity diagnosis (GPU box): every block of a
config is fed the ORACLE's block input and its output (and its attention /
MLP halves) compared with the oracle's. Prints one line per block.

    python scripts/diag_parity.py pvt_v1_tiny [batch]
"""

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import nets, ops  # noqa: E402
from paper_2306_06446_b200 import model as MD  # noqa: E402
from paper_2306_06446_b200 import specs  # noqa: E402

F32 = np.float32


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.detach().cpu().numpy()


def main():
    name = sys.argv[1]
    b = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    spec = specs.BUILDERS[name]()
    net = nets.build(spec)
    m = MD.Network(spec)
    images = ops.rng(12).uniform(0, 1, (b, 224, 224, 3)).astype(F32)
    grid = images - 0.5
    for si, (st, S, GS) in enumerate(zip(spec["stages"], net["stages"], m.stages)):
        patches = nets.patchify(grid, st["patch"])
        _, n, pd = patches.shape
        d = st["d"]
        tok = ops.mm(patches.reshape(b * n, pd), S["pe"]).reshape(b, n, d)
        if "cls" in S:
            tok = np.concatenate([np.broadcast_to(S["cls"], (b, 1, d)), tok], axis=1)
        if "pos" in S:
            tok = tok + S["pos"]
        one, zero = np.ones(d, F32), np.zeros(d, F32)
        if st.get("embed_norm"):
            tok = ops.layer_norm(tok, one, zero)
        for bi, (B, GB) in enumerate(zip(S["blocks"], GS.blocks)):
            nrows = tok.shape[1]
            tr = nets.Trace()
            h = tok + nets.attention_fwd(B, ops.layer_norm(tok, one, zero), "a", tr)
            flat = ops.layer_norm(h, one, zero).reshape(-1, d)
            out = h + nets.linear_fwd(B["mlp"], flat, "m", tr).reshape(b, nrows, d)
            g_out = host(GB.forward(dev(tok)))
            x = dev(tok)
            g_h = host(GB.attn.forward(GB.ln1.forward(x), residual=x))
            hh = dev(h)
            g_m = host(GB.mlp.forward(GB.ln2.forward(hh).reshape(-1, d),
                                      residual=hh.reshape(-1, d))).reshape(b, nrows, d)
            # route flips (teacher forced at the module level inside the block call)
            flips = []
            for rec in tr.moe:
                key = rec["name"]
                mod = GB.mlp if key == "m" else GB.attn.proj[key[-1]]
                if isinstance(mod, MD.MoeModule) and mod.last_plan is not None:
                    flips.append(int((mod.last_plan.expert_of != rec["expert_of"]).sum()))
            print(f"s{si}.b{bi} d={d} n={nrows} {B['cfg']['attn_mode']:>13s} "
                  f"block={rel(g_out, out):.2e} attn={rel(g_h, h):.2e} "
                  f"mlp={rel(g_m, out):.2e} last-call route flips={flips}", flush=True)
            tok = out
        if st.get("stage_norm"):
            tok = ops.layer_norm(tok, one, zero)
        if si + 1 < len(spec["stages"]):
            side = int(round(np.sqrt(n)))
            grid = tok.reshape(b, side, side, d)


if __name__ == "__main__":
    main()
