#!/usr/bin/env python3
"""One eager PVTv2-B0 forward (B=256) for an ncu launch list:
ncu --metrics gpu__time_duration.sum --csv python scripts/fwd_launches.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_06446_b200 import model as MD, specs  # noqa: E402

m = MD.Network(specs.pvt_v2_b0())
x = torch.from_numpy(np.random.default_rng(0).uniform(0, 1, (256, 224, 224, 3)).astype(np.float32)).cuda()
m.forward(x)
torch.cuda.synchronize()
