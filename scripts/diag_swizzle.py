#!/usr/bin/env python3
"""Diagnose the tensor-core operand layout: y = x @ I with structured x."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_06446_b200 import _lib, model as MD  # noqa: E402

M, K = 128, 32
x = (np.arange(M)[:, None] * 100 + np.arange(K)[None, :]).astype(np.float32)
w = np.eye(K, dtype=np.float32)
lay = MD.Linear(w)
pk, bn, kind = lay.tc_pack()
xd = torch.from_numpy(x).cuda()
y = torch.empty((M, K), dtype=torch.float32, device="cuda")
_lib.call("sa_tc_linear", _lib.ptr(xd), _lib.ptr(pk), kind, bn, _lib.ptr(y), M, K, K, None, 0,
          _lib.stream())
yh = y.cpu().numpy()
bad = np.argwhere(yh != x)
print("mismatches", len(bad), "of", yh.size)
for r in (0, 1, 2, 3, 8, 9):
    print(r, yh[r].astype(int).tolist())
# weights check: x = identity rows, w = arange
x2 = np.eye(K, dtype=np.float32)
w2 = (np.arange(K)[:, None] * 100 + np.arange(K)[None, :]).astype(np.float32)
lay2 = MD.Linear(w2)
pk2, bn2, _ = lay2.tc_pack()
xd2 = torch.from_numpy(np.tile(x2, (4, 1))).cuda()
y2 = torch.empty((128, K), dtype=torch.float32, device="cuda")
_lib.call("sa_tc_linear", _lib.ptr(xd2), _lib.ptr(pk2), 0, bn2, _lib.ptr(y2), 128, K, K, None, 0,
          _lib.stream())
y2h = y2.cpu().numpy()[:K]
print("weight-side mismatches", int((y2h != w2).sum()))
for r in (0, 1, 2, 3):
    print(r, y2h[r].astype(int).tolist())
