import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2306_06446_b200 import attention as A
B, n, d, h = [int(x) for x in sys.argv[1:5]]
g = np.random.default_rng(0)
q, k, v = (torch.from_numpy(g.standard_normal((B * n, d)).astype(np.float32)).cuda() for _ in range(3))
out = A.binary_core(q, k, v, B, h, None)
torch.cuda.synchronize()
print("ok", B, n, d, h, float(out.abs().sum()))
