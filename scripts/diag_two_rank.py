"""Two ranks sharing cuda:0 (gloo): compare each rank's shard logits with the
same images run in one process; argv[1] = 1 serialises the two forwards."""
import os
import socket
import sys

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import ops  # noqa: E402
from paper_2306_06446_b200 import specs  # noqa: E402


def worker(rank, port, serial, images, spec):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    from paper_2306_06446_b200 import model as MD
    m = MD.Network(spec)
    for turn in range(2):
        if serial:
            dist.barrier()
            if turn != rank:
                continue
        elif turn:
            continue
        y = m.forward(torch.from_numpy(images[2 * rank: 2 * rank + 2]).cuda()).cpu().numpy()
        np.save(f"/tmp/rank{rank}.npy", y)
    dist.barrier()
    dist.destroy_process_group()


def main():
    serial = int(sys.argv[1]) if len(sys.argv) > 1 else 0
    spec = specs.pvt_v2_b0(img=64, classes=10)
    images = ops.rng(5).uniform(0, 1, (4, 64, 64, 3)).astype(np.float32)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.spawn(worker, args=(port, serial, images, spec), nprocs=2, join=True)
    from paper_2306_06446_b200 import model as MD
    m = MD.Network(spec)
    full = m.forward(torch.from_numpy(images).cuda()).cpu().numpy()
    for r in range(2):
        y = np.load(f"/tmp/rank{r}.npy")
        sub = m.forward(torch.from_numpy(images[2 * r: 2 * r + 2]).cuda()).cpu().numpy()
        print(f"serial={serial} rank{r}: vs full {np.abs(y - full[2*r:2*r+2]).max():.3e} "
              f"vs in-process sub {np.abs(y - sub).max():.3e}; in-process sub vs full "
              f"{np.abs(sub - full[2*r:2*r+2]).max():.3e}")


if __name__ == "__main__":
    main()
