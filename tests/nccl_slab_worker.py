"""One rank of the multi-process NCCL slab path (launched by tests/test_gpu_parity.py through
torch.distributed.run when >= 2 GPUs are visible): solves a d >= 2 problem over all ranks (halo
rows by ncclSend/ncclRecv inside bsde_step) and writes its owned rows + y0 to <out>.rank<r>.npz."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_13560_b200 import workloads as W  # noqa: E402
from paper_1909_13560_b200.dist import make_slab_solver  # noqa: E402


def main():
    out = sys.argv[1]
    name = sys.argv[2] if len(sys.argv) > 2 else "ex4"
    rank = int(os.environ["RANK"])
    torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    dist.init_process_group("nccl")
    spec = {"ex4": W.ex4_2d(3, 8, npts=257), "basket3d": dict(W.basket_3d(3, 6, 4, P=120), npts=[120, 13, 11])}[name]
    with make_slab_solver(spec) as s:
        r = s.solve()
        np.savez(f"{out}.rank{rank}.npz", layers=s.layers(), own=np.array(s.own), y0=r.y0)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
