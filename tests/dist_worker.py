"""Worker for the multi-process distributed-driver test (launched by
tests/test_gpu_dist.py through torch.distributed.run; every rank on cuda:0,
gloo process group, host barrier -- several ranks share one device, so no
kernel ever waits on another rank's kernel).  Rank 0 writes the factors to
the .npz path given in argv[1]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as tdist

from paper_2411_09859_b200.dist import ltlt_blk_piv_dist
from paper_2411_09859_b200.inputs import skew_lower


def main():
    out, n, b, nbd = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
    torch.cuda.set_device(0)
    tdist.init_process_group("gloo")
    x = skew_lower(n, 11)
    ctx, L, tau, piv = ltlt_blk_piv_dist(x, b=b, nbd=nbd, barrier="host")
    torch.cuda.synchronize()
    tdist.barrier()
    if tdist.get_rank() == 0:
        # every column is readable from rank 0 through the mapped peer blocks
        np.savez(out, l=L.cpu().numpy(), tau=tau.cpu().numpy(), piv=piv.cpu().numpy(),
                 world=tdist.get_world_size())
    tdist.barrier()
    ctx.close()
    tdist.destroy_process_group()


if __name__ == "__main__":
    main()
