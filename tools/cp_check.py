"""Constraint-parallel run over the ranks of a gloo group (tests/test_gpu_cp.py launches
it with torch.distributed.run, 2 ranks on one GPU: host-driven collectives, no kernel
waits on another rank).  usage: cp_check.py out_dir world_rows_seed"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2407_10449_b200 as tm  # noqa: E402
from paper_2407_10449_b200 import synth  # noqa: E402
from paper_2407_10449_b200.cp import row_shard  # noqa: E402


def main():
    outdir = sys.argv[1]
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    A, b, x0 = synth.paper_random(200, seed=7)
    lo, hi = row_shard(A.shape[0], world, rank)
    cp = tm.ConstraintParallel(A[lo:hi].copy(), b[lo:hi].copy(), burn_in=3)
    X0 = np.tile(x0, (12, 1))
    out = cp.sample(X0, 40, seed=11)
    sm, sq, n = cp.moments()
    if rank == 0:
        np.save(os.path.join(outdir, "out.npy"), out.cpu().numpy())
        np.save(os.path.join(outdir, "mom.npy"), np.concatenate([sm, sq, [n, cp.stats()["rejections"]]]))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
