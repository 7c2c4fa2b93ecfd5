"""The N > 1 path on CPU: gloo, world_size 2 (no GPU needed).

Each rank runs the CPU oracle on its own chain shard (global chain offsets, the
same RNG counters the GPU uses), then the moments are all-reduced.  The result
must equal a single-process run over all chains: per-chain trajectories do not
depend on the split, and the reduced sums agree to rounding.
"""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2407_10449_b200 import dist as tdist


def test_shard_partition():
    for total in (1, 7, 4096, 65536):
        for world in (1, 2, 3, 8):
            parts = [tdist.shard(total, r, world) for r in range(world)]
            assert parts[0][0] == 0
            for (o, c), (o2, _) in zip(parts, parts[1:]):
                assert o + c == o2
            assert sum(c for _, c in parts) == total
            assert max(c for _, c in parts) - min(c for _, c in parts) <= 1
    assert tdist.weak_shard(4096, 3) == (3 * 4096, 4096)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outdir):
    import torch
    import torch.distributed as dist
    import oracle
    from paper_2407_10449_b200 import synth
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    A, b, x0 = synth.make_instance(3, m=40, d=12)
    off, cnt = tdist.shard(10, rank, world)
    r = oracle.run(A, b, np.tile(x0, (cnt, 1)), 15, seed=103, chain_offset=off, nthreads=1)
    s, q, n, rej = tdist.reduce_moments(r["sum"], r["sumsq"], r["n_rec"], r["rejections"], "cpu")
    tmax = tdist.max_over_ranks(float(rank + 1), "cpu")
    np.save(os.path.join(outdir, f"X{rank}.npy"), r["X"])
    if rank == 0:
        np.save(os.path.join(outdir, "red.npy"), np.concatenate([s, q, [n, rej, tmax]]))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_matches_single_process():
    import oracle
    from paper_2407_10449_b200 import synth
    with tempfile.TemporaryDirectory() as td:
        mp.spawn(_worker, args=(2, _free_port(), td), nprocs=2, join=True)
        X = np.concatenate([np.load(os.path.join(td, f"X{r}.npy")) for r in range(2)])
        red = np.load(os.path.join(td, "red.npy"))
    A, b, x0 = synth.make_instance(3, m=40, d=12)
    ref = oracle.run(A, b, np.tile(x0, (10, 1)), 15, seed=103, nthreads=1)
    assert np.array_equal(X, ref["X"])  # bitwise: the split does not change any chain
    d = A.shape[1]
    assert np.allclose(red[:d], ref["sum"], rtol=1e-13, atol=1e-13)
    assert np.allclose(red[d:2 * d], ref["sumsq"], rtol=1e-13, atol=1e-13)
    assert int(red[2 * d]) == ref["n_rec"] and int(red[2 * d + 1]) == ref["rejections"]
    assert red[2 * d + 2] == 2.0  # MAX over ranks
