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


def test_row_shard():
    from paper_2407_10449_b200.cp import row_shard
    for m in (1, 5, 2000, 16384):
        for world in (1, 2, 3, 8):
            parts = [row_shard(m, world, r) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == m
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            sizes = [h - l for l, h in parts]
            assert max(sizes) - min(sizes) <= 1


def _cp_worker(rank, world, port, outdir):
    import torch
    import torch.distributed as dist
    import oracle
    from paper_2407_10449_b200 import synth
    from paper_2407_10449_b200.cp import _Coll, row_shard
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    coll = _Coll(None)
    assert coll.world == world and coll.rank == rank
    # the collectives the constraint-parallel loop runs, on CPU tensors
    g = torch.tensor([[rank * 10 + 1, 5 - rank]], dtype=torch.int64)
    coll.all_reduce(g, "max")
    c = torch.tensor([rank + 1], dtype=torch.int32)
    coll.all_reduce(c, "sum")
    parts = torch.zeros((world, 3), dtype=torch.float64)
    coll.all_gather(parts, torch.full((3,), float(rank), dtype=torch.float64))
    # Prop. 1 on the oracle: the rows split over the ranks, each rank's
    # infeasible arcs gathered, I_act of the union equals I_act over all rows
    A, b, x0 = synth.make_instance(3, m=90, d=10)
    lo, hi = row_shard(A.shape[0], world, rank)
    nu = oracle.normals(7, 0, 0, A.shape[1])
    al, be, act = oracle.arcs(A[lo:hi] @ x0, A[lo:hi] @ nu, b[lo:hi])
    mine = torch.zeros((A.shape[0], 2), dtype=torch.float64)
    mine[lo:hi, 0] = torch.tensor(np.where(act, al, 0.0))
    mine[lo:hi, 1] = torch.tensor(np.where(act, be, 0.0))
    coll.all_reduce(mine, "sum")  # disjoint rows: the sum is the concatenation
    if rank == 0:
        segs = oracle.intervals(mine[:, 0].numpy(), mine[:, 1].numpy())
        al0, be0, act0 = oracle.arcs(A @ x0, A @ nu, b)
        ref = oracle.intervals(np.where(act0, al0, 0.0), np.where(act0, be0, 0.0))
        np.save(os.path.join(outdir, "cp.npy"), np.array([
            g.tolist() == [[(world - 1) * 10 + 1, 5]], int(c[0]) == world * (world + 1) // 2,
            parts.tolist() == [[float(r)] * 3 for r in range(world)],
            len(segs) == len(ref) and all(np.allclose(a, b_, rtol=0, atol=0) for a, b_ in zip(segs, ref))]))
    dist.barrier()
    dist.destroy_process_group()


def test_constraint_parallel_collectives_gloo():
    with tempfile.TemporaryDirectory() as td:
        mp.spawn(_cp_worker, args=(2, _free_port(), td), nprocs=2, join=True)
        ok = np.load(os.path.join(td, "cp.npy"))
    assert ok.all(), ok


def _bench_worker(rank, world, port, outdir):
    """bench.py's rank plumbing under gloo: strong-scaling shard plan (global chain
    blocks + options.total_chains), whole-job units = SUM over ranks, device time = MAX
    over ranks, and the moment / counter reduction."""
    import torch.distributed as dist
    import bench
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    res = []
    for C_cfg in (4096, 65536, 16, 7):
        opts, cnt = bench.plan_shard(C_cfg, rank, world, "strong")
        wopts, wcnt = bench.plan_shard(C_cfg, rank, world, "weak")
        # rank r "ran" cnt chains x 100 iterations in (10 + r) ms
        units, ms_max, rate = bench.job_rate(float(cnt * 100), 10.0 + rank, "cpu")
        res.append([opts["chain_offset"], cnt, opts["total_chains"], wopts["chain_offset"], wcnt,
                    wopts["total_chains"], units, ms_max, rate])
    np.save(os.path.join(outdir, f"b{rank}.npy"), np.array(res, dtype=np.float64))
    dist.barrier()
    dist.destroy_process_group()


def test_bench_rank_plumbing_gloo():
    world = 2
    with tempfile.TemporaryDirectory() as td:
        mp.spawn(_bench_worker, args=(world, _free_port(), td), nprocs=world, join=True)
        R = [np.load(os.path.join(td, f"b{r}.npy")) for r in range(world)]
    for i, C_cfg in enumerate((4096, 65536, 16, 7)):
        offs = [int(R[r][i, 0]) for r in range(world)]
        cnts = [int(R[r][i, 1]) for r in range(world)]
        assert offs[0] == 0 and offs[1] == cnts[0] and sum(cnts) == C_cfg  # strong: the config's C split
        assert all(int(R[r][i, 2]) == C_cfg for r in range(world))        # every rank: the job's total
        assert [int(R[r][i, 3]) for r in range(world)] == [0, C_cfg]         # weak: C per rank
        assert all(int(R[r][i, 4]) == C_cfg and int(R[r][i, 5]) == world * C_cfg for r in range(world))
        for r in range(world):
            units, ms_max, rate = R[r][i, 6:9]
            assert units == C_cfg * 100 and ms_max == 10.0 + world - 1
            assert abs(rate - C_cfg * 100 / (ms_max * 1e-3)) <= 1e-9 * rate
