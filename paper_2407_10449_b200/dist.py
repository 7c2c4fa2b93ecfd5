"""Multi-GPU plumbing (one process per GPU, torch.distributed).

Chains are independent (Alg. 1): rank g owns a contiguous
block of chains with global indices [offset, offset + count) -- the library's
`chain_offset` -- and A, b are replicated.  No per-iteration collective exists;
the only ones are the final all_reduce of the moments / counters and the MAX of
the timings.  Used by bench.py; tested on CPU with gloo,
world_size 2 (tests/test_dist.py).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard(total: int, rank: int, world: int):
    """(offset, count) of rank's contiguous block of `total` chains (near-equal split)."""
    base, rem = divmod(total, world)
    count = base + (1 if rank < rem else 0)
    offset = rank * base + min(rank, rem)
    return offset, count


def shard_options(total: int, rank: int, world: int):
    """Sampler options of rank's shard: its global chain offset and the job's chain count
    (options.total_chains: the automatic execution-path choice is then the same on every
    rank, so the shards' chains equal an unsharded run's bitwise)."""
    offset, count = shard(total, rank, world)
    return dict(chain_offset=offset, total_chains=total), count


def weak_shard(per_rank: int, rank: int):
    """(offset, count) when every rank runs `per_rank` chains (weak scaling)."""
    return rank * per_rank, per_rank


def reduce_moments(sum_, sumsq, n, rejections, device):
    """all_reduce(SUM) of [sum (d), sumsq (d), n, rejections]; returns numpy-like tensors."""
    import numpy as np
    buf = torch.tensor(np.concatenate([np.asarray(sum_, dtype=np.float64),
                                       np.asarray(sumsq, dtype=np.float64),
                                       [float(n), float(rejections)]]), dtype=torch.float64,
                       device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(buf, op=dist.ReduceOp.SUM)
    d = (buf.numel() - 2) // 2
    out = buf.cpu().numpy()
    return out[:d], out[d:2 * d], int(round(out[2 * d])), int(round(out[2 * d + 1]))


def max_over_ranks(x: float, device) -> float:
    t = torch.tensor([x], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, device) -> float:
    t = torch.tensor([x], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())
