"""Constraint-parallel sampling: the rows of A split over the ranks of
a torch.distributed group, all C chains on every rank.  Per iteration the library's
four tmvn_cp_* launches alternate with three collectives run here (argument
marshalling and collectives only; every step of the path runs in the library's
kernels, cp.cu).  Prop. 1: the union of the infeasible arcs is
associative, so the merged level-1 bucket tables plus the gathered live arcs give every
rank the same I_act, theta and iterate -- bitwise those of one rank with all rows."""
import ctypes

import numpy as np


def row_shard(m, world, rank):
    """Contiguous, balanced row range [lo, hi) of rank `rank` out of `world`."""
    per, extra = divmod(m, world)
    lo = rank * per + min(rank, extra)
    return lo, lo + per + (1 if rank < extra else 0)


class _Coll:
    """all_reduce / all_gather over a group (identity without one).  With the gloo
    backend CUDA tensors go through host copies (tests run two ranks on one GPU with
    host-driven collectives: no kernel waits on another rank)."""

    def __init__(self, group):
        import torch.distributed as dist
        self.dist = dist if (dist.is_available() and dist.is_initialized()) else None
        self.group = group
        self.world = self.dist.get_world_size(group) if self.dist else 1
        self.rank = self.dist.get_rank(group) if self.dist else 0
        self.host = bool(self.dist) and self.dist.get_backend(group) == "gloo"

    def all_reduce(self, t, op):
        if not self.dist:
            return
        op = {"max": self.dist.ReduceOp.MAX, "sum": self.dist.ReduceOp.SUM}[op]
        if self.host and t.is_cuda:
            h = t.cpu()
            self.dist.all_reduce(h, op=op, group=self.group)
            t.copy_(h)
        else:
            self.dist.all_reduce(t, op=op, group=self.group)

    def all_gather(self, out, t):
        """out: world x t.shape (rank order)."""
        if not self.dist:
            out[0].copy_(t)
            return
        if self.host and t.is_cuda:
            h = t.cpu()
            parts = [h.new_empty(h.shape) for _ in range(self.world)]
            self.dist.all_gather(parts, h, group=self.group)
            for r in range(self.world):
                out[r].copy_(parts[r])
        else:
            self.dist.all_gather(list(out.unbind(0)), t, group=self.group)


class ConstraintParallel:
    """Rank-local sampler over rows A_r, b_r of the polytope (pass the rank's own rows,
    e.g. A[lo:hi] with row_shard); X0 (C x d) is the same on every rank.

    >>> cp = ConstraintParallel(A[lo:hi], b[lo:hi], group=None, cap=1024)
    >>> out = cp.sample(X0, n_iter, seed)      # identical on every rank
    """

    # cp_theta keeps world * cap gathered arcs of a chain in shared memory (48 B each):
    # at most (227 KB - 32) / 48 per chain on B200
    SMEM_ARCS = (227 * 1024 - 32) // 48

    def __init__(self, A_rows, b_rows, group=None, cap=None, check_every=None, **opts):
        import torch
        from . import Sampler
        self.torch = torch
        if opts.get("precision", 0) != 0:
            raise ValueError("constraint-parallel iterations are FP64 only (precision 0)")
        self.s = Sampler(A_rows, b_rows, latency=0, **opts)
        self.coll = _Coll(group)
        limit = self.SMEM_ARCS // self.coll.world
        self.cap = min(1024, limit) if cap is None else int(cap)
        if self.cap > limit:
            raise ValueError(f"cap={self.cap} x world={self.coll.world} live arcs per chain exceed the "
                             f"shared memory of cp_theta (cap <= {limit})")
        # live-arc overflow is flagged on the device in the iteration it happens (the chain
        # stays); the host reads the flag every check_every iterations (default: K)
        self.check_every = int(check_every or self.s.options().recompute_every or 32)

    def sample(self, X0, n_iter, seed):
        torch = self.torch
        from . import _check, _f64, _ptr, lib
        L = lib()
        h = self.s.h
        X0 = _f64(X0)
        if not hasattr(X0, "data_ptr"):
            X0 = torch.tensor(X0)
        X0 = X0.to("cuda").contiguous()
        C, d = int(X0.shape[0]), int(X0.shape[1])
        dev = X0.device
        t0 = int(self.s.options().iter_offset)
        err = torch.zeros(1, dtype=torch.int64, device=dev)
        # the library launches on torch's current stream (set BEFORE tmvn_cp_begin, whose
        # load of X0 must follow the copy above): the NCCL collectives are ordered on it
        # (no host synchronisation per iteration); gloo's host copies synchronise
        self.s.set_options(stream=torch.cuda.current_stream())
        st = L.tmvn_cp_begin(h, _ptr(X0), C, n_iter, seed)
        err[0] = 1 if st != 0 else 0
        self.coll.all_reduce(err, "max")
        if st != 0:
            _check(st, h)
        if int(err[0]) != 0:
            raise RuntimeError("constraint-parallel start failed on another rank")
        nb = 128
        gx = torch.zeros((C, nb), dtype=torch.int64, device=dev)  # uint64 bit patterns < 2^63
        ma = torch.zeros((C, nb), dtype=torch.int64, device=dev)
        cnt = torch.zeros((C, nb), dtype=torch.int32, device=dev)
        live = torch.zeros((C, self.cap, 2), dtype=torch.float64, device=dev)
        nlive = torch.zeros(C, dtype=torch.int32, device=dev)
        W = self.coll.world
        all_live = torch.zeros((W, C, self.cap, 2), dtype=torch.float64, device=dev)
        all_n = torch.zeros((W, C), dtype=torch.int32, device=dev)
        flags = torch.zeros(C, dtype=torch.int32, device=dev)
        ovf = torch.zeros((), dtype=torch.int32, device=dev)
        for it in range(n_iter):
            t = t0 + it
            _check(L.tmvn_cp_stats(h, t, _ptr(gx), _ptr(ma), _ptr(cnt)), h)
            self.coll.all_reduce(gx, "max")
            self.coll.all_reduce(ma, "max")
            self.coll.all_reduce(cnt, "sum")
            _check(L.tmvn_cp_live(h, _ptr(gx), _ptr(ma), _ptr(cnt), self.cap, _ptr(live), _ptr(nlive)), h)
            if W == 1:
                all_n_it, all_live_it = nlive, live  # no copies on one rank
            else:
                self.coll.all_gather(all_live, live)
                self.coll.all_gather(all_n, nlive)
                all_n_it, all_live_it = all_n, all_live
            _check(L.tmvn_cp_theta(h, t, _ptr(gx), _ptr(ma), _ptr(cnt), _ptr(all_live_it), _ptr(all_n_it), W,
                                   self.cap, _ptr(flags)), h)
            self.coll.all_reduce(flags, "max")
            _check(L.tmvn_cp_commit(h, t, _ptr(flags)), h)  # flag 2 (overflow): the chain stays
            ovf = torch.maximum(ovf, flags.max())
            if (it + 1) % self.check_every == 0 or it + 1 == n_iter:
                if int(ovf) >= 2:
                    raise RuntimeError(
                        f"constraint-parallel: more than cap={self.cap} live arcs of one chain on one rank "
                        f"in iterations {t0 + it + 1 - ((it % self.check_every) + 1)}..{t0 + it} (flagged chains "
                        "were held, not advanced, from the overflowing iteration on); raise cap")
        out = torch.empty((C, d), dtype=torch.float64, device=dev)
        _check(L.tmvn_cp_end(h, n_iter, _ptr(out)), h)
        torch.cuda.synchronize()
        return out

    def stats(self):
        return self.s.stats()

    def moments(self):
        return self.s.moments()
