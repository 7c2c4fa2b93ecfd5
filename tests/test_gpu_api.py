"""Semantics of the public C-ABI on the GPU: errors, determinism, sharding
invariance, resume, device pointers, moments, App. A affine mode, and the
statistical pins of the paper's S4.1 experiment (closed-form 1-D moments)."""
import math

import numpy as np
import pytest

import oracle
import paper_2407_10449_b200 as tm
from paper_2407_10449_b200 import synth

pytestmark = pytest.mark.gpu


def test_errors():
    A, b, x0 = synth.make_instance(3, m=50, d=10)
    s = tm.Sampler(A, b)
    X = np.tile(x0, (8, 1))
    X[5] = 100 * A[17] / np.linalg.norm(A[17])  # violates constraint 17 (at least)
    with pytest.raises(tm.TmvnError) as ei:
        s.sample(X, 3, seed=1)
    assert ei.value.status == -3 and "chain 5" in str(ei.value)
    # boundary start (a_i . x0 == b_i exactly) is not strictly interior (C18)
    sb = tm.Sampler(np.array([[1.0, 0.0], [0.0, 1.0], [-1.0, -1.0]]), np.array([1.0, 2.0, 3.0]))
    with pytest.raises(tm.TmvnError) as eb:
        sb.sample(np.array([[0.0, 0.0], [1.0, 0.5]]), 1, seed=1)
    assert eb.value.status == -3 and "chain 1 violates constraint 0" in str(eb.value)
    # handle stays valid
    out = s.sample(np.tile(x0, (4, 1)), 3, seed=1)
    assert np.all(A @ out.T <= b[:, None])
    with pytest.raises(tm.TmvnError) as ei:
        Az = A.copy()
        Az[2] = 0
        bz = b.copy()
        bz[2] = -1
        tm.Sampler(Az, bz)
    assert ei.value.status == -2
    with pytest.raises(tm.TmvnError) as ei:
        s.set_affine(np.zeros(10), np.triu(np.ones((10, 10))))
    assert ei.value.status == -4
    with pytest.raises(tm.TmvnError):
        tm.Sampler(np.full((2, 2), np.nan), np.ones(2))


def test_shard_invariance_and_resume_bitwise():
    A, b, x0 = synth.make_instance(3, m=300, d=64)
    C = 300
    X0 = np.tile(x0, (C, 1))
    s = tm.Sampler(A, b)
    full = s.sample(X0, 64, seed=7)
    # two "ranks": chain_offset sharding (global chain index in the RNG counter, no split-K)
    s1 = tm.Sampler(A, b, chain_offset=0)
    s2 = tm.Sampler(A, b, chain_offset=173)
    h1 = s1.sample(X0[:173], 64, seed=7)
    h2 = s2.sample(X0[173:], 64, seed=7)
    assert np.array_equal(np.concatenate([h1, h2]), full)
    # resume at a multiple of recompute_every reproduces the run bitwise
    s3 = tm.Sampler(A, b)
    a = s3.sample(X0, 32, seed=7)
    a = s3.sample(a, 32, seed=7)  # iter_offset auto-advanced to 32
    assert np.array_equal(a, full)
    assert s3.options().iter_offset == 64


def test_device_tensors_inplace_and_stream():
    import torch
    A, b, x0 = synth.make_instance(3, m=200, d=50)
    C = 256
    s = tm.Sampler(A, b)
    ref = s.sample(np.tile(x0, (C, 1)), 10, seed=3)
    s2 = tm.Sampler(torch.tensor(A, device="cuda"), torch.tensor(b, device="cuda"))
    stream = torch.cuda.Stream()
    s2.set_options(stream=stream)
    X = torch.tensor(np.tile(x0, (C, 1)), device="cuda")
    s2.sample(X, 10, seed=3, out=X)  # in place
    torch.cuda.synchronize()
    assert np.array_equal(X.cpu().numpy(), ref)


def test_moments_match_trajectory_sums():
    A, b, x0 = synth.make_instance(3, m=120, d=30)
    C, T = 64, 40
    s = tm.Sampler(A, b, burn_in=10, thin=3)
    trace, out = s.test_trace(np.tile(x0, (C, 1)), T, seed=5, chains=np.arange(C))
    sm, sq, n = s.moments()
    rec = [t for t in range(T) if t >= 10 and (t - 10) % 3 == 0]
    X = trace[[t + 1 for t in rec]]  # iterate produced by iteration t
    assert n == C * len(rec)
    assert np.allclose(sm, X.sum(axis=(0, 1)), rtol=1e-12, atol=1e-12)
    assert np.allclose(sq, (X**2).sum(axis=(0, 1)), rtol=1e-12, atol=1e-12)


def trunc_normal_moments(lo, hi):
    phi = lambda z: math.exp(-0.5 * z * z) / math.sqrt(2 * math.pi)
    if lo > 0:
        Z = 0.5 * (math.erfc(lo / math.sqrt(2)) - math.erfc(hi / math.sqrt(2)))
    else:
        Z = 0.5 * (math.erf(hi / math.sqrt(2)) - math.erf(lo / math.sqrt(2)))
    mu = (phi(lo) - phi(hi)) / Z
    return mu, 1.0 + (lo * phi(lo) - hi * phi(hi)) / Z - mu * mu


@pytest.mark.parametrize("interval", [(-1.0, 3.0), (15.0, 16.0)])
def test_section_4_1_protocol(interval):
    """2000 chains, burn-in 500, thinning 10, 1e5 samples.  The chains run as
    20 shards of 100 (chain_offset: bitwise the same chains as one call, global RNG
    counters), so each shard's moments are an independent estimate: the pooled mean and
    variance must lie within 4 standard errors of the closed form (SURVEY 8(c)
    statistical recipe; on [15, 16] sigma^2 = 0.0043, so the paper's 0.01 alone would be
    vacuous) and within the paper's 0.01."""
    A, b, x0 = synth.one_dim(interval)
    G, Cg = 20, 100
    mu, var = trunc_normal_moments(*interval)
    means, vars_, ntot, steps, rej = [], [], 0, 0, 0
    for g in range(G):
        s = tm.Sampler(A, b, burn_in=500, thin=10, chain_offset=g * Cg)
        out = s.sample(np.tile(x0, (Cg, 1)), 1000, seed=2024)
        sm, sq, n = s.moments()
        assert n == Cg * 50
        means.append(sm[0] / n)
        vars_.append(sq[0] / n - (sm[0] / n) ** 2)
        ntot += n
        st = s.stats()
        steps += st["steps"]
        rej += st["rejections"]
        assert np.all(out >= interval[0]) and np.all(out <= interval[1])
    assert ntot == 100000 and steps == 2_000_000
    means, vars_ = np.array(means), np.array(vars_)
    m1, v1 = means.mean(), vars_.mean()
    se_m, se_v = means.std(ddof=1) / np.sqrt(G), vars_.std(ddof=1) / np.sqrt(G)
    assert abs(m1 - mu) <= 4 * se_m, (m1, mu, se_m)
    assert abs(v1 - var) <= 4 * se_v, (v1, var, se_v)
    assert abs(m1 - mu) < 0.01 and abs(v1 - var) < 0.01
    assert rej <= 200  # FP64: the paper saw 8 in FP32 on [15, 16]


def test_orthant_config2_moments():
    A, b, x0 = synth.make_instance(2)
    s = tm.Sampler(A, b, burn_in=15000)
    s.sample(np.tile(x0, (1024, 1)), 20000, seed=102)
    sm, sq, n = s.moments()
    mean = sm / n
    var = sq / n - mean**2
    assert abs(mean.mean() - math.sqrt(2 / math.pi)) < 0.01
    assert abs(var.mean() - (1 - 2 / math.pi)) < 0.01
    assert s.stats()["rejections"] == 0


def test_tiny2d_config1_vs_rejection():
    A, b, x0 = synth.make_instance(1)
    rng = np.random.default_rng(1)
    z = rng.standard_normal((4_000_000, 2))
    acc = z[np.all(z @ A.T <= b, axis=1)]
    s = tm.Sampler(A, b, burn_in=200)
    s.sample(np.tile(x0, (4096, 1)), 2000, seed=101)
    sm, sq, n = s.moments()
    assert np.all(np.abs(sm / n - acc.mean(0)) < 0.01)
    assert np.all(np.abs(sq / n - (acc**2).mean(0)) < 0.02)


def test_affine_change_of_variable():
    """App. A: N(mu, L L^T) truncated; the sampler reports x-space."""
    d = 6
    L, mu = synth.random_spd_factor(d, seed=3)
    rng = np.random.default_rng(4)
    A = rng.standard_normal((9, d))
    x_start = mu.copy()
    b = A @ x_start + rng.uniform(0.5, 1.5, 9)
    s = tm.Sampler(A, b, mu=mu, L=L)
    C = 64
    X0 = np.tile(x_start, (C, 1))
    out = s.sample(X0, 5, seed=11)
    assert np.all(A @ out.T <= b[:, None] + 1e-12)
    # oracle in u-space on the whitened polytope, then x = L u + mu
    Aw, bw = oracle.whiten(A, b, mu, L)
    u0 = oracle.whiten_point(x_start, mu, L)
    r = oracle.run(Aw, bw, np.tile(u0, (C, 1)), 5, seed=11)
    xo = np.array([oracle.unwhiten_point(u, mu, L) for u in r["X"]])
    assert np.max(np.abs(out - xo)) <= 1e-10 * max(1.0, np.max(np.abs(xo)))  # north_star bar
    # per step in x-space, each from the GPU's own x_t (x -> u by the library's trsv, the
    # oracle's own forward substitution on its side): x_{t+1} within 1e-10
    s2 = tm.Sampler(A, b, mu=mu, L=L, record=0)
    X = X0.copy()
    for t in range(6):
        Xn = s2.sample(X, 1, seed=11)
        for c in range(0, C, 9):
            un, _ = oracle.step(Aw, bw, oracle.whiten_point(X[c], mu, L), 11, t, c)
            xn = oracle.unwhiten_point(un, mu, L)
            assert np.max(np.abs(Xn[c] - xn)) <= 1e-10 * max(1.0, np.max(np.abs(xn))), (t, c)
        X = Xn
    # 1-D closed form: x ~ N(2, 4) truncated to [1, 5]
    s1 = tm.Sampler(np.array([[1.0], [-1.0]]), np.array([5.0, -1.0]), mu=np.array([2.0]),
                    L=np.array([[2.0]]), burn_in=100)
    s1.sample(np.full((2000, 1), 3.0), 600, seed=77)
    sm, sq, n = s1.moments()
    mu_u, var_u = trunc_normal_moments(-0.5, 1.5)
    m1 = sm[0] / n
    assert abs(m1 - (2 + 2 * mu_u)) < 0.01
    assert abs(sq[0] / n - m1 * m1 - 4 * var_u) < 0.03


def test_graph_replay_bitwise_equals_launches():
    """CUDA-graph replay of aligned blocks (options.graphs) changes nothing."""
    A, b, x0 = synth.make_instance(3, m=150, d=40)
    C = 200
    outs = []
    for graphs in (0, 1):
        s = tm.Sampler(A, b, burn_in=7, thin=3, graphs=graphs)
        s.set_options(iter_offset=5)  # unaligned head, then whole blocks of 32, then a tail
        out = s.sample(np.tile(x0, (C, 1)), 100, seed=13)
        outs.append((out, s.moments(), s.stats()))
    assert np.array_equal(outs[0][0], outs[1][0])
    assert np.array_equal(outs[0][1][0], outs[1][1][0]) and outs[0][1][2] == outs[1][1][2]
    assert outs[0][2] == outs[1][2]


def test_rng_ahead_and_projection_options_bitwise():
    """options.rng_ahead (nu drawn on a second stream beside the GEMM, double-buffered),
    the chain schedule (dynamic / round-robin) and the graph / plain launch paths give
    bitwise the same chains."""
    A, b, x0 = synth.make_instance(3, m=300, d=70)
    C = 200
    X0 = np.tile(x0, (C, 1))
    ref = tm.Sampler(A, b, rng_ahead=0, graphs=0).sample(X0, 70, seed=11)
    for ra, gr, sc, pi in ((1, 0, 0, 0), (1, 1, 0, 0), (0, 1, 0, 0), (0, 1, 1, 0), (0, 0, 1, 0),
                           (0, 0, 2, 0), (0, 1, 2, 0), (0, 0, 0, 1), (0, 1, 0, 1)):
        out = tm.Sampler(A, b, rng_ahead=ra, graphs=gr, schedule=sc, pipeline=pi).sample(X0, 70, seed=11)
        assert np.array_equal(out, ref), (ra, gr, sc, pi)
    for W in (1, 2, 4, 8, 16):  # warps per chain (16: one 512-thread CTA per chain)
        out = tm.Sampler(A, b, chain_warps=W).sample(X0, 70, seed=11)
        assert np.array_equal(out, ref), W
    for n in (1, 2, 3):  # short calls through the pipelined prologue
        o1 = tm.Sampler(A, b, pipeline=1).sample(X0, n, seed=11)
        o0 = tm.Sampler(A, b).sample(X0, n, seed=11)
        assert np.array_equal(o1, o0), n
    # resume at a multiple of recompute_every with nu drawn ahead (plain + graph blocks)
    for kw in (dict(rng_ahead=1), dict(pipeline=1), dict(rng_gemm=1), dict(rng_overlap=1)):
        s = tm.Sampler(A, b, **kw)
        a = s.sample(X0, 32, seed=11)
        a = s.sample(a, 38, seed=11)
        assert np.array_equal(a, ref), kw
    # round-2 options: nu drawn by the projection's epilogue (rng_gemm), nu drawn while
    # theta is computed (rng_overlap), arcs computed in the projection's epilogue
    # (fuse_arcs), the P/Q ring; plain and graph launches, several W
    for kw in (dict(rng_gemm=1), dict(rng_gemm=1, graphs=0), dict(rng_overlap=1), dict(rng_overlap=1, graphs=0),
               dict(rng_overlap=1, chain_warps=2), dict(fuse_arcs=1), dict(fuse_arcs=1, graphs=0),
               dict(fuse_arcs=1, chain_warps=4), dict(ring=1), dict(ring=1, graphs=0),
               dict(streams=2), dict(streams=3), dict(streams=2, rng_overlap=1),
               dict(streams=2, fuse_arcs=1), dict(streams=2, rng_gemm=1), dict(streams=3, ring=1),
               dict(buckets=1), dict(buckets=2), dict(buckets=2, graphs=0), dict(buckets=2, streams=2)):
        out = tm.Sampler(A, b, **kw).sample(X0, 70, seed=11)
        assert np.array_equal(out, ref), kw
    # chain shards on concurrent streams (the automatic choice from 2048 chains): the same
    # chains bitwise, moments to rounding (the per-group rows regroup)
    C2 = 2304
    X2 = np.tile(x0, (C2, 1))
    s1 = tm.Sampler(A, b, streams=1)
    r1 = s1.sample(X2, 40, seed=3)
    for S in (0, 2, 4):
        sS = tm.Sampler(A, b, streams=S)
        rS = sS.sample(X2, 40, seed=3)
        assert np.array_equal(rS, r1), S
        for u, v in zip(sS.moments()[:2], s1.moments()[:2]):
            assert np.allclose(u, v, rtol=1e-12, atol=1e-12)
        assert sS.stats() == s1.stats()


def test_bucket_mappings_bitwise_on_the_s42_geometry():
    """S4.2's instance (arcs bunched just after theta = 0 from a start deep
    inside): the octave level-1 buckets (options.buckets = 2) and the automatic switch
    (0, which turns octave on after one launch of crowded chains) give bit-identical
    chains to the linear mapping (any monotone bucketing: Prop. 1), one launch per
    iteration and graphed blocks alike."""
    A, b, x0 = synth.paper_random(400, seed=4)
    X0 = np.tile(x0, (300, 1))
    outs = {}
    for bk in (1, 2, 0):
        for g in (0, 1):
            s = tm.Sampler(A, b, buckets=bk, graphs=g, latency=0)
            outs[bk, g] = (s.sample(X0, 40, seed=3), s.moments(), s.stats())
            # the automatic switch turns octave on here (every chain crowds bucket 0)
            assert s.profile()["buckets_used"] == (1 if bk == 1 else 2), (bk, g)
    ref = outs[1, 0]
    # a unit-row random polytope from x0 = 0 (config 3's structure) does not crowd: linear
    A3, b3, x3 = synth.make_instance(3, m=600, d=200)
    s3 = tm.Sampler(A3, b3, latency=0)
    s3.sample(np.tile(x3, (300, 1)), 20, seed=3)
    assert s3.profile()["buckets_used"] == 1
    for key, (X, mom, st) in outs.items():
        assert np.array_equal(X, ref[0]), key
        assert all(np.array_equal(u, v) for u, v in zip(mom, ref[1])), key
        assert st == ref[2], key
    assert np.max(ref[0] @ A.T - b) <= 0.0


def test_odd_m_and_general_interval_path_on_default_options():
    """The production per-chain kernel with the chain's P / Q rows in shared memory on an
    odd m, and the S4.2 geometry, whose arcs crowd the first buckets so that
    more than 256 arcs are live (the general, bitonic-sorted interval path): every step
    against the oracle (north_star bar), feasibility, no rejections."""
    from test_gpu_step import check_trace
    A, b, x0 = synth.make_instance(3, m=301, d=70)
    C, T = 130, 40
    s = tm.Sampler(A, b, latency=0)
    chains = np.array([0, 7, 64, 129])
    trace, out = s.test_trace(np.tile(x0, (C, 1)), T, seed=5, chains=chains)
    check_trace(A, b, trace, 5, chains, projection=1 if s.profile()["oz_guard_ratio"] <= 16 else 2)
    A2, b2, x2 = synth.paper_random(600, seed=600)
    s2 = tm.Sampler(A2, b2, latency=0)
    chains = np.arange(20)
    trace, out = s2.test_trace(np.tile(x2, (20, 1)), 12, seed=42, chains=chains)
    check_trace(A2, b2, trace, 42, chains, projection=1 if s2.profile()["oz_guard_ratio"] <= 16 else 2)
    assert s2.stats()["rejections"] == 0


@pytest.mark.parametrize("latency", [0, 1, "warp"])
def test_degenerate_inputs(latency):  # "warp": options.warp_mode = 1
    kw = dict(warp_mode=1) if latency == "warp" else dict(latency=latency)
    """n_iter = 0, one chain, one dimension, no active constraint (every arc inactive:
    the whole ellipse, L = 2 pi), and a polytope whose every constraint is active at
    every step (orthant) -- on both execution paths."""
    A, b, x0 = synth.make_instance(3, m=40, d=7)
    s = tm.Sampler(A, b, **kw)
    X0 = np.tile(x0, (3, 1))
    out = s.sample(X0, 0, seed=1)
    assert np.array_equal(out, X0) and s.stats()["steps"] == 0
    # one chain, one dimension: N(0,1) on [-1, 3]
    A1, b1, x1 = synth.one_dim((-1.0, 3.0))
    s1 = tm.Sampler(A1, b1, **kw)
    o1 = s1.sample(x1[None, :], 5, seed=2)
    for t in range(5):
        xn, _ = oracle.step(A1, b1, x1, 2, t, 0)
        x1 = xn
    assert np.allclose(o1[0], x1, rtol=1e-12, atol=1e-12)
    # no active constraint: b far outside the reachable ellipse
    Ab = A.copy()
    bb = np.full(40, 1e6)
    s2 = tm.Sampler(Ab, bb, **kw, record=0)
    X = np.tile(x0, (4, 1))
    Xn = s2.sample(X, 1, seed=3)
    for c in range(4):
        xn, _ = oracle.step(Ab, bb, X[c], 3, 0, c)
        assert np.allclose(Xn[c], xn, rtol=1e-12, atol=1e-12)
    assert s2.stats()["rejections"] == 0
