"""The int8 Ozaki-split projection on tcgen05 (options.projection = 1, gemm_i8.cu).

Pins, independent of the FP64 path:
- exactness: dyadic inputs whose fixed-point digits fit in the kept diagonals
  give the exact integer product (catches digit, signedness, layout and
  accumulate-flag errors bit for bit);
- the stated error bound of include/tmvn.h against an extended-precision
  (x87 long double) product, over ragged shapes, K up to 4096, rows with
  scales over 12 decades and S = 6, 7, 8;
- the full ESS step and the production loop against the CPU oracle at the
  north_star bar (1e-10 relative), sharding invariance, and no rejections.
"""
import numpy as np
import pytest

import oracle
import paper_2407_10449_b200 as tm
from paper_2407_10449_b200 import synth
from test_gpu_step import REL, check_trace, compare_step, ozaki_qbound

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("slices", [4, 6, 7, 8])
@pytest.mark.parametrize("R,S,K", [(1, 1, 1), (130, 200, 100), (64, 128, 32), (257, 129, 1000)])
def test_ozaki_exact_on_dyadic_inputs(slices, R, S, K):
    rng = np.random.default_rng(R * 7 + S + K)
    Xi = rng.integers(-2**10, 2**10, size=(R, K))
    Wi = rng.integers(-2**12, 2**12, size=(S, K))
    Wi[:, 0] = 2**12 - 1  # every row has a large entry: short digit expansions
    Xi[0, 0] = -2**10
    X = Xi / 2.0**10
    rowscale = 2.0 ** rng.integers(-30, 30, size=S)
    W = (Wi / 2.0**12) * rowscale[:, None]
    out = tm.test_ozaki_gemm(X, W, slices=slices)
    ref = (Xi @ Wi.T).astype(np.float64) * 2.0**-22 * rowscale[None, :]
    assert np.array_equal(out, ref)


@pytest.mark.parametrize("slices", [4, 6, 7, 8])
@pytest.mark.parametrize("R,S,K", [(200, 300, 1000), (65, 131, 4096), (128, 256, 37)])
def test_ozaki_within_stated_bound(slices, R, S, K):
    rng = np.random.default_rng(R + S + K + slices)
    X = rng.standard_normal((R, K)) * 2.0  # nu-like
    W = rng.standard_normal((S, K)) * 10.0 ** rng.uniform(-6, 6, size=(S, 1))
    W[::7, ::3] = 0.0
    out = tm.test_ozaki_gemm(X, W, slices=slices)
    ref = X.astype(np.longdouble) @ W.T.astype(np.longdouble)
    ex = np.frexp(np.max(np.abs(X)))[1]
    e = np.frexp(np.max(np.abs(W), axis=1))[1]
    bound = 2.0 ** (e + ex)[None, :] * K * (slices + 1) * 2.0 ** (2 - 8 * slices) \
        + 2.0**-51 * np.abs(ref).astype(np.float64)
    err = np.abs(out - ref).astype(np.float64)
    assert np.all(err <= bound), float(np.max(err / bound))
    # FP64-class at S = 7, 8: far below the bound's worst case
    if slices >= 7:
        dmma = np.abs(tm.test_gemm(X, W) - ref).astype(np.float64)
        assert np.max(err) <= 64 * np.max(dmma) + 1e-300


@pytest.mark.parametrize("name,k,kw,C", [
    ("orthant", 2, dict(), 130),
    ("random", 3, dict(m=300, d=150), 131),
    ("heavy", 4, dict(m=6000, d=20), 37),
    ("boxscale", 5, dict(m=700, d=300), 129),
])
def test_ozaki_step_parity(name, k, kw, C):
    A, b, x0 = synth.make_instance(k, **kw)
    cfg = synth.CONFIGS[k]
    s = tm.Sampler(A, b, latency=0, projection=1)
    X = np.tile(x0, (C, 1))
    r = oracle.run(A, b, X[: min(C, 16)], 30, seed=cfg.chain_seed + 1000)
    X[: r["X"].shape[0]] = r["X"]
    rng = np.random.default_rng(k)
    log = []
    for t in (0, 9):
        g = s.test_step(X, cfg.chain_seed, t, seg_cap=64)
        fp64 = 2 * A.shape[1] * 2.0**-53 * (np.abs(g["nu"]) @ np.abs(A).T)  # numpy's own rounding
        assert np.all(np.abs(g["q"] - (g["nu"] @ A.T)) <= ozaki_qbound(A, g["q"]) + fp64)
        chains = rng.choice(C, size=min(C, 20), replace=False)
        assert compare_step(A, b, X, g, cfg.chain_seed, t, chains, log=log, projection=1) <= 2, log
        X = np.where(g["accept"][:, None], g["x_next"], X)
    s.close()


def test_ozaki_production_loop_parity_and_sharding():
    A, b, x0 = synth.make_instance(3, m=400, d=120)
    C, T = 200, 70
    s = tm.Sampler(A, b, latency=0, projection=1)
    chains = np.array([0, 1, 63, 64, 199])
    trace, out = s.test_trace(np.tile(x0, (C, 1)), T, seed=103, chains=chains)
    log = []
    check_trace(A, b, trace, 103, chains, projection=1, log=log)
    print("exempt steps", log)
    assert s.stats()["rejections"] == 0
    # sharding by chain_offset is bitwise invariant (per-element integer MMA, fixed Horner)
    X0 = np.tile(x0, (C, 1))
    full = tm.Sampler(A, b, latency=0, projection=1).sample(X0, 40, seed=9)
    h1 = tm.Sampler(A, b, latency=0, projection=1, chain_offset=0).sample(X0[:77], 40, seed=9)
    h2 = tm.Sampler(A, b, latency=0, projection=1, chain_offset=77).sample(X0[77:], 40, seed=9)
    assert np.array_equal(np.concatenate([h1, h2]), full)


def test_ozaki_full_size_config3_sampled():
    """BASELINE config 3 at full size through the int8 projection (bench launch config)."""
    A, b, x0 = synth.make_instance(3)
    C = 4096
    s = tm.Sampler(A, b, latency=0, projection=1)
    X = s.sample(np.tile(x0, (C, 1)), 20, seed=103)
    assert s.stats()["rejections"] == 0
    g = s.test_step(X, 103, 20, seg_cap=64)
    rng = np.random.default_rng(0)
    chains = np.concatenate([[0, C - 1], rng.choice(C, size=14, replace=False)])
    log = []
    assert compare_step(A, b, X, g, 103, 20, chains, log=log, projection=1) <= 1, log
    s.close()


def test_ozaki_rejects_large_d():
    A = np.ones((2, 4097)) / 100.0
    s = tm.Sampler(A, np.ones(2), latency=0)
    with pytest.raises(tm.TmvnError):
        s.set_options(projection=1)


def test_dynamic_range_guard_under_default_options():
    """VERDICT r1 item 6 / App. A.  The automatic projection takes the int8
    split only when its stated bound is within 16x the FP64 DMMA bound on every row
    (tmvn_profile.oz_guard_ratio): rows whose entries span 1e-8..1, and A' = A L for an
    ill-conditioned L, fall back to DMMA; unit Gaussian rows keep int8.  Either way the
    step matches the oracle at the north_star bar (1e-10) under default options."""
    rng = np.random.default_rng(11)
    m, d, C, seed = 90, 60, 130, 21
    A = rng.standard_normal((m, d)) * 10.0 ** rng.uniform(-8, 0, size=(m, d))
    b = rng.uniform(0.3, 1.0, m)
    x0 = np.zeros(d)
    s = tm.Sampler(A, b, warp_mode=0)  # the throughput path (small jobs default to the warp mode)
    pr = s.profile()
    assert pr["oz_guard_ratio"] > 16
    X = np.tile(x0, (C, 1))
    r = oracle.run(A, b, X[:16], 20, seed=seed + 1000)
    X[:16] = r["X"]
    log = []
    for t in (0, 7):
        g = s.test_step(X, seed, t, seg_cap=64)
        assert compare_step(A, b, X, g, seed, t, range(0, C, 5), log=log, projection=2) <= 2, log
        X = np.where(g["accept"][:, None], g["x_next"], X)
    s.sample(np.tile(x0, (C, 1)), 3, seed=seed)
    assert s.profile()["projection_used"] == 2
    # unit Gaussian rows: int8
    Ag, bg, xg = synth.make_instance(3, m=90, d=60)
    sg = tm.Sampler(Ag, bg, warp_mode=0)
    assert sg.profile()["oz_guard_ratio"] <= 16
    sg.sample(np.tile(xg, (C, 1)), 3, seed=seed)
    assert sg.profile()["projection_used"] == 1
    # App. A with an ill-conditioned L = D (I + N) (cond ~ 1e4: D spans four decades, N
    # strictly lower with small entries): A' = A L spans four decades per row
    D = np.diag(10.0 ** np.linspace(-4, 0, d))
    L = D @ (np.eye(d) + np.tril(rng.standard_normal((d, d)) * 0.02, -1))
    assert np.linalg.cond(L) > 1e3
    mu = 0.1 * rng.standard_normal(d)
    x_start = mu.copy()
    bL = Ag @ x_start + rng.uniform(0.3, 1.0, m)
    sa = tm.Sampler(Ag, bL, mu=mu, L=L, record=0)
    assert sa.profile()["oz_guard_ratio"] > 16
    Aw, bw = oracle.whiten(Ag, bL, mu, L)
    X = np.tile(x_start, (C, 1))
    for t in range(5):
        Xn = sa.sample(X, 1, seed=seed)
        for c in range(0, C, 13):
            un, o = oracle.step(Aw, bw, oracle.whiten_point(X[c], mu, L), seed, t, c)
            xn = oracle.unwhiten_point(un, mu, L)
            assert np.max(np.abs(Xn[c] - xn)) <= 1e-10 * max(1.0, np.max(np.abs(xn))), (t, c)
        X = Xn
    assert sa.profile()["projection_used"] == 2
