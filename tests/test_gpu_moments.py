"""a9: tmvn_get_moments against the oracle's moment sums.

The paper's output is the moment table of S4.1: sums of x
and x^2 over the recorded iterates (burn-in, thinning).  The oracle
(`oracle.run`) records the same iterates of the same chains (same Philox
counters, C12) and sums them in chain order; here the GPU's sums are compared
with it elementwise, in u-space, in x-space under App. A's change of variable
(P:898-904), with burn-in/thinning, across several tmvn_sample calls, on both
execution paths.

Bar: the north_star per-step bar (1e-10 relative to max(1, |x|_inf)) summed
over the n recorded iterates: |d sum_j| <= 1e-10 n M and |d sumsq_j| <=
2e-10 n M^2 with M = max(1, sqrt(max_j sumsq_j)) >= every recorded |x|_inf
(Cauchy-Schwarz); the record counts are equal exactly.
"""
import numpy as np
import pytest

import oracle
import paper_2407_10449_b200 as tm
from paper_2407_10449_b200 import synth

pytestmark = pytest.mark.gpu
REL = 1e-10


def assert_moments_equal(gpu, ref):
    sm, sq, n = gpu
    assert n == ref["n_rec"], (n, ref["n_rec"])
    M = max(1.0, float(np.sqrt(np.max(ref["sumsq"]))))
    err1 = float(np.max(np.abs(sm - ref["sum"])))
    err2 = float(np.max(np.abs(sq - ref["sumsq"])))
    assert err1 <= REL * n * M, (err1, REL * n * M)
    assert err2 <= 2 * REL * n * M * M, (err2, 2 * REL * n * M * M)
    return err1 / (n * M), err2 / (n * M * M)


@pytest.mark.parametrize("kw", [dict(), dict(projection=2), dict(recompute_every=1)])
def test_moments_u_space_burn_in_thin_vs_oracle(kw):
    """Throughput path (default options, int8 projection; FP64 DMMA; K = 1), two calls
    (the second resumes mid-way through the thinning pattern), against oracle.run of the
    same chains from the same start.  Short: trajectories from a common start separate
    at the rate the map amplifies rounding (measured ~3e-9 after 44 iterations), so
    whole-run agreement at 1e-10 only holds for a few iterations; the long run is
    test_moments_long_run_vs_oracle_steps."""
    A, b, x0 = synth.make_instance(3, m=300, d=150)
    C, T1, T2, seed, burn, thin = 200, 5, 7, 31, 2, 3
    X0 = np.tile(x0, (C, 1))
    s = tm.Sampler(A, b, latency=0, burn_in=burn, thin=thin, **kw)
    X = s.sample(X0, T1, seed=seed)
    X = s.sample(X, T2, seed=seed)
    ref = oracle.run(A, b, X0, T1 + T2, seed=seed, burn_in=burn, thin=thin)
    assert np.max(np.abs(X - ref["X"])) <= REL * max(1.0, np.max(np.abs(ref["X"])))
    print("moment errors (scaled)", assert_moments_equal(s.moments(), ref))
    assert s.stats()["recorded"] == ref["n_rec"]


@pytest.mark.parametrize("kw", [dict(), dict(recompute_every=1)])
def test_moments_long_run_vs_oracle_steps(kw):
    """44 iterations (two calls, burn-in 7, thinning 3): every recorded iterate is
    recomputed by the oracle from the GPU's previous iterate (oracle.step, P6), and the
    library's moment sums must equal the sums of those oracle iterates at the per-step
    bar; the record count equals oracle.run's."""
    A, b, x0 = synth.make_instance(3, m=300, d=150)
    C, T1, T2, seed, burn, thin = 200, 24, 20, 31, 7, 3
    X0 = np.tile(x0, (C, 1))
    s = tm.Sampler(A, b, latency=0, burn_in=burn, thin=thin, **kw)
    chains = np.arange(C)
    tr1, X = s.test_trace(X0, T1, seed=seed, chains=chains)
    tr2, X = s.test_trace(X, T2, seed=seed, chains=chains)
    trace = np.concatenate([tr1, tr2[1:]])  # (T1 + T2 + 1) x C x d, row t = x_t
    rec = [t for t in range(T1 + T2) if t >= burn and (t - burn) % thin == 0]
    sm, sq = np.zeros(A.shape[1]), np.zeros(A.shape[1])
    for t in rec:  # iteration t records x_{t+1}, here the oracle's step from the GPU's x_t
        for c in range(C):
            xn, _ = oracle.step(A, b, trace[t, c], seed, t, c)
            sm += xn
            sq += xn * xn
    ref_n = oracle.run(A, b, X0[:1], T1 + T2, seed=seed, burn_in=burn, thin=thin)["n_rec"] * C
    print("moment errors (scaled)",
          assert_moments_equal(s.moments(), dict(sum=sm, sumsq=sq, n_rec=ref_n)))


def test_moments_chain_offset_and_record_off():
    """Chains of a shard (chain_offset) record the global chains' iterates; record = 0
    records nothing."""
    A, b, x0 = synth.make_instance(2, m=60, d=60)
    C, T, seed = 150, 30, 77
    X0 = np.tile(x0, (C, 1))
    s = tm.Sampler(A, b, latency=0, chain_offset=1000, burn_in=4)
    s.sample(X0, T, seed=seed)
    ref = oracle.run(A, b, X0, T, seed=seed, chain_offset=1000, burn_in=4)
    assert_moments_equal(s.moments(), ref)
    s0 = tm.Sampler(A, b, latency=0, record=0)
    s0.sample(X0, 5, seed=seed)
    sm, sq, n = s0.moments()
    assert n == 0 and not np.any(sm) and not np.any(sq)


def test_moments_latency_mode_vs_oracle():
    """The latency mode (one cluster per chain) records in shared memory and adds once
    per call: the same sums."""
    A, b, x0 = synth.make_instance(3, m=200, d=40)
    C, T, seed = 7, 60, 8
    X0 = np.tile(x0, (C, 1))
    s = tm.Sampler(A, b, latency=1, burn_in=10, thin=3)
    s.sample(X0, T, seed=seed)
    assert s.profile()["latency_calls"] == 1
    ref = oracle.run(A, b, X0, T, seed=seed, burn_in=10, thin=3)
    assert_moments_equal(s.moments(), ref)


@pytest.mark.parametrize("projection", [0, 2])
def test_moments_x_space_affine_vs_oracle(projection):
    """App. A: N(mu, L L^T) truncated; the library runs u-space chains on
    A' = A L, b' = b - A mu and records x = L u + mu.  The oracle whitens with its own
    forward substitution and records unwhitened iterates (orc_run with mu, L)."""
    d, m = 24, 40
    L, mu = synth.random_spd_factor(d, seed=5)
    rng = np.random.default_rng(6)
    A = rng.standard_normal((m, d))
    x_start = mu + 0.05 * rng.standard_normal(d)
    b = A @ x_start + rng.uniform(0.3, 1.5, m)
    C, T, seed, burn, thin = 130, 30, 12, 5, 2
    s = tm.Sampler(A, b, mu=mu, L=L, projection=projection, burn_in=burn, thin=thin)
    X = s.sample(np.tile(x_start, (C, 1)), T, seed=seed)
    Aw, bw = oracle.whiten(A, b, mu, L)
    u0 = oracle.whiten_point(x_start, mu, L)
    ref = oracle.run(Aw, bw, np.tile(u0, (C, 1)), T, seed=seed, burn_in=burn, thin=thin, mu=mu, L=L)
    xo = np.array([oracle.unwhiten_point(u, mu, L) for u in ref["X"]])
    assert np.max(np.abs(X - xo)) <= REL * max(1.0, np.max(np.abs(xo)))
    print("moment errors (scaled)", assert_moments_equal(s.moments(), ref))
