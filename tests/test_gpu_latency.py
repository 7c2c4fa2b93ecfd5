"""The latency mode (options.latency = 1, latency.cu): one thread-block cluster per
chain runs every iteration in one launch.  Parity with the oracle step by step
(north_star bar: next iterate within 1e-10 relative), agreement with the default
path over many iterations, moments, the paper's S4.2 instances and the
orthant closed form."""
import math

import numpy as np
import pytest

import oracle
import paper_2407_10449_b200 as tm
from paper_2407_10449_b200 import synth
from test_gpu_step import step_exemption

pytestmark = pytest.mark.gpu
REL = 1e-10


@pytest.mark.parametrize("k,kw,C", [(3, dict(m=300, d=150), 10), (5, dict(m=700, d=300), 3),
                                    (4, dict(m=6000, d=20), 5), (1, dict(), 16)])
def test_latency_step_parity_with_oracle(k, kw, C):
    A, b, x0 = synth.make_instance(k, **kw)
    cfg = synth.CONFIGS[k]
    s = tm.Sampler(A, b, latency=1, record=0)
    X = np.tile(x0, (C, 1))
    log = []
    for t in range(25):  # one iteration per call: x_t -> x_{t+1}
        Xn = s.sample(X, 1, seed=cfg.chain_seed)
        for c in range(C):
            xn, o = oracle.step(A, b, X[c], cfg.chain_seed, t, c)
            err = np.max(np.abs(Xn[c] - xn))
            if err > REL * max(1.0, np.max(np.abs(xn))):
                # the latency kernel's dot products are FP64 (P from a fresh A x each call)
                why = step_exemption(A, b, X[c], o, projection=2,
                                     gpu_accept=not np.array_equal(Xn[c], X[c]))
                assert why is not None, (t, c, err)
                log.append((t, c, err, why))
            assert np.max(A @ Xn[c] - b) <= 0.0
        X = Xn
    print("exempt steps", log)
    assert s.stats()["rejections"] == 0


def test_latency_matches_default_path():
    """Same RNG counters and readings; the dot products sum in another order, so the
    trajectories agree to rounding at first and drift apart slowly (the map x -> x'
    amplifies differences through the arc endpoints): 20 iterations at 1e-9, and a
    long run only statistically (test_latency_orthant_moments)."""
    A, b, x0 = synth.make_instance(3, m=400, d=120)
    C, T = 12, 20
    X0 = np.tile(x0, (C, 1))
    ref = tm.Sampler(A, b, latency=0).sample(X0, T, seed=3)
    lat = tm.Sampler(A, b, latency=1).sample(X0, T, seed=3)
    assert np.max(np.abs(lat - ref)) <= 1e-9 * max(1.0, np.max(np.abs(ref)))


def test_latency_moments_and_counters():
    A, b, x0 = synth.make_instance(3, m=200, d=40)
    C, T = 7, 60
    s = tm.Sampler(A, b, latency=1, burn_in=10, thin=3)
    X = np.tile(x0, (C, 1))
    s.sample(X, T, seed=8)
    sm, sq, n = s.moments()
    # the same iterates one call at a time (the per-step path of the same mode)
    s2 = tm.Sampler(A, b, latency=1, record=0)
    Y = np.tile(x0, (C, 1))
    acc, acc2, cnt = np.zeros(40), np.zeros(40), 0
    for t in range(T):
        Y = s2.sample(Y, 1, seed=8)
        if t >= 10 and (t - 10) % 3 == 0:
            acc += Y.sum(0)
            acc2 += (Y ** 2).sum(0)
            cnt += C
    assert n == cnt
    assert np.allclose(sm, acc, rtol=1e-9, atol=1e-9)
    assert np.allclose(sq, acc2, rtol=1e-9, atol=1e-9)
    assert s.stats()["steps"] == C * T and s.stats()["rejections"] == 0


@pytest.mark.parametrize("d,chains", [(300, 1), (300, 10), (1000, 10), (2000, 10), (4000, 1)])
def test_latency_section_4_2_instances(d, chains):
    A, b, x0 = synth.paper_random(d, seed=d)
    s = tm.Sampler(A, b, latency=1)
    out = s.sample(np.tile(x0, (chains, 1)), 100, seed=42)
    assert s.stats()["rejections"] == 0
    assert np.max(out @ A.T - b) <= 0.0
    # step parity along the latency path's own trajectory (one iteration per call)
    s1 = tm.Sampler(A, b, latency=1, record=0)
    X = np.tile(x0, (chains, 1))
    for t in range(8):
        Xn = s1.sample(X, 1, seed=42)
        for c in range(chains):
            xn, _ = oracle.step(A, b, X[c], 42, t, c)
            assert np.max(np.abs(Xn[c] - xn)) <= REL * max(1.0, np.max(np.abs(xn)))
        X = Xn


def test_latency_orthant_moments():
    A, b, x0 = synth.make_instance(2)
    s = tm.Sampler(A, b, latency=1, burn_in=15000)  # the default path's protocol (slow mixing)
    s.sample(np.tile(x0, (256, 1)), 20000, seed=102)
    sm, sq, n = s.moments()
    mean, var = sm / n, sq / n - (sm / n) ** 2
    assert abs(mean.mean() - math.sqrt(2 / math.pi)) < 0.01
    assert abs(var.mean() - (1 - 2 / math.pi)) < 0.01


def test_latency_overflow_falls_back_to_default_path():
    """More live arcs in an iteration than CTA 0 holds (capacity forced down by the
    test hook): the call reruns on the default path from the same start, so the
    result, moments and counters equal the default path's bitwise."""
    A, b, x0 = synth.paper_random(300, seed=300)
    C, T = 10, 40
    X0 = np.tile(x0, (C, 1))
    ref_s = tm.Sampler(A, b, latency=0, burn_in=5)
    ref = ref_s.sample(X0, T, seed=42)
    s = tm.Sampler(A, b, latency=1, burn_in=5)
    s.test_latency_cap(1)  # some iteration of S4.2 at d = 300 has more than one live arc
    out = s.sample(X0, T, seed=42)
    pr = s.profile()
    assert pr["latency_calls"] == 1 and pr["latency_fallbacks"] == 1
    assert np.array_equal(out, ref)
    for a, r in zip(s.moments(), ref_s.moments()):
        assert np.array_equal(np.asarray(a), np.asarray(r))
    assert s.stats() == ref_s.stats()
    # capacity back to automatic (m): no fallback
    s.test_latency_cap(0)
    s.reset_stats()
    s.sample(X0, T, seed=42)
    assert s.profile()["latency_fallbacks"] == 0 and s.profile()["latency_calls"] == 1


def test_latency_auto_selection():
    """options.latency = 2: latency mode for at most SMs / 2 chains, else the default
    path (bitwise the default path's result)."""
    import torch
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    A, b, x0 = synth.make_instance(3, m=300, d=100)
    few = tm.Sampler(A, b, latency=2)
    few.sample(np.tile(x0, (10, 1)), 5, seed=1)
    assert few.profile()["latency_calls"] == 1
    C = sms // 2 + 1
    X0 = np.tile(x0, (C, 1))
    many = tm.Sampler(A, b, latency=2)
    out = many.sample(X0, 5, seed=1)
    assert many.profile()["latency_calls"] == 0
    assert np.array_equal(out, tm.Sampler(A, b, latency=0).sample(X0, 5, seed=1))
    # the cost model declines it when every chain would stream a large A from HBM
    # (d = m = 4000, 32 chains: ~0.56 ms vs ~0.17 ms per iteration measured)
    A4, b4, x4 = synth.paper_random(4000, seed=4000)
    big = tm.Sampler(A4, b4)
    big.sample(np.tile(x4, (32, 1)), 1, seed=1)
    assert big.profile()["latency_calls"] == 0
    one = tm.Sampler(A4, b4)
    one.sample(np.tile(x4, (1, 1)), 1, seed=1)
    assert one.profile()["latency_calls"] == 1


def test_auto_path_is_shard_invariant_with_total_chains():
    """options.latency = 2 (default) decides from the JOB's chain count
    (options.total_chains), so a job just above SMs / 2 chains split into shards below it
    takes the default path on every shard, bitwise equal to the unsharded run."""
    import torch
    from paper_2407_10449_b200 import dist as tdist
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    A, b, x0 = synth.make_instance(3, m=300, d=100)
    C = sms // 2 + 26
    X0 = np.tile(x0, (C, 1))
    full_s = tm.Sampler(A, b)
    full = full_s.sample(X0, 12, seed=5)
    assert full_s.profile()["latency_calls"] == 0
    parts = []
    for r in range(2):
        opts, n = tdist.shard_options(C, r, 2)
        s = tm.Sampler(A, b, **opts)
        o = opts["chain_offset"]
        parts.append(s.sample(X0[o:o + n], 12, seed=5))
        assert s.profile()["latency_calls"] == 0
    assert np.array_equal(np.concatenate(parts), full)
    # without total_chains a shard of <= SMs / 2 chains decides for itself (latency mode)
    lone = tm.Sampler(A, b, chain_offset=0)
    lone.sample(X0[: C // 2], 12, seed=5)
    assert lone.profile()["latency_calls"] == 1


# ---------------------------------------------------------------- FP32 (NEXT-2)
# options.precision = 1: the paper's single precision with S3.3's trimming and
# safeguard.  Parity with the FP64 oracle is statistical: the paper's own
# S4.1 table and rejection rate, the orthant closed form, and the
# first step against the oracle to FP32 accuracy.
EPS32 = 1e-5


def _trunc_normal_moments(lo, hi):
    phi = lambda z: math.exp(-0.5 * z * z) / math.sqrt(2 * math.pi)
    if lo > 0:
        Z = 0.5 * (math.erfc(lo / math.sqrt(2)) - math.erfc(hi / math.sqrt(2)))
    else:
        Z = 0.5 * (math.erf(hi / math.sqrt(2)) - math.erf(lo / math.sqrt(2)))
    mu = (phi(lo) - phi(hi)) / Z
    return mu, 1.0 + (lo * phi(lo) - hi * phi(hi)) / Z - mu * mu


def test_fp32_first_step_close_to_oracle():
    A, b, x0 = synth.paper_random(300, seed=300)
    C = 10
    s = tm.Sampler(A, b, precision=1, trim_eps=EPS32, record=0)
    X = np.tile(x0, (C, 1))
    Xn = s.sample(X, 1, seed=42)
    assert s.profile()["latency_calls"] == 1
    for c in range(C):
        xn, _ = oracle.step(A, b, X[c], 42, 0, c, eps=EPS32)
        assert np.max(np.abs(Xn[c] - xn)) <= 1e-3 * max(1.0, np.max(np.abs(xn)))


@pytest.mark.parametrize("interval,max_rej", [((-1.0, 3.0), 20), ((15.0, 16.0), 200)])
def test_fp32_section_4_1_protocol(interval, max_rej):
    """2000 chains, burn-in 500, thinning 10, 1e5 samples in FP32: moments
    within 0.01 of the closed form; rejections at most 0.01 % of the 2e6 steps (the
    paper saw 0 on [-1, 3] and 8 on [15, 16])."""
    A, b, x0 = synth.one_dim(interval)
    s = tm.Sampler(A, b, precision=1, trim_eps=EPS32, burn_in=500, thin=10)
    out = s.sample(np.tile(x0, (2000, 1)), 1000, seed=2024)
    sm, sq, n = s.moments()
    assert n == 100000
    mu, var = _trunc_normal_moments(*interval)
    m1 = sm[0] / n
    assert abs(m1 - mu) < 0.01 and abs(sq[0] / n - m1 * m1 - var) < 0.01
    st = s.stats()
    assert st["steps"] == 2_000_000 and st["rejections"] <= max_rej, st
    assert np.all(out >= interval[0] - 1e-5) and np.all(out <= interval[1] + 1e-5)


def test_fp32_orthant_moments():
    A, b, x0 = synth.make_instance(2)
    s = tm.Sampler(A, b, precision=1, trim_eps=EPS32, burn_in=15000)
    s.sample(np.tile(x0, (256, 1)), 20000, seed=102)
    sm, sq, n = s.moments()
    mean, var = sm / n, sq / n - (sm / n) ** 2
    assert abs(mean.mean() - math.sqrt(2 / math.pi)) < 0.01
    assert abs(var.mean() - (1 - 2 / math.pi)) < 0.01


@pytest.mark.parametrize("d,chains", [(1000, 10), (4000, 1)])
def test_fp32_section_4_2_no_rejections(d, chains):
    """S4.2 in FP32: the paper saw no safeguard rejection in high dimension."""
    A, b, x0 = synth.paper_random(d, seed=d)
    s = tm.Sampler(A, b, precision=1, trim_eps=EPS32)
    out = s.sample(np.tile(x0, (chains, 1)), 200, seed=42)
    assert s.stats()["rejections"] == 0
    slack = out @ A.T - b
    assert np.max(slack) <= 1e-4 * np.max(np.abs(A @ x0))  # feasible to FP32 rounding


def test_fp32_throughput_path_section_4_1():
    """precision = 1 on the throughput path (latency = 0: 2000 chains, int8 projection at
    4 digits, FP32-class): the paper's S4.1 protocol and table."""
    for interval, max_rej in (((-1.0, 3.0), 20), ((15.0, 16.0), 200)):
        A, b, x0 = synth.one_dim(interval)
        s = tm.Sampler(A, b, precision=1, latency=0, trim_eps=EPS32, burn_in=500, thin=10)
        s.sample(np.tile(x0, (2000, 1)), 1000, seed=2024)
        assert s.profile()["latency_calls"] == 0
        sm, sq, n = s.moments()
        mu, var = _trunc_normal_moments(*interval)
        m1 = sm[0] / n
        assert abs(m1 - mu) < 0.01 and abs(sq[0] / n - m1 * m1 - var) < 0.01
        assert s.stats()["rejections"] <= max_rej, s.stats()


def test_fp32_throughput_path_steps_close_to_oracle():
    """Every traced step of the FP32-class throughput path against the FP64 oracle
    step from the same state (same nu, u, trim): the 4-digit projection's ~1e-8
    relative error moves the arc endpoints and the iterate by far less than 1e-5."""
    A, b, x0 = synth.make_instance(3, m=300, d=70)
    C, T = 150, 6
    s = tm.Sampler(A, b, precision=1, latency=0, trim_eps=EPS32)
    chains = np.array([0, 77, 149])
    trace, out = s.test_trace(np.tile(x0, (C, 1)), T, seed=103, chains=chains)
    for it in range(T):
        for k, c in enumerate(chains):
            xn, _ = oracle.step(A, b, trace[it, k], 103, it, int(c), eps=EPS32)
            assert np.max(np.abs(trace[it + 1, k] - xn)) <= 1e-5 * max(1.0, np.max(np.abs(xn)))
    assert np.max(out @ A.T - b) <= 1e-6


def test_fp32_affine_on_throughput_path():
    """App. A with precision = 1 runs on the throughput path: x ~ N(2, 4) on [1, 5]."""
    s = tm.Sampler(np.array([[1.0], [-1.0]]), np.array([5.0, -1.0]), mu=np.array([2.0]),
                   L=np.array([[2.0]]), burn_in=100, precision=1, trim_eps=EPS32)
    out = s.sample(np.full((2000, 1), 3.0), 600, seed=77)
    sm, sq, n = s.moments()
    mu_u, var_u = _trunc_normal_moments(-0.5, 1.5)
    m1 = sm[0] / n
    assert abs(m1 - (2 + 2 * mu_u)) < 0.01
    assert abs(sq[0] / n - m1 * m1 - 4 * var_u) < 0.03
    assert np.all(out >= 1.0 - 1e-6) and np.all(out <= 5.0 + 1e-6)



def test_latency_shard_invariance_and_resume_bitwise():
    """A row's dot product has a fixed order whichever CTA (and cluster size) holds it,
    so the latency mode is bitwise invariant to the chain split (multi-GPU sharding:
    chain_offset) and a call split at a multiple of recompute_every resumes bitwise."""
    A, b, x0 = synth.paper_random(300, seed=301)
    C, T = 10, 64
    X0 = np.tile(x0, (C, 1))
    full = tm.Sampler(A, b, latency=1).sample(X0, T, seed=5)
    h1 = tm.Sampler(A, b, latency=1, chain_offset=0).sample(X0[:3], T, seed=5)
    h2 = tm.Sampler(A, b, latency=1, chain_offset=3).sample(X0[3:], T, seed=5)
    assert np.array_equal(np.concatenate([h1, h2]), full)
    s = tm.Sampler(A, b, latency=1)
    a = s.sample(X0, 32, seed=5)
    a = s.sample(a, 32, seed=5)
    assert np.array_equal(a, full)
    # FP32 too
    f = tm.Sampler(A, b, precision=1, trim_eps=1e-5).sample(X0, T, seed=5)
    g1 = tm.Sampler(A, b, precision=1, trim_eps=1e-5, chain_offset=0).sample(X0[:4], T, seed=5)
    g2 = tm.Sampler(A, b, precision=1, trim_eps=1e-5, chain_offset=4).sample(X0[4:], T, seed=5)
    assert np.array_equal(np.concatenate([g1, g2]), f)


@pytest.mark.parametrize("case", range(12))
def test_latency_random_shapes_vs_oracle(case):
    """Ragged shapes through the latency mode (forced): d, m, C drawn per case, unit
    and unnormalised rows, one iteration per call against the oracle step."""
    rng = np.random.default_rng(1000 + case)
    d = int(rng.integers(1, 90))
    m = int(rng.integers(1, 400))
    C = int(rng.integers(1, 40))
    A = rng.standard_normal((m, d))
    if case % 2:
        A /= np.linalg.norm(A, axis=1, keepdims=True)
    b = rng.uniform(0.05, 2.0, m)
    x0 = np.zeros(d)
    s = tm.Sampler(A, b, latency=1, record=0)
    if case % 3 == 0:
        s.test_latency_grid(1)  # the cooperative-grid variant
    X = np.tile(x0, (C, 1))
    for t in range(4):
        Xn = s.sample(X, 1, seed=case)
        assert s.profile()["latency_calls"] == t + 1
        for c in range(C):
            xn, _ = oracle.step(A, b, X[c], case, t, c)
            assert np.max(np.abs(Xn[c] - xn)) <= REL * max(1.0, np.max(np.abs(xn))), (d, m, C, t, c)
        X = Xn


@pytest.mark.parametrize("d,m,C,prec", [(60, 200, 1, 0), (150, 700, 3, 0), (1000, 1000, 1, 0), (300, 300, 2, 1)])
def test_latency_grid_variant(d, m, C, prec):
    """The cooperative-grid variant (SMs / C CTAs per chain, exchanges through global
    scratch and grid barriers): oracle steps (FP64) and bitwise equality with the
    cluster variant (each row's dot product has one fixed order in both)."""
    A, b, x0 = synth.paper_random(d, seed=d + m) if d == m else synth.make_instance(3, m=m, d=d)
    kw = dict(latency=1, record=0, precision=prec, trim_eps=1e-5 if prec else 0.0)
    g = tm.Sampler(A, b, **kw)
    g.test_latency_grid(1)
    c = tm.Sampler(A, b, **kw)
    c.test_latency_grid(-1)
    X = np.tile(x0, (C, 1))
    for t in range(5):
        Xg = g.sample(X, 1, seed=17)
        Xc = c.sample(X, 1, seed=17)
        assert np.array_equal(Xg, Xc), t
        if prec == 0:
            for k in range(C):
                xn, _ = oracle.step(A, b, X[k], 17, t, k)
                assert np.max(np.abs(Xg[k] - xn)) <= REL * max(1.0, np.max(np.abs(xn)))
        X = Xg
    long_g = g.sample(X, 40, seed=17)
    long_c = c.sample(X, 40, seed=17)
    assert np.array_equal(long_g, long_c)
    assert g.profile()["latency_calls"] == 6
