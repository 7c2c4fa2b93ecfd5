"""Per-step parity of the full CUDA step against the oracle (P6, P7).

Each GPU step starts from the GPU's own x_t; the oracle runs Alg. 1 from the
same x_t with the same counters.  Bars (north_star): next iterate and sampled
arcs within 1e-10 relative in FP64, feasibility verdict bit-exact; exemptions
only where the paper's own conditioning argument applies (near-tangent arcs,
P:736-740; verdicts within the fp64 rounding bound of a facet) and logged.
There is no count-based allowance: a mismatch outside these readings fails.
"""
import math
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import oracle
import paper_2407_10449_b200 as tm
from paper_2407_10449_b200 import synth

pytestmark = pytest.mark.gpu
REL = 1e-10
# incremental P = A x (Eq. 1 updates between refreshes, C13): drift allowance on p
# relative to max(1, |p|_inf), SURVEY 8(c) P6 ("should be <= 1e-12 at K = 32")
DRIFT = 1e-12


def ozaki_qbound(A, q, slices=7, e_v=4):
    """Stated bound of the int8 tcgen05 projection (include/tmvn.h, options.projection = 1):
    |Q - a.v| <= 2^(e_i + e_v) d (S + 1) 2^(2 - 8S) + 2^-51 |Q| with max_j |a_ij| < 2^e_i and
    |v| < 2^e_v (e_v = 4 for nu; per chain for the refresh of P = A x)."""
    m, d = A.shape
    e = np.frexp(np.max(np.abs(A), axis=1))[1].astype(np.float64)  # max_j |a_ij| < 2^e_i
    return 2.0 ** (e + e_v) * d * (slices + 1) * 2.0 ** (2 - 8 * slices) + 2.0**-51 * np.abs(q)


def proj_bound(A, v, val, projection, slices=7, e_v=None):
    """Bound on |computed A.v - exact| for one vector v: FP64 dot products (P2) or the int8
    projection's stated bound (e_v: fixed exponent, else the one of max |v| as the refresh
    of P = X A'^T uses per chain)."""
    d = A.shape[1]
    fp64 = 2 * d * 2.0**-53 * (np.abs(A) @ np.abs(v)) + 1e-300
    if projection != 1:
        return fp64
    if e_v is None:
        mx = float(np.max(np.abs(v)))
        e_v = int(np.frexp(mx)[1]) if mx > 0 else 0
    return ozaki_qbound(A, val, slices, e_v) + fp64


def step_exemption(A, b, x, o, projection, drift=0.0, gpu_accept=None):
    """Reason a GPU step from x may differ from the oracle's beyond REL under SURVEY 8(c)'s
    readings, or None.  o: the oracle's dump for the step from x.
      * an active arc with 1 - |rho| < 1e-8 (ill-conditioned endpoint, P3);
      * an active flag decided within the rounding of p, q (|r - b| at the bound, C3/C25);
      * a safeguard verdict (C8) that differs while the oracle's tightest slack is
        within the rounding bound of P' (P6)."""
    r = np.hypot(o["p"], o["q"])
    rho = np.clip(b / np.where(r > 0, r, 1.0), -1, 1)
    if np.any(o["active"] & (1 - np.abs(rho) < 1e-8)):
        return "ill-conditioned arc"
    bp = proj_bound(A, x, o["p"], projection) + drift * max(1.0, float(np.max(np.abs(o["p"]))))
    bq = proj_bound(A, o["nu"], o["q"], projection, e_v=4)
    if np.any(np.abs(r - b) <= 8 * np.spacing(r) + 4 * (bp + bq)):
        return "active-flag tie"
    if gpu_accept is not None and bool(gpu_accept) != o["accept"]:
        xp = o["x_prop"]
        bound = float(np.max(bp + bq + 2 * A.shape[1] * 2.0**-53 * (np.abs(A) @ np.abs(xp))))
        if abs(o["max_slack"]) <= bound:
            return "verdict at facet"
    return None


def _pool():
    return ThreadPoolExecutor(max_workers=max(1, min(32, os.cpu_count() or 1)))


def check_trace(A, b, trace, seed, chains, projection=2, drift=DRIFT, log=None, chain_offset=0,
                iter_offset=0, eps=0.0):
    """P6/P7 along a production-loop trace (tmvn_test_trace): every step it -> it + 1 of
    every traced chain is recomputed by the oracle from the GPU's own x_it (ctypes releases
    the GIL: the oracle steps run in a thread pool).  A next iterate beyond REL fails unless
    step_exemption names a reading; every iterate satisfies A x <= b (fresh FP64 dot
    products, P7).  Returns the number of exempt steps (each logged)."""
    T = trace.shape[0] - 1
    jobs = [(it, k, int(c)) for it in range(T) for k, c in enumerate(chains)]

    def one(job):
        it, k, c = job
        x = trace[it, k]
        xn, o = oracle.step(A, b, x, seed, iter_offset + it, chain_offset + c, eps=eps)
        err = float(np.max(np.abs(trace[it + 1, k] - xn)))
        if err <= REL * max(1.0, float(np.max(np.abs(xn)))):
            return None
        gpu_acc = not np.array_equal(trace[it + 1, k], x)
        why = step_exemption(A, b, x, o, projection, drift, gpu_accept=gpu_acc)
        return (it, c, err, why)

    with _pool() as ex:
        res = [r for r in ex.map(one, jobs) if r is not None]
    bad = [r for r in res if r[3] is None]
    assert not bad, f"unexplained step mismatches (it, chain, err): {bad[:5]}"
    if log is not None:
        log.extend(res)
    for it in range(1, T + 1):
        assert np.max(trace[it] @ A.T - b) <= 0.0, it  # P7: feasible under fresh FP64 dots
    return len(res)


def compare_step(A, b, X, g, seed, t, chains, chain_offset=0, log=None, projection=2):
    """projection: 2 = FP64 DMMA bound on q (P2), 1 = the int8 projection's stated bound."""
    m, d = A.shape
    exempt = 0
    for c in chains:
        x = X[c]
        xn, o = oracle.step(A, b, x, seed, t, chain_offset + c)
        # P1: nu within 4 ulp, u bitwise
        assert np.all(np.abs(g["nu"][c] - o["nu"]) <= 4 * np.spacing(np.abs(o["nu"])) + 1e-300)
        assert g["u"][c] == o["u"]
        # P2: projections within the dot-product rounding bound
        # (GPU - exact) + (exact - oracle): the product's own bound plus FP64's; the refresh
        # P = X A'^T runs on the same projection as Q (test_step uses the production refresh)
        bp = proj_bound(A, x, o["p"], projection)
        bq = proj_bound(A, o["nu"], o["q"], projection, e_v=4)
        assert np.all(np.abs(g["p"][c] - o["p"]) <= 2 * bp)
        assert np.all(np.abs(g["q"][c] - o["q"]) <= 2 * bq)
        # P3: arcs
        r = np.hypot(o["p"], o["q"])
        same = g["active"][c] == o["active"]
        assert np.all(np.abs(r - b)[~same] <= 8 * np.spacing(r[~same]) + 4 * (bp + bq)[~same])
        both = g["active"][c] & o["active"]
        rho = np.clip(b / np.where(r > 0, r, 1.0), -1, 1)
        well = both & (1 - np.abs(rho) >= 1e-8)
        assert np.all(np.abs(g["alpha"][c] - o["alpha"])[well] <= REL * np.maximum(1, o["alpha"][well]))
        assert np.all(np.abs(g["beta"][c] - o["beta"])[well] <= REL * np.maximum(1, o["beta"][well]))
        ill = both & ~well
        # P6: segments, theta, verdict, next iterate
        if not same.all() or ill.any():
            exempt += 1
            if log is not None:
                log.append(("ill-conditioned/tangent", c))
            continue
        ns = int(g["nseg"][c])
        assert ns == o["nseg"], (c, ns, o["nseg"])
        cap = g["seg_lo"].shape[1]
        k = min(ns, cap)
        assert np.allclose(g["seg_lo"][c, :k], o["segs"][:k, 0], rtol=REL, atol=REL)
        assert np.allclose(g["seg_hi"][c, :k], o["segs"][:k, 1], rtol=REL, atol=REL)
        assert abs(g["L"][c] - o["L"]) <= REL * max(1, o["L"])
        assert abs(g["theta"][c] - o["theta"]) <= REL * max(1, abs(o["theta"]))
        if bool(g["accept"][c]) != o["accept"]:
            # exempt only if the oracle's tightest slack is within the rounding bound
            xp = o["x_prop"]
            bound = 2 * d * 2.0**-53 * np.max(np.abs(A) @ np.abs(xp)) + 1e-14 * max(1, np.max(np.abs(xp)))
            assert abs(o["max_slack"]) <= bound, (c, o["max_slack"], bound)
            exempt += 1
            if log is not None:
                log.append(("verdict at facet", c))
            continue
        scale = max(1.0, np.max(np.abs(xn)))
        assert np.max(np.abs(g["x_next"][c] - xn)) <= REL * scale, c
        # P7: every iterate feasible under the oracle's own dot products
        assert np.max(A @ g["x_next"][c] - b) <= 0.0 or not g["accept"][c] or \
            np.max(A @ g["x_next"][c] - b) <= 2 * d * 2.0**-53 * np.max(np.abs(A) @ np.abs(g["x_next"][c]))
    return exempt


SMALL = {
    "tiny2d": (1, dict()),
    "orthant": (2, dict()),
    "random": (3, dict(m=300, d=150)),
    "heavy": (4, dict(m=6000, d=20)),    # m > in-smem stash: global-scratch path
    "boxscale": (5, dict(m=700, d=300)),
}


@pytest.mark.parametrize("projection", [2, 1])
@pytest.mark.parametrize("name", list(SMALL))
def test_step_parity_from_start_and_along_oracle_path(name, projection):
    k, kw = SMALL[name]
    A, b, x0 = synth.make_instance(k, **kw)
    m, d = A.shape
    C = {1: 16, 2: 130, 3: 131, 4: 37, 5: 129}[k]
    cfg = synth.CONFIGS[k]
    s = tm.Sampler(A, b, latency=0, projection=projection)
    rng = np.random.default_rng(k)
    # interior points: x0, and points reached by oracle chains (stationary-ish)
    X = np.tile(x0, (C, 1))
    r = oracle.run(A, b, X[: min(C, 16)], 30, seed=cfg.chain_seed + 1000)
    X[: r["X"].shape[0]] = r["X"]
    log = []
    for t in (0, 5, 123456):
        g = s.test_step(X, cfg.chain_seed, t, seg_cap=64)
        chains = rng.choice(C, size=min(C, 24), replace=False)
        ex = compare_step(A, b, X, g, cfg.chain_seed, t, chains, log=log, projection=projection)
        assert ex <= 2, log
        X = np.where(g["accept"][:, None], g["x_next"], X)
    s.close()


def test_trace_production_loop_parity():
    """tmvn_sample's own loop (incremental P, refresh every K, fused RNG) step by step."""
    A, b, x0 = synth.make_instance(3, m=400, d=120)
    C, T = 200, 70
    for K in (32, 1):
        s = tm.Sampler(A, b, latency=0, recompute_every=K, projection=2)
        chains = np.array([0, 1, 57, 128, 199])
        trace, out = s.test_trace(np.tile(x0, (C, 1)), T, seed=103, chains=chains)
        assert np.array_equal(trace[-1], out[chains])
        log = []
        check_trace(A, b, trace, 103, chains, projection=2, log=log)
        print("exempt steps", K, log)
        st = s.stats()
        assert st["steps"] == C * T and st["rejections"] == 0
        s.close()


def test_full_size_config3_default_options_trace():
    """BASELINE config 3 at full size (d=1000, m=2000, C=4096) on the DEFAULT options --
    the path bench.py times: int8 tcgen05 projection for Q and for the P refresh every
    K = 32, incremental P between refreshes, nu drawn inside the per-chain kernel, CUDA-graph
    blocks -- traced for 80 iterations (two refreshes and graph blocks) on 16 chains spread
    over the grid, every step against the oracle from the GPU's own x_t (north_star: 1e-10).
    (Tracing launches kernel by kernel; CUDA-graph replay is bitwise equal to that,
    test_gpu_api.py::test_graph_replay_bitwise_equals_launches.)"""
    A, b, x0 = synth.make_instance(3)
    C, T = 4096, 80
    s = tm.Sampler(A, b)
    rng = np.random.default_rng(3)
    chains = np.unique(np.concatenate([[0, 1, 2047, C - 1], rng.choice(C, size=12, replace=False)]))
    trace, out = s.test_trace(np.tile(x0, (C, 1)), T, seed=103, chains=chains)
    assert np.array_equal(trace[-1], out[chains])
    log = []
    check_trace(A, b, trace, 103, chains, projection=1, log=log)
    print("exempt steps", log)
    assert s.stats()["rejections"] == 0
    assert np.max(out @ A.T - b) <= 0.0  # every chain's final iterate feasible (P7)
    s.close()


def test_full_size_config3_sampled():
    """BASELINE config 3 at full size (d=1000, m=2000, C=4096) in the bench launch config."""
    A, b, x0 = synth.make_instance(3)
    C = 4096
    s = tm.Sampler(A, b, latency=0, projection=2)
    X = s.sample(np.tile(x0, (C, 1)), 20, seed=103)
    assert s.stats()["rejections"] == 0
    g = s.test_step(X, 103, 20, seg_cap=64)
    rng = np.random.default_rng(0)
    chains = np.concatenate([[0, C - 1], rng.choice(C, size=14, replace=False)])
    log = []
    assert compare_step(A, b, X, g, 103, 20, chains, log=log) <= 1, log
    s.close()


def test_full_size_config4_sampled():
    """BASELINE config 4 (m=100000, sort-bound; arcs spill to global scratch)."""
    A, b, x0 = synth.make_instance(4)
    C = 1024
    for projection in (2, 1):
        s = tm.Sampler(A, b, latency=0, projection=projection)
        X = s.sample(np.tile(x0, (C, 1)), 5, seed=104)
        g = s.test_step(X, 104, 5, seg_cap=64)
        log = []
        assert compare_step(A, b, X, g, 104, 5, [0, 511, 1023], log=log, projection=projection) <= 1, log
        s.close()


@pytest.mark.parametrize("k,T,nchains", [(4, 6, 8), (2, 40, 16), (1, 200, 16)])
def test_full_size_default_options_trace(k, T, nchains):
    """BASELINE configs 4 (m = 100000: arcs in global scratch, the sort-bound case), 2
    (orthant: every constraint active every step; the dynamic-range guard takes DMMA for
    A = -I) and 1 (tiny 2-D: the latency mode is the automatic choice, so the throughput
    path is forced here) at full size on default options, traced and checked step by step
    against the oracle (north_star: 1e-10)."""
    A, b, x0 = synth.make_instance(k)
    cfg = synth.CONFIGS[k]
    s = tm.Sampler(A, b, latency=0)
    rng = np.random.default_rng(k)
    chains = np.unique(np.concatenate([[0, cfg.C - 1], rng.choice(cfg.C, size=nchains - 2, replace=False)]))
    trace, out = s.test_trace(np.tile(x0, (cfg.C, 1)), T, seed=cfg.chain_seed, chains=chains)
    log = []
    check_trace(A, b, trace, cfg.chain_seed, chains, projection=s.profile()["projection_used"] or 2, log=log)
    print("exempt steps", log)
    assert s.stats()["rejections"] == 0
    s.close()


def test_full_size_config5_trace():
    """BASELINE config 5 at full single-GPU size (d=4096, m=16384, C=65536; ~45 GB of
    device state) through the production loop on the default options (int8 projection,
    d = 4096 at its limit): 16 chains spread over the grid traced for 10 iterations, every
    step against the oracle from the GPU's own x_t at the north_star bar (1e-10)."""
    A, b, x0 = synth.make_instance(5)
    C, T, seed = 65536, 10, 105
    s = tm.Sampler(A, b)
    rng = np.random.default_rng(5)
    chains = np.unique(np.concatenate([[0, 1, 40000, C - 1], rng.choice(C, size=12, replace=False)]))
    trace, out = s.test_trace(np.tile(x0, (C, 1)), T, seed=seed, chains=chains)
    assert s.stats()["rejections"] == 0
    log = []
    check_trace(A, b, trace, seed, chains, projection=1, log=log)
    print("exempt steps", log)
    s.close()
