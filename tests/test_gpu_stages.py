"""Stage-level parity of the CUDA path against the CPU oracle.

P1 RNG: Philox words bitwise (device vs oracle vs cuRAND), uniforms bitwise, nu within 4 ulp.
P2 GEMM: |Q - q| <= 2K 2^-53 sum_j |A_ij nu_j| elementwise (vs exact-ish fp64 reference).
P3 arcs: active flag identical unless |r - b| <= 4 ulp(r); alpha/beta within 1e-10 relative
   when 1 - |rho| >= 1e-8.
P4 I_act: canonical segments bit-identical to Alg. 2 on identical (alpha, beta).
P5 theta: |dtheta| <= 1e-13 on identical segments and u.
"""
import math

import numpy as np
import pytest

import oracle
import paper_2407_10449_b200 as tm

pytestmark = pytest.mark.gpu
TWO_PI = 6.283185307179586


# ------------------------------------------------------------------ P1
def test_philox_bitwise_three_ways():
    rng = np.random.default_rng(0)
    ctr = rng.integers(0, 2**32, size=(20000, 4), dtype=np.uint64).astype(np.uint32)
    key = rng.integers(0, 2**32, size=(20000, 2), dtype=np.uint64).astype(np.uint32)
    ctr[:100, 1:] = 0
    dev = tm.test_philox(ctr, key)
    cur = tm.test_philox(ctr, key, curand=True)
    assert np.array_equal(dev, cur)
    orc = np.stack([oracle.philox4x32_10(ctr[i], key[i]) for i in range(0, 20000, 10)])
    assert np.array_equal(dev[::10], orc)


@pytest.mark.parametrize("d", [1, 2, 7, 100, 1001])
def test_normals_and_uniform(d):
    seed, t, c0, C = 0xDEADBEEF12345, 77, 1000, 33
    nu, u = tm.test_normals(seed, t, c0, C, d)
    for c in range(C):
        ref = oracle.normals(seed, t, c0 + c, d)
        ulp = np.spacing(np.maximum(np.abs(ref), 1e-300))
        assert np.all(np.abs(nu[c] - ref) <= 4 * ulp + 1e-300), c
        assert u[c] == oracle.uniform(seed, t, c0 + c)


# ------------------------------------------------------------------ P2
@pytest.mark.parametrize("R,S,K", [(1, 1, 1), (130, 257, 37), (300, 128, 1000), (512, 640, 16),
                                   (129, 1000, 100)])
def test_gemm_bound(R, S, K):
    rng = np.random.default_rng(R * 7 + S)
    X = rng.standard_normal((R, K))
    W = rng.standard_normal((S, K))
    out = tm.test_gemm(X, W)
    ref = X @ W.T
    bound = 2 * K * 2.0**-53 * (np.abs(X) @ np.abs(W).T)
    assert np.all(np.abs(out - ref) <= 2 * bound + 1e-300)
    # oracle-style sequential dot products on a sample of rows
    for r in rng.choice(R, size=min(R, 5), replace=False):
        seq = np.array([sum(float(a) * float(b) for a, b in zip(X[r], W[s])) for s in range(min(S, 20))])
        assert np.all(np.abs(out[r, :seq.size] - seq) <= 2 * bound[r, :seq.size] + 1e-300)


# ------------------------------------------------------------------ P3
def _pqb(n, seed):
    rng = np.random.default_rng(seed)
    p = rng.standard_normal(n) * rng.choice([1e-3, 1.0, 30.0], n)
    q = rng.standard_normal(n) * rng.choice([1e-9, 1.0, 30.0], n)
    b = p + rng.exponential(1.0, n) * rng.choice([1e-12, 1e-3, 1.0, 100.0], n)
    # edge cases: zero rows, tangency, exactly-boundary, signed zeros, Fig. 2
    p = np.concatenate([p, [0.0, 0.0, -2.0, -2.0, -2.0, -2.0, -0.7, 3.0, -1.0]])
    q = np.concatenate([q, [0.0, 0.0, 0.0, 0.0, 0.0, -0.0, 1e-17, 4.0, 0.0]])
    b = np.concatenate([b, [0.0, 1.0, 2.5, 2.0, 1.0, 1.0, -0.7, 5.0, 0.0]])
    return p, q, b


def test_arcs_parity():
    p, q, b = _pqb(200000, 1)
    al, be, act = tm.test_arcs(p, q, b)
    ral, rbe, ract = oracle.arcs(p, q, b)
    r = np.hypot(p, q)
    differ = act != ract
    assert np.all(np.abs(r[differ] - b[differ]) <= 4 * np.spacing(r[differ]))
    both = act & ract
    rho = np.clip(b / np.where(r > 0, r, 1), -1, 1)
    well = both & (1 - np.abs(rho) >= 1e-8)
    tol = 1e-10 * np.maximum(1.0, np.abs(ral))
    assert np.all(np.abs(al - ral)[well] <= tol[well])
    assert np.all(np.abs(be - rbe)[well] <= 1e-10 * np.maximum(1.0, np.abs(rbe))[well])
    assert np.all((al[act] >= 0) & (al[act] <= be[act]) & (be[act] <= TWO_PI))


# ------------------------------------------------------------------ P4 / P5
def _canon_gpu(lo, hi, ns, c):
    n = int(ns[c])
    return np.stack([lo[c, :n], hi[c, :n]], 1)


def _check_intervals(alpha, beta, u, eps=0.0):
    lo, hi, ns, L, th = tm.test_intervals(alpha, beta, u=u, eps=eps)
    for c in range(alpha.shape[0]):
        ref = oracle.intervals(alpha[c], beta[c])
        got = _canon_gpu(lo, hi, ns, c)
        assert got.shape == ref.shape, (c, got.shape, ref.shape)
        assert np.array_equal(got, ref), c  # bit-identical (comparisons only)
        tr = oracle.trim(ref, eps) if len(ref) else ref
        if len(tr):
            th_ref, L_ref = oracle.sample_theta(tr, u[c])
            assert abs(L[c] - L_ref) <= 1e-13 * max(1.0, L_ref)
            assert abs(th[c] - th_ref) <= 1e-13, (c, th[c], th_ref)
        else:
            assert L[c] == 0.0


def test_intervals_random_with_padding_and_ties():
    rng = np.random.default_rng(2)
    C, m = 64, 300
    al = rng.uniform(0, TWO_PI, (C, m))
    be = np.minimum(al + rng.exponential(0.02, (C, m)), TWO_PI)
    pad = rng.random((C, m)) < 0.3
    al[pad] = 0.0
    be[pad] = 0.0
    dup = rng.random((C, m)) < 0.05
    al[:, 1:][dup[:, 1:]] = al[:, :-1][dup[:, 1:]]  # duplicate alphas
    deg = rng.random((C, m)) < 0.05
    be[deg] = al[deg]  # zero-length arcs
    be = np.maximum(be, al)
    _check_intervals(al, be, rng.random(C))


def test_intervals_paper_examples():
    # App. "Brute Force" worst case (k+1 segments) and the S3.1 sorting reduction:
    # thousands of live arcs -> exercises the batched / refined bucket sort.
    k = 60
    i = np.arange(1, k + 1, dtype=np.float64)
    al = (TWO_PI * 3.0 ** (-i))[None]
    be = (TWO_PI * (2.0 * 3.0 ** (-i)))[None]
    _check_intervals(al, be, np.array([0.37]))
    rng = np.random.default_rng(3)
    for m in (100, 2000, 6000):
        c = np.unique(rng.uniform(0.001, 6.2, m))
        rng.shuffle(c)
        eps = 0.5 * np.min(np.diff(np.sort(c)))
        _check_intervals(c[None], (c + eps)[None], np.array([0.81]))


def test_intervals_large_m_and_clusters():
    rng = np.random.default_rng(4)
    C, m = 6, 20000  # > in-smem stash: arcs spill to the global scratch
    al = np.concatenate([rng.uniform(0, TWO_PI, (C, m // 2)),
                         1.0 + 1e-9 * rng.random((C, m // 2))], axis=1)  # a dense cluster
    be = np.minimum(al + rng.exponential(0.0005, (C, m)), TWO_PI)
    al[:, ::7] = 2.5  # many identical alphas
    be = np.maximum(be, al)
    _check_intervals(al, be, rng.random(C))


def test_intervals_trim():
    rng = np.random.default_rng(5)
    C, m = 32, 50
    al = rng.uniform(0, TWO_PI, (C, m))
    be = np.minimum(al + rng.exponential(0.05, (C, m)), TWO_PI)
    _check_intervals(al, be, rng.random(C), eps=1e-3)


@pytest.mark.parametrize("warps,mode", [(0, 2), (8, 2), (2, 2), (1, 2), (16, 1), (4, 1)])
def test_intervals_bucket_mappings_and_group_sizes(warps, mode):
    """Alg. 3's bucketed form with the octave level-1 mapping (options.buckets = 2) and
    other group sizes: bit-identical to Alg. 2 (any monotone bucketing, Prop. 1),
    including arcs crowded just after theta = 0 (the S4.2 geometry the octave mapping
    is for), ties, padding and the paper's worst case."""
    tm.test_interval_config(warps, mode)
    try:
        rng = np.random.default_rng(11 + warps + 10 * mode)
        C, m = 24, 600
        al = 10.0 ** rng.uniform(-6, -1, (C, m))  # crowded near 0
        be = np.minimum(al + 10.0 ** rng.uniform(-5, 0.5, (C, m)), TWO_PI)
        al[:, ::9] = al[:, 1::9]  # ties
        pad = rng.random((C, m)) < 0.2
        al[pad] = 0.0
        be[pad] = 0.0
        _check_intervals(al, be, rng.random(C))
        test_intervals_random_with_padding_and_ties()
        test_intervals_paper_examples()
    finally:
        tm.test_interval_config(0, 1)
