"""Pins for the oracle's I_act (Alg. 2 by definition) and theta sampler.

Pinned by: Fig. 1 caption, the closed-form worst case of the
appendix "Brute Force", the sorting reduction of S3.1
(P:406-419), dense-theta-grid membership, Prop. 1 invariants (theta = 0 in
I_act), and closed forms / chi-square for the sampler.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
from test_oracle_arcs import fig1_halfspaces

GOLD = os.path.join(os.path.dirname(__file__), "golden")
TWO_PI = 6.283185307179586


def test_fig1_caption():
    g, x, nu, A, b = fig1_halfspaces()
    al, be, act = oracle.arcs(A @ x, A @ nu, b)
    segs = oracle.intervals(al, be, act)
    want = np.array(g["I_act_over_pi"]) * math.pi
    assert segs.shape == want.shape
    assert np.allclose(segs, want, atol=1e-13)
    # the inactive pair (2/5 pi, 4/5 pi) contributes no endpoint
    ends = set(segs.ravel().tolist())
    assert al[1] not in ends and be[1] not in ends


@pytest.mark.parametrize("k", json.load(open(os.path.join(GOLD, "app_brute_force.json")))["k_values"])
def test_appendix_worst_case_closed_form(k):
    i = np.arange(1, k + 1, dtype=np.float64)
    al = TWO_PI * 3.0 ** (-i)
    be = TWO_PI * (2.0 * 3.0 ** (-i))
    segs = oracle.intervals(al, be)
    # [0, 3^-k] U_{i=1..k} [2*3^-i, 3^-(i-1)], endpoints as the very same doubles:
    # 3^-(i-1) is alpha_{i-1} for i >= 2 and 1 (-> 2 pi) for i = 1
    want = [(0.0, al[k - 1])]
    for ii in range(k, 0, -1):
        want.append((be[ii - 1], al[ii - 2] if ii >= 2 else TWO_PI))
    assert len(segs) == k + 1
    assert np.array_equal(segs, np.array(want))  # comparisons only: exact
    counts = oracle.intervals_trace(al, be)
    assert np.array_equal(counts, np.arange(2, k + 2))


def test_sorting_reduction():
    rng = np.random.default_rng(3)
    c = np.unique(rng.uniform(0.1, 6.0, 200))
    rng.shuffle(c)
    eps = 0.5 * np.min(np.diff(np.sort(c)))
    segs = oracle.intervals(c, c + eps)
    cs = np.sort(c)
    want = [(0.0, cs[0])] + [(cs[k - 1] + eps, cs[k]) for k in range(1, cs.size)] + [(cs[-1] + eps, TWO_PI)]
    assert np.array_equal(segs, np.array(want))


def _dense_grid_case(rng, m, d):
    A = rng.standard_normal((m, d))
    x = rng.standard_normal(d) * 0.3
    b = A @ x + rng.exponential(0.5, m)
    nu = rng.standard_normal(d)
    return A, b, x, nu


def test_dense_theta_grid_membership():
    rng = np.random.default_rng(4)
    th = np.linspace(0.0, TWO_PI, 2**16 + 1)
    for case in range(60):
        m, d = int(rng.integers(1, 12)), int(rng.integers(1, 5))
        A, b, x, nu = _dense_grid_case(rng, m, d)
        p, q = A @ x, A @ nu
        al, be, act = oracle.arcs(p, q, b)
        segs = oracle.intervals(al, be, act)
        feas = np.max(p[:, None] * np.cos(th)[None] + q[:, None] * np.sin(th)[None] - b[:, None], 0) <= 0
        inside = np.zeros_like(feas)
        for lo, hi in segs:
            inside |= (th >= lo) & (th <= hi)
        mism = feas != inside
        if mism.any():
            ends = np.concatenate([segs.ravel(), al[act], be[act]])
            near = np.min(np.abs(th[mism][:, None] - ends[None]), axis=1)
            assert np.all(near < 1e-9), case
        assert segs[0, 0] == 0.0  # theta = 0 (x_t) is in I_act


def test_invariants_padding_and_monotone():
    rng = np.random.default_rng(5)
    for _ in range(200):
        m = int(rng.integers(1, 30))
        al = rng.uniform(0, TWO_PI, m)
        be = np.minimum(al + rng.exponential(0.5, m), TWO_PI)
        base = oracle.intervals(al, be)
        # padding pairs (0, 0) are no-ops, even when flagged active
        pal = np.concatenate([al, np.zeros(5)])
        pbe = np.concatenate([be, np.zeros(5)])
        perm = rng.permutation(m + 5)
        assert np.array_equal(oracle.intervals(pal[perm], pbe[perm]), base)
        # one more constraint never grows the total length
        L0 = np.sum(base[:, 1] - base[:, 0]) if len(base) else 0.0
        a2 = rng.uniform(0, TWO_PI)
        ext = oracle.intervals(np.append(al, a2), np.append(be, min(a2 + 0.3, TWO_PI)))
        L1 = np.sum(ext[:, 1] - ext[:, 0]) if len(ext) else 0.0
        assert L1 <= L0 + 1e-15
        # order independence (intersection is commutative)
        assert np.array_equal(oracle.intervals(al[::-1], be[::-1]), base)


def test_ties_and_degenerate_pairs():
    # duplicate alphas, alpha == beta (zero-length arcs split nothing, C2)
    al = np.array([1.0, 1.0, 2.0, 3.0, 3.0])
    be = np.array([1.5, 1.2, 2.0, 3.5, 3.0])
    segs = oracle.intervals(al, be)
    assert np.array_equal(segs, np.array([[0.0, 1.0], [1.5, 3.0], [3.5, TWO_PI]]))


def test_trim_rule_c7():
    segs = np.array([[0.0, 0.5], [2.0, 3.0], [4.0, TWO_PI]])
    out = oracle.trim(segs, 0.1)
    assert np.allclose(out, [[0.0, 0.4], [2.1, 2.9], [4.1, TWO_PI]])
    assert np.array_equal(oracle.trim(segs, 0.0), segs)
    # everything trimmed away -> untrimmed set (C7)
    tiny = np.array([[1.0, 1.1]])
    assert np.array_equal(oracle.trim(tiny, 0.06), tiny)


def test_sample_theta_closed_forms():
    th, L = oracle.sample_theta([[0.0, TWO_PI]], 0.25)
    assert L == TWO_PI and abs(th - math.pi / 2) < 1e-15
    th, L = oracle.sample_theta([[0.0, 1.0], [5.0, 6.0]], 0.75)
    assert L == 2.0 and th == 5.5
    th, L = oracle.sample_theta([[0.0, 1.0], [5.0, 6.0]], 0.0)
    assert th == 0.0


def test_sample_theta_uniform_chi2():
    segs = np.array([[0.0, 1.0], [2.0, 2.5], [5.0, 6.0]])
    rng = np.random.default_rng(6)
    us = rng.random(100000)
    ths = np.array([oracle.sample_theta(segs, u)[0] for u in us])
    # map back to the cumulative length -> must be uniform on [0, L)
    cum = np.where(ths <= 1.0, ths, np.where(ths <= 2.5, 1.0 + ths - 2.0, 1.5 + ths - 5.0))
    assert np.all(((ths >= 0) & (ths <= 1)) | ((ths >= 2) & (ths <= 2.5)) | ((ths >= 5) & (ths <= 6)))
    hist, _ = np.histogram(cum / 2.5, bins=100, range=(0, 1))
    e = us.size / 100
    chi2 = np.sum((hist - e) ** 2 / e)
    assert chi2 < 160  # p ~ 1e-4 at 99 dof
