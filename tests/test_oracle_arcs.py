"""Pins for the oracle's arcs (Eq. 2 roots by eq:roots, C1-C5).

Pinned by the paper's printed worked examples (Fig. 1, Fig. 2), the closed
form of Eq. 2 at the roots, and a brute-force sign scan of Eq. 2 on a grid.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")
TWO_PI = 6.283185307179586


def fig1_halfspaces():
    g = json.load(open(os.path.join(GOLD, "fig1.json")))
    x, nu = np.array(g["x_t"]), np.array(g["nu"])
    E = lambda th: x * math.cos(th) + nu * math.sin(th)
    A, b = [], []
    for t1, t2 in g["pairs_over_pi"]:
        P1, P2 = E(t1 * math.pi), E(t2 * math.pi)
        v = P2 - P1
        a = np.array([v[1], -v[0]])
        bb = a @ P1
        if a @ x > bb:  # orient so that x_t = E(0) is feasible
            a, bb = -a, -bb
        A.append(a)
        b.append(bb)
    return g, x, nu, np.array(A), np.array(b)


def test_fig1_roots():
    g, x, nu, A, b = fig1_halfspaces()
    p, q = A @ x, A @ nu
    al, be, act = oracle.arcs(p, q, b)
    assert act.all()
    want = np.array(g["pairs_over_pi"]) * math.pi
    assert np.allclose(al, want[:, 0], atol=1e-13)
    assert np.allclose(be, want[:, 1], atol=1e-13)


def test_fig2_cases():
    g = json.load(open(os.path.join(GOLD, "fig2.json")))
    x, nu, a = np.array(g["x"]), np.array(g["nu"]), np.array(g["a"])
    p, q = a @ x, a @ nu
    for case in g["cases"]:
        al, be, act = oracle.arcs([p], [q], [case["b"]])
        r = math.hypot(p, q)
        assert abs(case["b"] / r - case["ratio"]) < 1e-15
        if case["expect"] == "inactive":
            assert not act[0] and al[0] == 0.0 and be[0] == 0.0
        elif case["expect"] == "arc":
            assert act[0]
            assert abs(al[0] - case["alpha_over_pi"] * math.pi) < 1e-14
            assert abs(be[0] - case["beta_over_pi"] * math.pi) < 1e-14
        elif case["expect"] == "boundary":
            # delta = pi: the whole ellipse except theta = 0 is infeasible -> L = 0
            assert act[0] and al[0] == 0.0 and abs(be[0] - TWO_PI) < 1e-15
            segs = oracle.intervals(al, be, act)
            assert len(segs) == 0
        elif case["expect"] == "infeasible_start":
            assert p > case["b"]  # x violates the constraint: rejected by the start check


def _random_feasible_pqb(n, seed):
    rng = np.random.default_rng(seed)
    p = rng.standard_normal(n) * rng.choice([1e-3, 1.0, 30.0], n)
    q = rng.standard_normal(n) * rng.choice([1e-6, 1.0, 30.0], n)
    slack = rng.exponential(1.0, n) * rng.choice([1e-9, 1e-3, 1.0], n)
    b = p + slack
    return p, q, b


def test_roots_satisfy_eq2_and_orientation():
    p, q, b = _random_feasible_pqb(20000, 1)
    al, be, act = oracle.arcs(p, q, b)
    r = np.hypot(p, q)
    assert np.array_equal(act, r > b)
    a, bb, pp, qq, rr = al[act], be[act], p[act], q[act], r[act]
    assert np.all((0.0 <= a) & (a <= bb) & (bb <= TWO_PI))
    rho = b[act] / rr
    well = (np.abs(rho) < 1 - 1e-6)
    for ang in (a, bb):
        on_edge = (ang == 0.0) | (ang == TWO_PI)
        res = np.abs(pp * np.cos(ang) + qq * np.sin(ang) - b[act])
        ok = res <= 1e-12 * np.maximum(1.0, rr)
        assert np.all(ok | on_edge | ~well)
    mid = 0.5 * (a + bb)
    wide = (bb - a) > 1e-6
    assert np.all(pp * np.cos(mid) + qq * np.sin(mid) - b[act] > 0) or not wide.any()
    assert np.all((pp * np.cos(mid) + qq * np.sin(mid) - b[act] > 0)[wide])


def test_sign_scan_brute_force():
    """The infeasible set {theta: p cos + q sin > b} on a grid equals (alpha, beta)."""
    p, q, b = _random_feasible_pqb(300, 2)
    al, be, act = oracle.arcs(p, q, b)
    th = np.linspace(0.0, TWO_PI, 100001)
    ct, st = np.cos(th), np.sin(th)
    for i in range(p.size):
        infeas = p[i] * ct + q[i] * st > b[i]
        pred = (th > al[i]) & (th < be[i]) if act[i] else np.zeros_like(infeas)
        mism = infeas != pred
        if mism.any():
            near = np.minimum(np.abs(th - al[i]), np.abs(th - be[i]))
            assert np.all(near[mism] < 1e-4), (i, p[i], q[i], b[i])


def test_zero_row_and_straddle_snap():
    # r = 0, b >= 0: tautology -> padding (C4)
    al, be, act = oracle.arcs([0.0], [0.0], [0.0])
    assert not act[0]
    # near-boundary straddle (C1): p ~ b < 0, tiny q.  theta = 0 must stay outside the arc
    p = np.full(2000, -0.7)
    q = np.linspace(-1e-12, 1e-12, 2000)
    b = p.copy()
    al, be, act = oracle.arcs(p, q, b)
    for i in np.nonzero(act)[0]:
        assert al[i] >= 0.0 and be[i] <= TWO_PI
        mid = 0.5 * (al[i] + be[i])
        assert p[i] * math.cos(mid) + q[i] * math.sin(mid) > b[i] - 1e-15
