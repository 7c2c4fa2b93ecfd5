"""Fit atan(t) = t * P(t^2) on |t| <= tan(pi/8) (tooling for common.cuh: fast_atan2).
Chebyshev interpolation in mpmath at high precision, monomial coefficients,
error of the FP64 Horner/FMA evaluation measured against mpmath."""
import mpmath as mp
import numpy as np
mp.mp.dps = 50
zmax = mp.tan(mp.pi / 8) ** 2
def f(z):
    if z == 0:
        return mp.mpf(1)
    t = mp.sqrt(z)
    return mp.atan(t) / t
for deg in range(7, 13):
    # Chebyshev nodes on [0, zmax]
    n = deg + 1
    nodes = [zmax / 2 * (1 - mp.cos(mp.pi * (k + mp.mpf(1) / 2) / n)) for k in range(n)]
    vals = [f(z) for z in nodes]
    # solve Vandermonde in mp
    V = mp.matrix([[z ** j for j in range(n)] for z in nodes])
    c = mp.lu_solve(V, mp.matrix(vals))
    coef = [float(c[j]) for j in range(n)]
    # evaluate in fp64 with fma-style horner (numpy has no fma; emulate with mp rounding per step)
    worst = 0.0
    for t in np.linspace(-float(mp.tan(mp.pi/8)), float(mp.tan(mp.pi/8)), 20001):
        z = t * t
        acc = coef[-1]
        for j in range(n - 2, -1, -1):
            acc = float(mp.mpf(acc) * mp.mpf(z) + mp.mpf(coef[j]))  # fused: one rounding
        y = t * acc
        ex = mp.atan(mp.mpf(t))
        if t != 0:
            worst = max(worst, abs(float((mp.mpf(y) - ex) / ex)))
    print(deg, f"max rel err {worst:.3e}", coef if deg == 10 else "")
