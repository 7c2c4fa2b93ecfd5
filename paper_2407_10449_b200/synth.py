"""Seeded synthetic inputs shared by the tests, bench.py and smoke().

This module holds NONE of the method's arithmetic: it only draws problem
instances (A, b, x0) with the shapes and distributions of BASELINE.json's
configs and of the paper's own experiments (S4.1 one-dimensional intervals,
P:774-784; S4.2 random instances).  The recipe is stated in
DESIGN.md section "Inputs".  Every instance is generated on the host in FP64
with ``numpy.random.default_rng(instance_seed)``: A first, then b.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Config:
    key: str
    d: int
    m: int
    C: int
    T: int
    inst_seed: int
    chain_seed: int
    desc: str


# BASELINE.json "configs" (index = position in that list + 1).
CONFIGS = {
    1: Config("tiny2d", 2, 3, 16, 2000, 1, 101,
              "d=2, m=3, A rows iid N(0,1), b ~ U[0.5,1.5], x0=0"),
    2: Config("orthant", 100, 100, 1024, 5000, 2, 102,
              "d=100, A=-I, b=0, x0=0.1*ones"),
    3: Config("random", 1000, 2000, 4096, 1000, 3, 103,
              "d=1000, m=2000, unit-norm Gaussian rows, b ~ U[0.1,1.0], x0=0"),
    4: Config("heavy", 100, 100000, 1024, 200, 4, 104,
              "d=100, m=100000, unit-norm Gaussian rows, b ~ U[0.5,2.0], x0=0"),
    5: Config("boxscale", 4096, 16384, 65536, 100, 5, 105,
              "d=4096, m=16384, unit-norm Gaussian rows, b ~ U[0.2,1.0], x0=0"),
    # not a BASELINE config: the paper's own timing workload (S4.2; SURVEY
    # 8(f) NEXT-1) -- m = d, A iid N(0,1) (not normalised), x0 ~ N(0, I),
    # b = A x0 + U[0,1]^d, 10 chains
    6: Config("paper_s42", 1000, 1000, 10, 1000, 42, 106,
              "paper S4.2: d=m=1000, A iid N(0,1), x0 ~ N(0,I), b = A x0 + U[0,1]^d, 10 chains"),
    7: Config("paper_s42_single", 4000, 4000, 1, 1000, 4000, 107,
              "paper S4.2 single chain at the high end of Fig. 4 (P:839-842): d=m=4000, 1 chain"),
}

_B_RANGE = {1: (0.5, 1.5), 3: (0.1, 1.0), 4: (0.5, 2.0), 5: (0.2, 1.0)}


def unit_rows(A: np.ndarray) -> np.ndarray:
    return A / np.linalg.norm(A, axis=1, keepdims=True)


def make_instance(k: int, m: int | None = None, d: int | None = None):
    """(A [m x d], b [m], x0 [d]) for config k (optionally with overridden sizes)."""
    cfg = CONFIGS[k]
    m = cfg.m if m is None else m
    d = cfg.d if d is None else d
    rng = np.random.default_rng(cfg.inst_seed)
    if k in (6, 7):
        return paper_random(d, seed=cfg.inst_seed)
    if k == 2:
        A = -np.eye(d, dtype=np.float64)[:m]
        b = np.zeros(m)
        x0 = np.full(d, 0.1)
        return A, b, x0
    A = rng.standard_normal((m, d))
    if k != 1:
        A = unit_rows(A)
    lo, hi = _B_RANGE[k]
    b = rng.uniform(lo, hi, m)
    x0 = np.zeros(d)
    return A, b, x0


def one_dim(interval):
    """S4.1: N(0,1) truncated to [lo, hi] as A=[[1],[-1]], b=[hi,-lo]."""
    lo, hi = interval
    A = np.array([[1.0], [-1.0]])
    b = np.array([hi, -lo])
    x0 = np.array([0.5 * (lo + hi)])
    return A, b, x0


def paper_random(d: int, seed: int = 0):
    """S4.2: A d x d iid N(0,1); x0 ~ N(0,I); b = A x0 + U[0,1]^d."""
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((d, d))
    x0 = rng.standard_normal(d)
    b = A @ x0 + rng.uniform(0.0, 1.0, d)
    return A, b, x0


def random_spd_factor(d: int, seed: int = 0):
    """A lower-triangular L with positive diagonal (App. A change of variable)."""
    rng = np.random.default_rng(seed)
    M = rng.standard_normal((d, d)) / np.sqrt(d)
    S = M @ M.T + 0.5 * np.eye(d)
    return np.linalg.cholesky(S), rng.standard_normal(d)
