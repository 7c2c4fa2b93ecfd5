"""CPU oracle for arXiv 2407.10449 -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package.  The product package
``paper_2407_10449_b200`` never imports it, and the two share no code: this is
a thin ctypes wrapper over ``oracle/oracle.cpp`` (plain C++17, FP64, naive
loops, Alg. 2 by definition).  See the header of ``oracle.cpp`` for the
citations and for the pin behind every function.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.cpp")

TWO_PI = 6.283185307179586


def build(force: bool = False) -> str:
    """Compile oracle.cpp -> liboracle.so (g++ -O2, no fast-math, no FMA contraction)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        cmd = ["g++", "-std=c++17", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
               "-fPIC", "-shared", "-o", _SO, _SRC]
        subprocess.check_call(cmd)
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        P = ctypes.c_void_p
        i64, u64, u32, f64 = ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_double
        L.orc_philox4x32_10.argtypes = [P, P, P]
        L.orc_philox_block.argtypes = [u64, u32, u64, u64, u32, P]
        L.orc_normals.argtypes = [u64, u64, u64, i64, P]
        L.orc_uniform.argtypes = [u64, u64, u64]
        L.orc_uniform.restype = f64
        L.orc_arcs.argtypes = [P, P, P, i64, P, P, P]
        L.orc_intervals.argtypes = [P, P, P, i64, P, P, i64]
        L.orc_intervals.restype = i64
        L.orc_intervals_trace.argtypes = [P, P, i64, P]
        L.orc_trim.argtypes = [P, P, i64, f64, P, P]
        L.orc_trim.restype = i64
        L.orc_sample_theta.argtypes = [P, P, i64, f64, P]
        L.orc_sample_theta.restype = f64
        L.orc_step.argtypes = [P, P, i64, i64, P, u64, u64, u64, f64, P, P]
        L.orc_step.restype = ctypes.c_int
        L.orc_whiten.argtypes = [P, P, i64, i64, P, P, P, P]
        L.orc_whiten_point.argtypes = [P, i64, P, P, P]
        L.orc_unwhiten_point.argtypes = [P, i64, P, P, P]
        L.orc_run.argtypes = [P, P, i64, i64, P, i64, i64, u64, i64, i64, f64, i64, i64, P, P, P,
                              P, P, P, P, P, ctypes.c_int]
        L.orc_num_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class StepDump(ctypes.Structure):
    _fields_ = [("nu", ctypes.c_void_p), ("u", ctypes.c_void_p), ("p", ctypes.c_void_p),
                ("q", ctypes.c_void_p), ("alpha", ctypes.c_void_p), ("beta", ctypes.c_void_p),
                ("active", ctypes.c_void_p), ("seg_lo", ctypes.c_void_p),
                ("seg_hi", ctypes.c_void_p), ("seg_cap", ctypes.c_int64),
                ("nseg", ctypes.c_void_p), ("L", ctypes.c_void_p), ("theta", ctypes.c_void_p),
                ("x_prop", ctypes.c_void_p), ("max_slack", ctypes.c_void_p),
                ("accept", ctypes.c_void_p)]


# --------------------------------------------------------------------------- RNG (C12)
def philox4x32_10(ctr, key):
    ctr = np.ascontiguousarray(ctr, dtype=np.uint32)
    key = np.ascontiguousarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    lib().orc_philox4x32_10(_p(ctr), _p(key), _p(out))
    return out


def philox_block(seed, j, t, c, s):
    out = np.zeros(4, dtype=np.uint32)
    lib().orc_philox_block(seed, j, t, c, s, _p(out))
    return out


def normals(seed, t, c, d):
    nu = np.zeros(d, dtype=np.float64)
    lib().orc_normals(seed, t, c, d, _p(nu))
    return nu


def uniform(seed, t, c):
    return lib().orc_uniform(seed, t, c)


# --------------------------------------------------------------------------- arcs (eq:roots)
def arcs(p, q, b):
    p, q, b = _f64(p), _f64(q), _f64(b)
    n = p.size
    al, be = np.zeros(n), np.zeros(n)
    act = np.zeros(n, dtype=np.uint8)
    lib().orc_arcs(_p(p), _p(q), _p(b), n, _p(al), _p(be), _p(act))
    return al, be, act.astype(bool)


# --------------------------------------------------------------------------- Alg. 2
def intervals(alpha, beta, active=None):
    """Canonical I_act (list of (lo, hi)) by Alg. 2."""
    alpha, beta = _f64(alpha), _f64(beta)
    m = alpha.size
    act = None if active is None else np.ascontiguousarray(active, dtype=np.uint8)
    cap = m + 2
    lo, hi = np.zeros(cap), np.zeros(cap)
    n = lib().orc_intervals(_p(alpha), _p(beta), _p(act), m, _p(lo), _p(hi), cap)
    return np.stack([lo[:n], hi[:n]], axis=1)


def intervals_trace(alpha, beta):
    alpha, beta = _f64(alpha), _f64(beta)
    counts = np.zeros(alpha.size, dtype=np.int64)
    lib().orc_intervals_trace(_p(alpha), _p(beta), alpha.size, _p(counts))
    return counts


def trim(segs, eps):
    segs = np.asarray(segs, dtype=np.float64).reshape(-1, 2)
    lo, hi = _f64(segs[:, 0]), _f64(segs[:, 1])
    n = lo.size
    olo, ohi = np.zeros(max(n, 1)), np.zeros(max(n, 1))
    k = lib().orc_trim(_p(lo), _p(hi), n, eps, _p(olo), _p(ohi))
    return np.stack([olo[:k], ohi[:k]], axis=1)


def sample_theta(segs, u):
    segs = np.asarray(segs, dtype=np.float64).reshape(-1, 2)
    lo, hi = _f64(segs[:, 0]), _f64(segs[:, 1])
    L = ctypes.c_double(0.0)
    th = lib().orc_sample_theta(_p(lo), _p(hi), lo.size, u, ctypes.byref(L))
    return th, L.value


# --------------------------------------------------------------------------- Alg. 1
def step(A, b, x, seed, t, c, eps=0.0, seg_cap=None):
    """One oracle step for global chain c at iteration t; returns (x_next, dump dict)."""
    A, b, x = _f64(A), _f64(b), _f64(x)
    m, d = A.shape
    seg_cap = seg_cap or (m + 2)
    out = dict(nu=np.zeros(d), u=np.zeros(1), p=np.zeros(m), q=np.zeros(m), alpha=np.zeros(m),
               beta=np.zeros(m), active=np.zeros(m, np.uint8), seg_lo=np.zeros(seg_cap),
               seg_hi=np.zeros(seg_cap), nseg=np.zeros(1, np.int64), L=np.zeros(1),
               theta=np.zeros(1), x_prop=np.zeros(d), max_slack=np.zeros(1),
               accept=np.zeros(1, np.int32))
    dump = StepDump(*[_p(out[k]) if k != "seg_cap" else seg_cap for k in
                      ["nu", "u", "p", "q", "alpha", "beta", "active", "seg_lo", "seg_hi",
                       "seg_cap", "nseg", "L", "theta", "x_prop", "max_slack", "accept"]])
    xn = np.zeros(d)
    lib().orc_step(_p(A), _p(b), m, d, _p(x), seed, t, c, eps, _p(xn), ctypes.byref(dump))
    ns = int(out["nseg"][0])
    res = dict(nu=out["nu"], u=float(out["u"][0]), p=out["p"], q=out["q"], alpha=out["alpha"],
               beta=out["beta"], active=out["active"].astype(bool),
               segs=np.stack([out["seg_lo"][:min(ns, seg_cap)], out["seg_hi"][:min(ns, seg_cap)]], 1),
               nseg=ns, L=float(out["L"][0]), theta=float(out["theta"][0]), x_prop=out["x_prop"],
               max_slack=float(out["max_slack"][0]), accept=bool(out["accept"][0]))
    return xn, res


def run(A, b, X0, n_iter, seed, chain_offset=0, iter_offset=0, eps=0.0, burn_in=0, thin=1,
        mu=None, L=None, nthreads=0):
    """Run C chains; returns dict(X, sum, sumsq, n_rec, rejections, per_chain_rej)."""
    A, b, X0 = _f64(A), _f64(b), _f64(X0)
    m, d = A.shape
    C = X0.shape[0]
    X = np.zeros((C, d))
    s, sq = np.zeros(d), np.zeros(d)
    nrec, nrej = ctypes.c_int64(0), ctypes.c_int64(0)
    pcr = np.zeros(C, dtype=np.int64)
    mu = None if mu is None else _f64(mu)
    L = None if L is None else _f64(L)
    lib().orc_run(_p(A), _p(b), m, d, _p(X0), C, n_iter, seed, chain_offset, iter_offset, eps,
                  burn_in, thin, _p(mu), _p(L), _p(X), _p(s), _p(sq), ctypes.byref(nrec),
                  ctypes.byref(nrej), _p(pcr), nthreads)
    return dict(X=X, sum=s, sumsq=sq, n_rec=nrec.value, rejections=nrej.value, per_chain_rej=pcr)


# --------------------------------------------------------------------------- App. A
def whiten(A, b, mu=None, L=None):
    A, b = _f64(A), _f64(b)
    m, d = A.shape
    Ao, bo = np.zeros((m, d)), np.zeros(m)
    lib().orc_whiten(_p(A), _p(b), m, d, _p(None if mu is None else _f64(mu)),
                     _p(None if L is None else _f64(L)), _p(Ao), _p(bo))
    return Ao, bo


def whiten_point(x, mu=None, L=None):
    x = _f64(x)
    u = np.zeros(x.size)
    lib().orc_whiten_point(_p(x), x.size, _p(None if mu is None else _f64(mu)),
                           _p(None if L is None else _f64(L)), _p(u))
    return u


def unwhiten_point(u, mu=None, L=None):
    u = _f64(u)
    x = np.zeros(u.size)
    lib().orc_unwhiten_point(_p(u), u.size, _p(None if mu is None else _f64(mu)),
                             _p(None if L is None else _f64(L)), _p(x))
    return x


def num_threads():
    return lib().orc_num_threads()
