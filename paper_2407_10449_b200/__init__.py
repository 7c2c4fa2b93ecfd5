"""B200-native batched linear elliptical slice sampling (arXiv 2407.10449).

Thin ctypes binding over ``libtmvn.so`` (C ABI: ``include/tmvn.h``).  Argument
marshalling only: every step of the sampler runs in the library's sm_100a
kernels.  There is no CPU fallback -- if the library is missing, the first call
raises ``RuntimeError``.

Array arguments may be numpy arrays (host) or torch tensors (host or CUDA);
they must be C-contiguous float64 (the library copies with cudaMemcpyDefault).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

__all__ = ["Sampler", "TmvnError", "lib", "options", "default_options", "tmvn_create",
           "tmvn_set_affine", "tmvn_set_options", "tmvn_get_options", "tmvn_sample",
           "tmvn_get_stats", "tmvn_get_moments", "tmvn_reset_stats", "tmvn_get_profile", "tmvn_destroy",
           "tmvn_last_error", "tmvn_version", "LIB_PATH"]

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libtmvn.so")

STATUS = {0: "TMVN_OK", -1: "TMVN_E_ARG", -2: "TMVN_E_EMPTY_POLYTOPE",
          -3: "TMVN_E_INFEASIBLE_START", -4: "TMVN_E_FACTOR", -5: "TMVN_E_CUDA",
          -6: "TMVN_E_OOM", -7: "TMVN_E_STATE"}

EXPORTS = ["tmvn_default_options", "tmvn_create", "tmvn_set_affine", "tmvn_set_options",
           "tmvn_get_options", "tmvn_sample", "tmvn_get_stats", "tmvn_get_moments",
           "tmvn_reset_stats", "tmvn_get_profile", "tmvn_last_error", "tmvn_version", "tmvn_struct_sizes",
           "tmvn_destroy", "tmvn_test_philox", "tmvn_test_curand_philox", "tmvn_test_normals", "tmvn_test_arcs",
           "tmvn_test_intervals", "tmvn_test_interval_config", "tmvn_test_gemm", "tmvn_test_ozaki_gemm", "tmvn_test_step",
           "tmvn_test_trace", "tmvn_test_latency_cap", "tmvn_test_latency_grid", "tmvn_cp_begin", "tmvn_cp_stats", "tmvn_cp_live",
           "tmvn_cp_theta", "tmvn_cp_commit", "tmvn_cp_end"]


class TmvnError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class options(ctypes.Structure):
    _fields_ = [("trim_eps", ctypes.c_double), ("recompute_every", ctypes.c_int64),
                ("burn_in", ctypes.c_int64), ("thin", ctypes.c_int64), ("record", ctypes.c_int32),
                ("chain_offset", ctypes.c_int64), ("iter_offset", ctypes.c_int64),
                ("auto_advance", ctypes.c_int32), ("stream", ctypes.c_void_p),
                ("profile", ctypes.c_int32), ("chain_warps", ctypes.c_int32),
                ("streams", ctypes.c_int32), ("ring", ctypes.c_int32),
                ("graphs", ctypes.c_int32), ("projection", ctypes.c_int32),
                ("ozaki_slices", ctypes.c_int32), ("rng_ahead", ctypes.c_int32),
                ("schedule", ctypes.c_int32), ("pipeline", ctypes.c_int32),
                ("latency", ctypes.c_int32), ("precision", ctypes.c_int32),
                ("total_chains", ctypes.c_int64), ("fuse_arcs", ctypes.c_int32),
                ("rng_gemm", ctypes.c_int32), ("rng_overlap", ctypes.c_int32),
                ("warp_mode", ctypes.c_int32), ("buckets", ctypes.c_int32),
                ("small_warps", ctypes.c_int32)]


class profile(ctypes.Structure):
    _fields_ = [("launches", ctypes.c_int64), ("gemm_launches", ctypes.c_int64),
                ("gemm_ms", ctypes.c_double), ("gemm_flops", ctypes.c_double),
                ("ess_launches", ctypes.c_int64), ("ess_ms", ctypes.c_double),
                ("ess_bytes", ctypes.c_double), ("tc_launches", ctypes.c_int64),
                ("tc_ms", ctypes.c_double), ("tc_ops", ctypes.c_double),
                ("tc_flops", ctypes.c_double), ("latency_calls", ctypes.c_int64),
                ("latency_fallbacks", ctypes.c_int64), ("latency_grid_calls", ctypes.c_int64),
                ("oz_guard_ratio", ctypes.c_double), ("projection_used", ctypes.c_int32),
                ("warp_mode_calls", ctypes.c_int64),
                ("buckets_used", ctypes.c_int32)]


class stats(ctypes.Structure):
    _fields_ = [("steps", ctypes.c_int64), ("rejections", ctypes.c_int64),
                ("recorded", ctypes.c_int64)]


class step_dump(ctypes.Structure):
    _fields_ = [("nu", ctypes.c_void_p), ("u", ctypes.c_void_p), ("p", ctypes.c_void_p),
                ("q", ctypes.c_void_p), ("alpha", ctypes.c_void_p), ("beta", ctypes.c_void_p),
                ("active", ctypes.c_void_p), ("seg_lo", ctypes.c_void_p),
                ("seg_hi", ctypes.c_void_p), ("seg_cap", ctypes.c_int64),
                ("nseg", ctypes.c_void_p), ("L", ctypes.c_void_p), ("theta", ctypes.c_void_p),
                ("x_next", ctypes.c_void_p), ("max_slack", ctypes.c_void_p),
                ("accept", ctypes.c_void_p)]


_LIB = None


def lib():
    """Load libtmvn.so (raises RuntimeError if it was not built)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} not found: build it with `make` (or "
                               "__graft_entry__.build()); there is no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        P, i64, u64, f64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double
        H = ctypes.c_void_p
        sig = {
            "tmvn_default_options": [P],
            "tmvn_create": [P, P, i64, i64, P],
            "tmvn_set_affine": [H, P, P],
            "tmvn_set_options": [H, P],
            "tmvn_get_options": [H, P],
            "tmvn_sample": [H, P, i64, i64, u64, P],
            "tmvn_get_stats": [H, P],
            "tmvn_get_moments": [H, P, P, P],
            "tmvn_reset_stats": [H],
            "tmvn_get_profile": [H, P],
            "tmvn_struct_sizes": [P],
            "tmvn_test_philox": [P, P, i64, P],
            "tmvn_test_curand_philox": [P, P, i64, P],
            "tmvn_test_normals": [u64, u64, i64, i64, i64, P, P],
            "tmvn_test_arcs": [P, P, P, i64, P, P, P],
            "tmvn_test_intervals": [P, P, i64, i64, P, f64, P, P, i64, P, P, P],
            "tmvn_test_interval_config": [ctypes.c_int32, ctypes.c_int32],
            "tmvn_test_gemm": [P, i64, P, i64, i64, P],
            "tmvn_test_ozaki_gemm": [P, i64, P, i64, i64, ctypes.c_int32, P],
            "tmvn_test_step": [H, P, i64, u64, i64, P],
            "tmvn_test_trace": [H, P, i64, i64, u64, P, i64, P, P],
            "tmvn_test_latency_cap": [H, ctypes.c_int32],
            "tmvn_test_latency_grid": [H, ctypes.c_int32],
            "tmvn_cp_begin": [H, P, i64, i64, u64],
            "tmvn_cp_stats": [H, i64, P, P, P],
            "tmvn_cp_live": [H, P, P, P, ctypes.c_int32, P, P],
            "tmvn_cp_theta": [H, i64, P, P, P, P, P, ctypes.c_int32, ctypes.c_int32, P],
            "tmvn_cp_commit": [H, i64, P],
            "tmvn_cp_end": [H, i64, P],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = ctypes.c_int
        L.tmvn_last_error.argtypes = [H]
        L.tmvn_last_error.restype = ctypes.c_char_p
        L.tmvn_version.argtypes = []
        L.tmvn_version.restype = ctypes.c_char_p
        L.tmvn_destroy.argtypes = [H]
        L.tmvn_destroy.restype = None
        _LIB = L
    return _LIB


def _ptr(a):
    """Raw pointer of a float64/int C-contiguous numpy array or torch tensor (None -> NULL)."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):  # torch.Tensor
        if not a.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return ctypes.c_void_p(a.data_ptr())
    if not a.flags["C_CONTIGUOUS"]:
        raise ValueError("array must be C-contiguous")
    return a.ctypes.data_as(ctypes.c_void_p)


def _check(status, handle=None):
    if status != 0:
        msg = lib().tmvn_last_error(handle)
        raise TmvnError(status, msg.decode() if msg else "")


def _f64(a):
    if a is None or hasattr(a, "data_ptr"):
        if a is not None:
            import torch
            if a.dtype != torch.float64:
                raise TypeError("tensor must be float64")
        return a
    return np.ascontiguousarray(a, dtype=np.float64)


def _expect(a, shape, name, writable=False):
    """Shape / dtype / layout check before a pointer crosses the ABI (the library copies
    prod(shape) doubles with cudaMemcpyDefault: a narrower or float32 buffer would be an
    out-of-bounds read or write, not an error)."""
    if hasattr(a, "data_ptr"):
        import torch
        if a.dtype != torch.float64:
            raise TypeError(f"{name} must be float64, got {a.dtype}")
        if not a.is_contiguous():
            raise ValueError(f"{name} must be contiguous")
    else:
        if not isinstance(a, np.ndarray) or a.dtype != np.float64:
            raise TypeError(f"{name} must be a float64 array")
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError(f"{name} must be C-contiguous")
        if writable and not a.flags["WRITEABLE"]:
            raise ValueError(f"{name} must be writable")
    if tuple(int(x) for x in a.shape) != tuple(shape):
        raise ValueError(f"{name} must have shape {tuple(shape)}, got {tuple(a.shape)}")


# ---------------------------------------------------------------- C-ABI mirrors
def default_options():
    o = options()
    _check(lib().tmvn_default_options(ctypes.byref(o)))
    return o


def tmvn_create(A, b, m, d):
    h = ctypes.c_void_p()
    _check(lib().tmvn_create(_ptr(A), _ptr(b), m, d, ctypes.byref(h)))
    return h


def tmvn_set_affine(h, mu, L):
    _check(lib().tmvn_set_affine(h, _ptr(mu), _ptr(L)), h)


def tmvn_set_options(h, opt):
    _check(lib().tmvn_set_options(h, ctypes.byref(opt)), h)


def tmvn_get_options(h):
    o = options()
    _check(lib().tmvn_get_options(h, ctypes.byref(o)), h)
    return o


def tmvn_sample(h, X0, C, n_iter, seed, out):
    _check(lib().tmvn_sample(h, _ptr(X0), C, n_iter, seed, _ptr(out)), h)


def tmvn_get_stats(h):
    s = stats()
    _check(lib().tmvn_get_stats(h, ctypes.byref(s)), h)
    return s


def tmvn_get_moments(h, sum_, sumsq):
    n = ctypes.c_int64(0)
    _check(lib().tmvn_get_moments(h, _ptr(sum_), _ptr(sumsq), ctypes.byref(n)), h)
    return n.value


def tmvn_reset_stats(h):
    _check(lib().tmvn_reset_stats(h), h)


def tmvn_get_profile(h):
    p = profile()
    _check(lib().tmvn_get_profile(h, ctypes.byref(p)), h)
    return p


def tmvn_last_error(h=None):
    s = lib().tmvn_last_error(h)
    return s.decode() if s else ""


def tmvn_version():
    return lib().tmvn_version().decode()


def tmvn_destroy(h):
    lib().tmvn_destroy(h)


# ---------------------------------------------------------------- convenience
class Sampler:
    """Owns one tmvn handle on the current CUDA device.

    >>> s = Sampler(A, b)            # A: m x d, b: m (numpy or torch, fp64)
    >>> out = s.sample(X0, n_iter=1000, seed=1)
    """

    def __init__(self, A, b, mu=None, L=None, **opts):
        A, b = _f64(A), _f64(b)
        if len(A.shape) != 2:
            raise ValueError(f"A must be m x d, got shape {tuple(A.shape)}")
        self.m, self.d = int(A.shape[0]), int(A.shape[1])
        _expect(b, (self.m,), "b")
        self.h = tmvn_create(A, b, self.m, self.d)
        if mu is not None or L is not None:
            self.set_affine(mu, L)
        if opts:
            self.set_options(**opts)

    def set_affine(self, mu=None, L=None):
        mu, L = _f64(mu), _f64(L)
        if mu is not None:
            _expect(mu, (self.d,), "mu")
        if L is not None:
            _expect(L, (self.d, self.d), "L")
        tmvn_set_affine(self.h, mu, L)

    def set_options(self, **kw):
        o = tmvn_get_options(self.h)
        for k, v in kw.items():
            if k == "stream" and v is not None and hasattr(v, "cuda_stream"):
                v = v.cuda_stream
            setattr(o, k, v)
        tmvn_set_options(self.h, o)

    def options(self):
        return tmvn_get_options(self.h)

    def sample(self, X0, n_iter, seed, out=None):
        X0 = _f64(X0)
        if len(X0.shape) != 2 or int(X0.shape[1]) != self.d:
            raise ValueError(f"X0 must be C x {self.d}, got shape {tuple(X0.shape)}")
        C = int(X0.shape[0])
        if out is None:
            out = X0.new_empty(X0.shape) if hasattr(X0, "new_empty") else np.empty_like(X0)
        else:
            _expect(out, (C, self.d), "out", writable=True)
        tmvn_sample(self.h, X0, C, n_iter, seed, out)
        return out

    def stats(self):
        s = tmvn_get_stats(self.h)
        return dict(steps=s.steps, rejections=s.rejections, recorded=s.recorded)

    def moments(self):
        s, q = np.zeros(self.d), np.zeros(self.d)
        n = tmvn_get_moments(self.h, s, q)
        return s, q, n

    def reset_stats(self):
        tmvn_reset_stats(self.h)

    def profile(self):
        p = tmvn_get_profile(self.h)
        return {k: getattr(p, k) for k, _ in p._fields_}

    def test_latency_cap(self, cap):
        """Test hook: cap latency mode's live-arc capacity (0 = automatic)."""
        _check(lib().tmvn_test_latency_cap(self.h, int(cap)), self.h)

    def test_latency_grid(self, mode):
        """Test hook: latency mode's cooperative-grid variant (1 force, -1 never, 0 auto)."""
        _check(lib().tmvn_test_latency_grid(self.h, int(mode)), self.h)

    def close(self):
        if getattr(self, "h", None):
            tmvn_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------ test hooks
    def test_step(self, Xt, seed, t, seg_cap=8):
        Xt = _f64(Xt)
        C = int(Xt.shape[0])
        m, d = self.m, self.d
        out = dict(nu=np.zeros((C, d)), u=np.zeros(C), p=np.zeros((C, m)), q=np.zeros((C, m)),
                   alpha=np.zeros((C, m)), beta=np.zeros((C, m)),
                   active=np.zeros((C, m), np.uint8), seg_lo=np.zeros((C, seg_cap)),
                   seg_hi=np.zeros((C, seg_cap)), nseg=np.zeros(C, np.int64), L=np.zeros(C),
                   theta=np.zeros(C), x_next=np.zeros((C, d)), max_slack=np.zeros(C),
                   accept=np.zeros(C, np.int32))
        dump = step_dump(*[seg_cap if k == "seg_cap" else _ptr(out[k]) for k in
                           [f[0] for f in step_dump._fields_]])
        _check(lib().tmvn_test_step(self.h, _ptr(Xt), C, seed, t, ctypes.byref(dump)), self.h)
        out["active"] = out["active"].astype(bool)
        out["accept"] = out["accept"].astype(bool)
        return out

    def test_trace(self, X0, n_iter, seed, chains, out=None):
        X0 = _f64(X0)
        C = int(X0.shape[0])
        chains = np.ascontiguousarray(chains, dtype=np.int64)
        trace = np.zeros((n_iter + 1, chains.size, self.d))
        if out is None:
            out = np.empty_like(X0) if not hasattr(X0, "new_empty") else X0.new_empty(X0.shape)
        _check(lib().tmvn_test_trace(self.h, _ptr(X0), C, n_iter, seed, _ptr(chains), chains.size,
                                     _ptr(trace), _ptr(out)), self.h)
        return trace, out


# ---------------------------------------------------------------- stage hooks
def test_philox(ctr, key, curand=False):
    ctr = np.ascontiguousarray(ctr, dtype=np.uint32).reshape(-1, 4)
    key = np.ascontiguousarray(key, dtype=np.uint32).reshape(-1, 2)
    out = np.zeros_like(ctr)
    f = lib().tmvn_test_curand_philox if curand else lib().tmvn_test_philox
    _check(f(_ptr(ctr), _ptr(key), ctr.shape[0], _ptr(out)))
    return out


def test_normals(seed, t, c0, C, d):
    nu, u = np.zeros((C, d)), np.zeros(C)
    _check(lib().tmvn_test_normals(seed, t, c0, C, d, _ptr(nu), _ptr(u)))
    return nu, u


def test_arcs(p, q, b):
    p, q, b = (np.ascontiguousarray(x, dtype=np.float64) for x in (p, q, b))
    n = p.size
    al, be, act = np.zeros(n), np.zeros(n), np.zeros(n, np.uint8)
    _check(lib().tmvn_test_arcs(_ptr(p), _ptr(q), _ptr(b), n, _ptr(al), _ptr(be), _ptr(act)))
    return al, be, act.astype(bool)


def test_interval_config(chain_warps=0, bucket_mode=1):
    """Launch configuration of test_intervals (process-wide): warps per chain, level-1
    buckets (1 linear, 2 by octave)."""
    _check(lib().tmvn_test_interval_config(int(chain_warps), int(bucket_mode)))


def test_intervals(alpha, beta, u=None, eps=0.0, seg_cap=None):
    alpha = np.ascontiguousarray(alpha, dtype=np.float64)
    beta = np.ascontiguousarray(beta, dtype=np.float64)
    C, m = alpha.shape
    seg_cap = seg_cap or (m + 2)
    lo, hi = np.zeros((C, seg_cap)), np.zeros((C, seg_cap))
    ns, L, th = np.zeros(C, np.int64), np.zeros(C), np.zeros(C)
    uu = None if u is None else np.ascontiguousarray(u, dtype=np.float64)
    _check(lib().tmvn_test_intervals(_ptr(alpha), _ptr(beta), m, C, _ptr(uu), eps, _ptr(lo),
                                     _ptr(hi), seg_cap, _ptr(ns), _ptr(L), _ptr(th)))
    return lo, hi, ns, L, th


def test_gemm(X, W):
    X = np.ascontiguousarray(X, dtype=np.float64)
    W = np.ascontiguousarray(W, dtype=np.float64)
    R, K = X.shape
    S = W.shape[0]
    out = np.zeros((R, S))
    _check(lib().tmvn_test_gemm(_ptr(X), R, _ptr(W), S, K, _ptr(out)))
    return out


def test_ozaki_gemm(X, W, slices=7):
    """X W^T through the production int8 tcgen05 projection (gemm_i8.cu)."""
    X = np.ascontiguousarray(X, dtype=np.float64)
    W = np.ascontiguousarray(W, dtype=np.float64)
    R, K = X.shape
    S = W.shape[0]
    out = np.zeros((R, S))
    _check(lib().tmvn_test_ozaki_gemm(_ptr(X), R, _ptr(W), S, K, slices, _ptr(out)))
    return out


from .cp import ConstraintParallel  # noqa: E402  (constraint-parallel driver)
