"""ctypes wrapper around oracle/genred_oracle.c -- TEST INFRASTRUCTURE ONLY.

The C file holds all of the oracle's arithmetic (fp64, Neumaier sums, plain double loops; see
its header for the paper passage each function follows).  This module only marshals arguments:
it widens the (usually fp32) inputs to fp64 exactly and passes pointers.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "genred_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def lib_path() -> str:
    return _LIB


def build(force: bool = False) -> str:
    """Compile the oracle (gcc -O2 -fopenmp, no fast-math).  Building the checker is not using it."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fopenmp", "-fPIC", "-shared",
                               "-fno-fast-math", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB)
            P = ctypes.c_void_p
            I64, I32, F64 = ctypes.c_int64, ctypes.c_int, ctypes.c_double
            lib.oracle_num_threads.restype = I32
            lib.oracle_gauss_sum.argtypes = [I64, I64, I32, I32, F64, P, P, P, P, I64, P, P]
            lib.oracle_gauss_gradx.argtypes = [I64, I64, I32, I32, F64, P, P, P, P, P, I64, P, P]
            lib.oracle_lse.argtypes = [I64, I64, I32, F64, P, P, P, P, I64, P, P]
            lib.oracle_lse_cond.argtypes = [I64, I64, I32, F64, P, P, P, P, I64, P, P]
            lib.oracle_lse_cond.restype = None
            lib.oracle_gauss_cond.argtypes = [I64, I64, I32, I32, F64, I32, P, P, P, P, P, I64, P, P]
            lib.oracle_gauss_cond.restype = None
            lib.oracle_softmax_cond.argtypes = [I64, I64, I32, F64, P, P, P, P, P, P, P, I64, P, P, P, P]
            lib.oracle_softmax_cond.restype = None
            lib.oracle_argkmin.argtypes = [I64, I64, I32, I32, P, P, P, I64, P, P]
            lib.oracle_sqdist_sum.argtypes = [I64, I64, I32, I32, P, P, P, P, I64, P, P]
            lib.oracle_softmax_grad.argtypes = [I64, I64, I32, F64, P, P, P, P, P, P, P, I64, P, P, P, P]
            lib.oracle_softmax_grad.restype = None
            for f in ("oracle_gauss_sum", "oracle_gauss_gradx", "oracle_lse", "oracle_argkmin",
                      "oracle_sqdist_sum"):
                getattr(lib, f).restype = None
            _lib = lib
    return _lib


def num_threads() -> int:
    return int(_load().oracle_num_threads())


def set_num_threads(n: int) -> None:
    """OpenMP threads for the oracle (torchrun sets OMP_NUM_THREADS=1 per rank)."""
    lib = _load()
    lib.oracle_set_num_threads.argtypes = [ctypes.c_int]
    lib.oracle_set_num_threads.restype = None
    lib.oracle_set_num_threads(int(n))


def _f64(a, ncols=None):
    if a is None:
        return None
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if ncols is not None:
        a = a.reshape(-1, ncols)
    return a


def _ptr(a):
    return None if a is None else a.ctypes.data


def _rows(rows):
    if rows is None:
        return None, 0
    r = np.ascontiguousarray(np.asarray(rows, dtype=np.int64))
    return r, int(r.shape[0])


def gauss_sum(x, y, b=None, sigma=1.0, rows=None, cond=False):
    """O1.  Returns (a [R,E], denom [R,E]) in fp64.  cond=True also returns the R4c metric's
    (cond [R,E], tail [R,E]) (oracle_gauss_cond)."""
    x = _f64(x); y = _f64(y)
    M, D = x.shape; N = y.shape[0]
    b = _f64(b)
    E = 1 if b is None else (b.shape[1] if b.ndim == 2 else 1)
    r, nr = _rows(rows)
    R = nr if r is not None else M
    out = np.empty((R, E)); den = np.empty((R, E))
    _load().oracle_gauss_sum(M, N, D, E, float(sigma), _ptr(x), _ptr(y), _ptr(b), _ptr(r), nr,
                             _ptr(out), _ptr(den))
    if not cond:
        return out, den
    cc = np.empty((R, E)); tt = np.empty((R, E))
    _load().oracle_gauss_cond(M, N, D, E, float(sigma), 0, _ptr(x), _ptr(y), _ptr(b), None,
                              _ptr(r), nr, _ptr(cc), _ptr(tt))
    return out, den, cc, tt


def gauss_gradx(x, y, b=None, g=None, sigma=1.0, rows=None, cond=False):
    """O2.  Returns (G [R,D], denom [R,D]) in fp64.  cond=True also returns the R4c metric's
    (cond [R,D], tail [R,D]) (oracle_gauss_cond)."""
    x = _f64(x); y = _f64(y)
    M, D = x.shape; N = y.shape[0]
    b = _f64(b); g = _f64(g)
    E = 1
    if b is not None:
        E = b.shape[1] if b.ndim == 2 else 1
    elif g is not None:
        E = g.shape[1] if g.ndim == 2 else 1
    r, nr = _rows(rows)
    R = nr if r is not None else M
    out = np.empty((R, D)); den = np.empty((R, D))
    _load().oracle_gauss_gradx(M, N, D, E, float(sigma), _ptr(x), _ptr(y), _ptr(b), _ptr(g),
                               _ptr(r), nr, _ptr(out), _ptr(den))
    if not cond:
        return out, den
    cc = np.empty((R, D)); tt = np.empty((R, D))
    _load().oracle_gauss_cond(M, N, D, E, float(sigma), 1, _ptr(x), _ptr(y), _ptr(b), _ptr(g),
                              _ptr(r), nr, _ptr(cc), _ptr(tt))
    return out, den, cc, tt


def lse(x, y, h=None, eps=1.0, rows=None, cond=False):
    """O3.  Returns (a [R], m [R]) in fp64; m_i = max_j F_ij.  cond=True also returns
    C_i = sum_j p_ij (|x_i - y_j|^2/eps + |h_j|), the metric's conditioning (reading R6b)."""
    x = _f64(x); y = _f64(y)
    M, D = x.shape; N = y.shape[0]
    h = None if h is None else _f64(h).reshape(-1)
    r, nr = _rows(rows)
    R = nr if r is not None else M
    out = np.empty(R); mm = np.empty(R)
    _load().oracle_lse(M, N, D, float(eps), _ptr(x), _ptr(y), _ptr(h), _ptr(r), nr,
                       _ptr(out), _ptr(mm))
    if not cond:
        return out, mm
    cc = np.empty(R)
    _load().oracle_lse_cond(M, N, D, float(eps), _ptr(x), _ptr(y), _ptr(h), _ptr(r), nr,
                            _ptr(out), _ptr(cc))
    return out, mm, cc


def argkmin(x, y, K, rows=None):
    """O4.  Returns (d [R,K] fp64 squared distances, j [R,K] int64), ascending in (d, j)."""
    x = _f64(x); y = _f64(y)
    M, D = x.shape; N = y.shape[0]
    r, nr = _rows(rows)
    R = nr if r is not None else M
    dist = np.empty((R, K)); idx = np.empty((R, K), dtype=np.int64)
    _load().oracle_argkmin(M, N, D, int(K), _ptr(x), _ptr(y), _ptr(r), nr, _ptr(dist), _ptr(idx))
    return dist, idx


def sqdist_sum(x, y, b=None, rows=None):
    """O5.  Returns (a [R,E], denom [R,E])."""
    x = _f64(x); y = _f64(y)
    M, D = x.shape; N = y.shape[0]
    b = _f64(b)
    E = 1 if b is None else (b.shape[1] if b.ndim == 2 else 1)
    r, nr = _rows(rows)
    R = nr if r is not None else M
    out = np.empty((R, E)); den = np.empty((R, E))
    _load().oracle_sqdist_sum(M, N, D, E, _ptr(x), _ptr(y), _ptr(b), _ptr(r), nr,
                              _ptr(out), _ptr(den))
    return out, den


def softmax_grad(x, y, alpha=None, beta=None, sig=None, coef=None, eps=1.0, rows=None, cond=False):
    """O6.  p_ij = exp(-|x_i-y_j|^2/eps + alpha_i + beta_j); returns (S [R], G [R,D], denS, denG)
    with S_i = sum_j sig_j p_ij and G_i = coef_i sum_j sig_j p_ij (-2/eps)(x_i - y_j).
    cond=True appends the R4c metric's (condS, condG, tailS, tailG) (oracle_softmax_cond)."""
    x = _f64(x); y = _f64(y)
    M, D = x.shape; N = y.shape[0]
    a, b_, s_, c_ = (None if v is None else _f64(v).reshape(-1) for v in (alpha, beta, sig, coef))
    r, nr = _rows(rows)
    R = nr if r is not None else M
    S = np.empty(R); G = np.empty((R, D)); dS = np.empty(R); dG = np.empty((R, D))
    _load().oracle_softmax_grad(M, N, D, float(eps), _ptr(x), _ptr(y), _ptr(a), _ptr(b_), _ptr(s_),
                                _ptr(c_), _ptr(r), nr, _ptr(S), _ptr(G), _ptr(dS), _ptr(dG))
    if not cond:
        return S, G, dS, dG
    cS = np.empty(R); cG = np.empty((R, D)); tS = np.empty(R); tG = np.empty((R, D))
    _load().oracle_softmax_cond(M, N, D, float(eps), _ptr(x), _ptr(y), _ptr(a), _ptr(b_), _ptr(s_),
                                _ptr(c_), _ptr(r), nr, _ptr(cS), _ptr(cG), _ptr(tS), _ptr(tG))
    return S, G, dS, dG, cS, cG, tS, tG
