"""PARITY ORACLE — test infrastructure only.

ctypes bridge to ``oracle/liboracle.so`` (built from ``pqr_oracle.c`` with gcc).
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this module.  It shares nothing with the
CUDA library under ``paper_2204_13393_b200/``; neither imports the other.

Every wrapper takes numpy arrays in Fortran (column-major) order and follows
one function of ``pqr_oracle.h`` (each cites its PAPER.md passage there).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "pqr_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

CFLAGS = ["-O2", "-fno-fast-math", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared", "-std=c11"]


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (plain C, OpenMP over independent columns)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "pqr_oracle.h"))
    ):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        d, i, i64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
        pd = ctypes.c_double
        L = _lib
        L.orc_householder_pqr.argtypes = [i64, i, i, d, i64, d, i64, pd, d, i64, d, i64, d, i64, d, d, d]
        L.orc_gram.argtypes = [i64, i, i, d, i64, d, i64, d, i64]
        L.orc_cholesky_deflate.argtypes = [i, i, d, i64, pd, pd, d, i64, d, d]
        L.orc_update.argtypes = [i64, i, i, d, i64, d, i64, d, i64, d, i64, i, d, d, i64]
        L.orc_bcgs_pip.argtypes = [i64, i, i, d, i64, d, i64, pd, pd, d, i64, d, i64, d, i64, d, d]
        L.orc_bcgs_pip_plus.argtypes = [i64, i, i, d, i64, d, i64, pd, pd, d, i64, d, i64, d, i64, d, d]
        L.orc_matmul.argtypes = [i64, i, i, d, i64, d, i64, d, i64]
        L.orc_hh_local.argtypes = [i64, i, d, i64, d]
        L.orc_hh_apply.argtypes = [i64, i, d, i64, i, i, d, i64]
        L.orc_num_threads.argtypes = []
        for f in ("orc_householder_pqr", "orc_gram", "orc_cholesky_deflate", "orc_update",
                  "orc_bcgs_pip", "orc_bcgs_pip_plus", "orc_matmul", "orc_hh_local",
                  "orc_hh_apply", "orc_num_threads"):
            getattr(L, f).restype = ctypes.c_int
    return _lib


def _f(a, rows=None, cols=None):
    """Fortran-ordered float64 array (copy only if needed)."""
    a = np.asarray(a, dtype=np.float64)
    if a.ndim == 1:
        a = a.reshape(-1, 1)
    return np.asfortranarray(a)


def _ptr(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None and a.size else ctypes.c_void_p(0)


def _ld(a):
    return max(1, a.shape[0]) if a is not None else 1


def _check(rc, what):
    if rc != 0:
        raise RuntimeError(f"oracle {what} failed with code {rc}")


def num_threads() -> int:
    return lib().orc_num_threads()


def householder_pqr(Q, X, tau_abs=None, defl_tol=1e-12):
    """PQR of [Q X] by Householder (Alg. 6) with sign canonicalisation.

    Returns dict(U, P, N, t, dependent, diag_q_err).  ``tau_abs`` defaults to
    ``defl_tol * ||X||_F`` (reading R3)."""
    X = _f(X)
    n, s = X.shape
    Q = _f(Q) if Q is not None and np.size(Q) else np.zeros((n, 0), order="F")
    k = Q.shape[1]
    if tau_abs is None:
        tau_abs = defl_tol * float(np.linalg.norm(X))
    U = np.zeros((n, s), order="F")
    P = np.zeros((k, s), order="F")
    N = np.zeros((s, s), order="F")
    t = ctypes.c_int(0)
    dep = (ctypes.c_int * max(1, s))()
    dq = ctypes.c_double(0.0)
    rc = lib().orc_householder_pqr(n, k, s, _ptr(Q), _ld(Q), _ptr(X), _ld(X), tau_abs,
                                   _ptr(U), _ld(U), _ptr(P), max(1, k), _ptr(N), max(1, s),
                                   ctypes.byref(t), dep, ctypes.byref(dq))
    _check(rc, "householder_pqr")
    tt = t.value
    return dict(U=U[:, :tt].copy(order="F"), P=P, N=N, t=tt,
                dependent=[bool(dep[c]) for c in range(s)], diag_q_err=dq.value)


def gram(Q, X):
    """W = [Q X]^T X, (k+s) x s (step a1)."""
    X = _f(X)
    n, s = X.shape
    Q = _f(Q) if Q is not None and np.size(Q) else np.zeros((n, 0), order="F")
    k = Q.shape[1]
    W = np.zeros((k + s, s), order="F")
    _check(lib().orc_gram(n, k, s, _ptr(Q), _ld(Q), _ptr(X), _ld(X), _ptr(W), max(1, k + s)), "gram")
    return W


def cholesky_deflate(W, k, tau_abs2=0.0, eta_rel=0.0):
    """N^T N = G - P^T P with in-order deflation (step a3). Returns (N, t, piv)."""
    W = _f(W)
    s = W.shape[1]
    N = np.zeros((s, s), order="F")
    t = ctypes.c_int(0)
    piv = (ctypes.c_int * max(1, s))()
    _check(lib().orc_cholesky_deflate(k, s, _ptr(W), max(1, W.shape[0]), tau_abs2, eta_rel,
                                      _ptr(N), max(1, s), ctypes.byref(t), piv), "cholesky_deflate")
    return N, t.value, [piv[i] for i in range(t.value)]


def update(Q, X, P, N, t, piv):
    """U = (X - Q P) N_J^{-1} (step a4)."""
    X = _f(X)
    n, s = X.shape
    Q = _f(Q) if Q is not None and np.size(Q) else np.zeros((n, 0), order="F")
    k = Q.shape[1]
    P = _f(P) if k else np.zeros((1, s), order="F")
    N = _f(N)
    U = np.zeros((n, max(t, 1)), order="F")
    cpiv = (ctypes.c_int * max(1, s))(*piv)
    _check(lib().orc_update(n, k, s, _ptr(Q), _ld(Q), _ptr(X), _ld(X), _ptr(P), max(1, P.shape[0]),
                            _ptr(N), max(1, N.shape[0]), t, cpiv, _ptr(U), max(1, n)), "update")
    return U[:, :t].copy(order="F")


def _pip(fn, Q, X, tau_abs2, eta_rel):
    X = _f(X)
    n, s = X.shape
    Q = _f(Q) if Q is not None and np.size(Q) else np.zeros((n, 0), order="F")
    k = Q.shape[1]
    U = np.zeros((n, max(s, 1)), order="F")
    P = np.zeros((max(k, 1), s), order="F")
    N = np.zeros((max(s, 1), s), order="F")
    t = ctypes.c_int(0)
    piv = (ctypes.c_int * max(1, s))()
    rc = fn(n, k, s, _ptr(Q), _ld(Q), _ptr(X), _ld(X), tau_abs2, eta_rel, _ptr(U), max(1, n),
            _ptr(P), max(1, k), _ptr(N), max(1, s), ctypes.byref(t), piv)
    _check(rc, fn.__name__)
    tt = t.value
    return dict(U=U[:, :tt].copy(order="F"), P=P[:k], N=N[:s], t=tt, piv=[piv[i] for i in range(tt)])


def bcgs_pip(Q, X, tau_abs2=0.0, eta_rel=0.0):
    """Alg. 7 (BCGS-PIP)."""
    return _pip(lib().orc_bcgs_pip, Q, X, tau_abs2, eta_rel)


def bcgs_pip_plus(Q, X, tau_abs2=0.0, eta_rel=0.0):
    """Alg. 8 (BCGS-PIP+), recombination P = P1 + P2 N1, N = N2 N1."""
    return _pip(lib().orc_bcgs_pip_plus, Q, X, tau_abs2, eta_rel)


def matmul(Q, C):
    """Y = Q C (stage-2 product)."""
    Q = _f(Q)
    C = _f(C)
    n, k = Q.shape
    m = C.shape[1]
    Y = np.zeros((n, m), order="F")
    _check(lib().orc_matmul(n, k, m, _ptr(Q), _ld(Q), _ptr(C), max(1, C.shape[0]), _ptr(Y), max(1, n)), "matmul")
    return Y


def hh_local(A):
    """Alg. 6 with k=0 on a block, in place on a copy. Returns (V_and_R, rdiag)."""
    A = np.array(_f(A), order="F", copy=True)
    n, m = A.shape
    rd = np.zeros(max(1, m))
    _check(lib().orc_hh_local(n, m, _ptr(A), max(1, n), _ptr(rd)), "hh_local")
    return A, rd[:m]


def hh_apply(V, m, C, trans=False):
    """C <- Q_m C (or Q_m^T C) with the reflectors stored in V (from hh_local)."""
    V = _f(V)
    C = np.array(_f(C), order="F", copy=True)
    n = V.shape[0]
    _check(lib().orc_hh_apply(n, m, _ptr(V), max(1, n), 1 if trans else 0, C.shape[1], _ptr(C), max(1, n)),
           "hh_apply")
    return C
