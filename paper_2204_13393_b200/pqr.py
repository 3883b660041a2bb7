"""Thin ctypes binding of libpqr.so (include/pqr.h, include/pqr_steps.h).

Argument marshalling only — every step of the PQR path runs in the library's
CUDA kernels.  If libpqr.so is missing or cannot be loaded this module raises;
there is no CPU fallback.

Matrices are passed as torch tensors (CUDA or CPU) or numpy arrays, float64,
column-major: an n x m matrix is a tensor of shape (n, m) with stride(0) == 1
(e.g. ``inputs.colmajor_empty(n, m, device)``); its leading dimension is
stride(1).  CPU tensors / numpy arrays are host memory: the library stages them.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PQR_LIB") or os.path.join(_HERE, "libpqr.so")  # PQR_LIB: A/B builds

PQR_OK, PQR_EARG, PQR_ECAPACITY, PQR_EBREAKDOWN, PQR_EPLAN, PQR_ECUDA, PQR_ENCCL, PQR_ENOMEM = 0, -1, -2, -3, -4, -5, -6, -7
PQR_CHOLQR2, PQR_TSQR = 0, 1
PQR_NO_APPEND, PQR_NO_DEFLATION, PQR_SINGLE_PASS = 1, 2, 4
VARIANTS = {"cholqr2": PQR_CHOLQR2, "tsqr": PQR_TSQR}
PQR_REDUCTION_HH, PQR_REDUCTION_PIP2 = 0, 1
REDUCTIONS = {"hh": PQR_REDUCTION_HH, "pip2": PQR_REDUCTION_PIP2}
PQR_LOCAL_HH, PQR_LOCAL_PIP2 = 0, 1
LOCALS = {"hh": PQR_LOCAL_HH, "pip2": PQR_LOCAL_PIP2}
PQR_EXCHANGE_AUTO, PQR_EXCHANGE_COLLECTIVE, PQR_EXCHANGE_LSA = 0, 1, 2
EXCHANGES = {"auto": PQR_EXCHANGE_AUTO, "collective": PQR_EXCHANGE_COLLECTIVE, "lsa": PQR_EXCHANGE_LSA}
PQR_CHAINS_AUTO, PQR_CHAINS_OFF, PQR_CHAINS_ON = 0, 1, 2
CHAINS = {"auto": PQR_CHAINS_AUTO, "off": PQR_CHAINS_OFF, "on": PQR_CHAINS_ON}


class PQRError(RuntimeError):
    def __init__(self, code, what):
        self.code = code
        super().__init__(f"{what}: {strerror(code)} ({code})")


class pqr_config(ctypes.Structure):
    _fields_ = [
        ("n_local", ctypes.c_int64), ("k_max", ctypes.c_int), ("s_max", ctypes.c_int),
        ("variant", ctypes.c_int), ("defl_tol", ctypes.c_double), ("gram_eta", ctypes.c_double),
        ("block_rows", ctypes.c_int), ("stream", ctypes.c_void_p), ("rank", ctypes.c_int),
        ("nranks", ctypes.c_int), ("nccl_id", ctypes.c_void_p), ("vgroup", ctypes.c_void_p),
        ("reduction", ctypes.c_int), ("local", ctypes.c_int), ("exchange", ctypes.c_int),
        ("chains", ctypes.c_int),
    ]


class pqr_stats(ctypes.Structure):
    _fields_ = [
        ("k", ctypes.c_int), ("last_t", ctypes.c_int), ("calls", ctypes.c_int64),
        ("collectives", ctypes.c_int64), ("collective_bytes", ctypes.c_int64),
        ("kernel_launches", ctypes.c_int64), ("block_rows", ctypes.c_int), ("tree_levels", ctypes.c_int),
        ("exchange", ctypes.c_int), ("leaf_chains", ctypes.c_int),
    ]


class pqr_profile(ctypes.Structure):
    _fields_ = [("ms", ctypes.c_double * 9), ("launches", ctypes.c_int64 * 9)]


PROFILE_KINDS = ["gram", "factor", "update", "nccl", "tsqr_local", "tsqr_tree", "tsqr_apply", "other", "update_gram"]

EXPORTS = ["pqr_create", "pqr_project_normalize", "pqr_basis_apply", "pqr_destroy", "pqr_strerror",
           "pqr_get_stats", "pqr_profile_enable", "pqr_get_profile", "pqr_nccl_unique_id",
           "pqr_vgroup_create", "pqr_vgroup_destroy",
           "pqr_step_gram", "pqr_step_factor", "pqr_step_update", "pqr_laplacian7_apply"]

_lib = None


def lib():
    """Load libpqr.so (raises if it is missing: the product path has no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libpqr.so not built at {LIB_PATH}; run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(LIB_PATH)
    vp, i, i64, d, u = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double, ctypes.c_uint
    L.pqr_create.argtypes = [ctypes.POINTER(vp), ctypes.POINTER(pqr_config), vp, i64, i]
    L.pqr_project_normalize.argtypes = [vp, vp, i64, i, u, vp, i64, vp, i, vp, i, ctypes.POINTER(ctypes.c_int)]
    L.pqr_basis_apply.argtypes = [vp, vp, i, i, vp, i64]
    L.pqr_destroy.argtypes = [vp]
    L.pqr_strerror.argtypes = [i]
    L.pqr_strerror.restype = ctypes.c_char_p
    L.pqr_get_stats.argtypes = [vp, ctypes.POINTER(pqr_stats)]
    L.pqr_profile_enable.argtypes = [vp, i]
    L.pqr_get_profile.argtypes = [vp, ctypes.POINTER(pqr_profile)]
    L.pqr_nccl_unique_id.argtypes = [vp]
    L.pqr_vgroup_create.argtypes = [i, ctypes.POINTER(vp)]
    L.pqr_vgroup_destroy.argtypes = [vp]
    L.pqr_step_gram.argtypes = [i64, i, i, vp, i64, vp, i64, vp, i, vp]
    L.pqr_step_factor.argtypes = [i, i, vp, i, d, d, vp, i, vp, i, ctypes.POINTER(ctypes.c_int),
                                  ctypes.POINTER(ctypes.c_int), vp]
    L.pqr_step_update.argtypes = [i64, i, i, vp, i64, vp, i64, vp, i, i, vp, i64, vp]
    L.pqr_laplacian7_apply.argtypes = [i, i, i, i, vp, i64, vp, i64, vp]
    for f in EXPORTS:
        if f != "pqr_strerror":
            getattr(L, f).restype = ctypes.c_int
    _lib = L
    return L


def strerror(code: int) -> str:
    try:
        return lib().pqr_strerror(code).decode()
    except Exception:  # pragma: no cover
        return "error"


def _check(rc, what):
    if rc != PQR_OK:
        raise PQRError(rc, what)


def _mat(a, rows=None):
    """(pointer, leading dimension) of a column-major float64 torch tensor / numpy array."""
    if a is None:
        return None, 1
    try:
        import torch

        if isinstance(a, torch.Tensor):
            if a.dtype != torch.float64:
                raise TypeError("pqr: matrices must be float64")
            # every column must be contiguous (a strided view such as A[:, j] of a row-major
            # matrix would otherwise be read as contiguous rows)
            if a.dim() not in (1, 2) or (a.shape[0] > 1 and a.stride(0) != 1):
                raise ValueError("pqr: matrices must be column-major (stride(0) == 1)")
            if a.dim() == 1:
                return a.data_ptr(), max(1, a.shape[0])
            ld = a.stride(1) if a.shape[1] > 1 else max(1, a.shape[0])
            return a.data_ptr(), ld
    except ImportError:  # pragma: no cover
        pass
    import numpy as np

    if isinstance(a, np.ndarray):
        if a.dtype != np.float64:
            raise TypeError("pqr: matrices must be float64")
        if a.ndim not in (1, 2) or (a.shape[0] > 1 and a.strides[0] != 8) or (a.ndim == 2 and a.strides[1] % 8):
            raise ValueError("pqr: matrices must be column-major (contiguous columns)")
        if a.ndim == 1:
            return a.ctypes.data, max(1, a.shape[0])
        ld = a.strides[1] // 8 if a.shape[1] > 1 else max(1, a.shape[0])
        return a.ctypes.data, ld
    if isinstance(a, int):
        if rows is None:
            raise ValueError("raw pointer needs an explicit ld")
        return a, rows
    raise TypeError(f"pqr: unsupported matrix type {type(a)}")


def _stream_ptr(stream):
    if stream is None:
        return None
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


# ---------------------------------------------------------------------------
# C-ABI mirror (same names)
# ---------------------------------------------------------------------------
def pqr_create(n_local, k_max, s_max, Q=None, k=0, variant="cholqr2", defl_tol=0.0, gram_eta=0.0, block_rows=0,
               stream=None, rank=0, nranks=1, nccl_id: bytes | None = None, vgroup=None, reduction="hh",
               local="hh", exchange="auto", chains="auto"):
    cfg = pqr_config()
    cfg.n_local = int(n_local)
    cfg.k_max = int(k_max)
    cfg.s_max = int(s_max)
    cfg.variant = VARIANTS[variant] if isinstance(variant, str) else int(variant)
    cfg.defl_tol = float(defl_tol)
    cfg.gram_eta = float(gram_eta)
    cfg.block_rows = int(block_rows)
    cfg.stream = _stream_ptr(stream)
    cfg.rank = int(rank)
    cfg.nranks = int(nranks)
    cfg.vgroup = vgroup.value if isinstance(vgroup, ctypes.c_void_p) else vgroup
    cfg.reduction = REDUCTIONS[reduction] if isinstance(reduction, str) else int(reduction)
    cfg.local = LOCALS[local] if isinstance(local, str) else int(local)
    cfg.exchange = EXCHANGES[exchange] if isinstance(exchange, str) else int(exchange)
    cfg.chains = CHAINS[chains] if isinstance(chains, str) else int(chains)
    idbuf = None
    if nccl_id is not None:
        idbuf = ctypes.create_string_buffer(bytes(nccl_id), 128)
        cfg.nccl_id = ctypes.cast(idbuf, ctypes.c_void_p)
    qp, ldq = _mat(Q) if (Q is not None and k > 0) else (None, max(1, int(n_local)))
    h = ctypes.c_void_p()
    if Q is not None and k > 0:
        _need(Q, int(n_local), int(k), "Q")
    _check(lib().pqr_create(ctypes.byref(h), ctypes.byref(cfg), qp, ldq, int(k)), "pqr_create")
    _n_local[h.value] = int(n_local)
    return h


def _shape(a):
    if a is None or isinstance(a, int):
        return None
    sh = tuple(a.shape)
    return sh if len(sh) == 2 else (sh[0], 1)


def _need(a, rows, cols, what):
    """Refuse an undersized buffer (the library would read or write past its end)."""
    sh = _shape(a)
    if sh is not None and (sh[0] < rows or sh[1] < cols):
        raise ValueError(f"pqr: {what} has shape {sh}, needs at least ({rows}, {cols})")


_n_local = {}  # handle value -> n_local (shape checks of the wrappers)


def pqr_project_normalize(h, X, s=None, flags=0, U=None, P=None, N=None):
    xp, ldx = _mat(X)
    s = int(s if s is not None else X.shape[1])
    n = _n_local.get(h.value if isinstance(h, ctypes.c_void_p) else h, 0)
    _need(X, n, s, "X")
    _need(U, n, s, "U")
    _need(N, s, s, "N")
    if P is not None:
        _need(P, pqr_get_stats(h)["k"], s, "P")
    up, ldu = _mat(U)
    pp, ldp = _mat(P)
    np_, ldn = _mat(N)
    t = ctypes.c_int(0)
    _check(lib().pqr_project_normalize(h, xp, ldx, s, int(flags), up, ldu, pp, ldp, np_, ldn, ctypes.byref(t)),
           "pqr_project_normalize")
    return t.value


def pqr_basis_apply(h, C, m, Y):
    n = _n_local.get(h.value if isinstance(h, ctypes.c_void_p) else h, 0)
    _need(Y, n, int(m), "Y")
    if C is not None:
        _need(C, pqr_get_stats(h)["k"], int(m), "C")
    cp, ldc = _mat(C)
    yp, ldy = _mat(Y)
    _check(lib().pqr_basis_apply(h, cp, ldc, int(m), yp, ldy), "pqr_basis_apply")


def pqr_destroy(h):
    if h is not None and h.value:
        _n_local.pop(h.value, None)
        _check(lib().pqr_destroy(h), "pqr_destroy")


def pqr_get_stats(h) -> dict:
    st = pqr_stats()
    _check(lib().pqr_get_stats(h, ctypes.byref(st)), "pqr_get_stats")
    return {f: getattr(st, f) for f, _ in pqr_stats._fields_}


def pqr_profile_enable(h, enable=True):
    _check(lib().pqr_profile_enable(h, 1 if enable else 0), "pqr_profile_enable")


def pqr_get_profile(h) -> dict:
    p = pqr_profile()
    _check(lib().pqr_get_profile(h, ctypes.byref(p)), "pqr_get_profile")
    return {kind: dict(ms=p.ms[i], launches=p.launches[i]) for i, kind in enumerate(PROFILE_KINDS)}


def pqr_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().pqr_nccl_unique_id(buf), "pqr_nccl_unique_id")
    return buf.raw


def pqr_vgroup_create(nranks):
    """A group of `nranks` virtual ranks (handles in this process exchanging through device copies)."""
    g = ctypes.c_void_p()
    _check(lib().pqr_vgroup_create(int(nranks), ctypes.byref(g)), "pqr_vgroup_create")
    return g


def pqr_vgroup_destroy(g):
    if g is not None and g.value:
        _check(lib().pqr_vgroup_destroy(g), "pqr_vgroup_destroy")


def pqr_step_gram(n, k, s, Q, X, W, stream=None):
    qp, ldq = _mat(Q) if k > 0 else (None, max(1, n))
    xp, ldx = _mat(X)
    wp, ldw = _mat(W)
    _check(lib().pqr_step_gram(int(n), int(k), int(s), qp, ldq, xp, ldx, wp, ldw, _stream_ptr(stream)), "pqr_step_gram")


def pqr_step_factor(k, s, W, N, M, tol2_rel=0.0, eta=0.0, stream=None):
    wp, ldw = _mat(W)
    np_, ldn = _mat(N)
    mp, ldm = _mat(M)
    t = ctypes.c_int(0)
    piv = (ctypes.c_int * 16)()
    _check(lib().pqr_step_factor(int(k), int(s), wp, ldw, float(tol2_rel), float(eta), np_, ldn, mp, ldm,
                                 ctypes.byref(t), piv, _stream_ptr(stream)), "pqr_step_factor")
    return t.value, [piv[i] for i in range(t.value)]


def pqr_step_update(n, k, s, Q, X, M, t, U, stream=None):
    qp, ldq = _mat(Q) if k > 0 else (None, max(1, n))
    xp, ldx = _mat(X)
    mp, ldm = _mat(M)
    up, ldu = _mat(U)
    _check(lib().pqr_step_update(int(n), int(k), int(s), qp, ldq, xp, ldx, mp, ldm, int(t), up, ldu,
                                 _stream_ptr(stream)), "pqr_step_update")


def pqr_laplacian7_apply(nx, ny, nz, s, V, Y, stream=None):
    vp, ldv = _mat(V)
    yp, ldy = _mat(Y)
    _check(lib().pqr_laplacian7_apply(int(nx), int(ny), int(nz), int(s), vp, ldv, yp, ldy, _stream_ptr(stream)),
           "pqr_laplacian7_apply")


# ---------------------------------------------------------------------------
# convenience object (same calls, RAII-style)
# ---------------------------------------------------------------------------
class PQR:
    """A PQR handle: ``PQR(n_local, k_max, s_max, Q, variant=...)``; ``solve(X, ...)`` returns t."""

    def __init__(self, n_local, k_max, s_max, Q=None, k=None, **kw):
        if k is None:
            k = 0 if Q is None else Q.shape[1]
        self.n_local = n_local
        self.h = pqr_create(n_local, k_max, s_max, Q=Q, k=k, **kw)

    def solve(self, X, U=None, P=None, N=None, flags=0, s=None):
        return pqr_project_normalize(self.h, X, s=s, flags=flags, U=U, P=P, N=N)

    def apply(self, C, m, Y):
        pqr_basis_apply(self.h, C, m, Y)

    def stats(self):
        return pqr_get_stats(self.h)

    def profile(self, enable=None):
        if enable is not None:
            pqr_profile_enable(self.h, enable)
            return None
        return pqr_get_profile(self.h)

    @property
    def k(self):
        return self.stats()["k"]

    def close(self):
        if self.h is not None:
            pqr_destroy(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass
