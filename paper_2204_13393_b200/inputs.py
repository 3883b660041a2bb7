"""Seeded synthetic input generators (shared by tests, bench.py and smoke()).

This module holds NONE of the PQR method's arithmetic: it only draws seeded
Gaussians and turns them into the matrices BASELINE.json's configs describe.
Where an input needs an orthonormal matrix ("Q orthonormal from a seeded
Gaussian"), it calls a LIBRARY QR (numpy.linalg.qr / LAPACK on the host,
torch.linalg.qr / cuSOLVER on the device) — never the oracle, never the CUDA
library under test.  Recipes are documented in DESIGN.md §"Inputs".

All host matrices are numpy float64 in Fortran (column-major) order; device
matrices are torch float64 tensors of shape (n, m) with strides (1, n), i.e.
column-major with leading dimension n (the C-ABI's layout).
"""
from __future__ import annotations

import math

import numpy as np

SEED_BASE = 2204133930

CONFIGS = {
    # BASELINE.json configs[0..4]
    "tiny": dict(n=10_000, k=32, s=4, seed=SEED_BASE + 0),
    "single": dict(n=2 ** 24, k=64, s=8, seed=SEED_BASE + 1),
    "arnoldi": dict(grid=256, s=4, steps=32, seed=SEED_BASE + 2),
    "deflation": dict(n=2 ** 22, k=96, s=16, seed=SEED_BASE + 3, dependent=(5, 11)),
    "weak": dict(n=2 ** 25, k=128, s=8, seed=SEED_BASE + 4),  # rows per GPU
}


# --------------------------------------------------------------------------
# host (numpy) generators
# --------------------------------------------------------------------------
def rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(seed))


def gaussian(seed: int, n: int, m: int) -> np.ndarray:
    """n x m i.i.d. N(0,1), column-major, drawn column by column."""
    return np.asfortranarray(rng(seed).standard_normal((m, n)).T)


def orthonormal(seed: int, n: int, k: int) -> np.ndarray:
    """Q = orthonormal factor of a seeded n x k Gaussian (LAPACK Householder QR)."""
    if k == 0:
        return np.zeros((n, 0), order="F")
    q, _ = np.linalg.qr(gaussian(seed, n, k), mode="reduced")
    return np.asfortranarray(q)


def bartlett(seed: int, s: int, dof_rows: int) -> np.ndarray:
    """Upper-triangular Bartlett factor: D_ii = sqrt(chi2(dof_rows - i)), D_ij ~ N(0,1) (i<j).

    If Y (n x s) is orthonormal and independent of the draw, Y D has the law of an
    n x s Gaussian projected onto span(Y) — used by the manufactured inputs so that
    X = Q C + Y D is distributed like an i.i.d. Gaussian block."""
    g = rng(seed)
    D = np.triu(g.standard_normal((s, s)), 1)
    for i in range(s):
        D[i, i] = math.sqrt(g.chisquare(max(1, dof_rows - i)))
    return np.asfortranarray(D)


def manufactured(seed: int, n: int, k: int, s: int, c_scale: float = 1.0, d: np.ndarray | None = None):
    """Inputs with a known PQR solution ("manufactured").

    [Q Y] = orthonormal factor of a seeded n x (k+s) Gaussian; C ~ N(0,1)*c_scale (k x s);
    D upper triangular with positive diagonal (Bartlett by default);  X = Q C + Y D.
    Then by Eq. (1) the unique solution with positive pivots is P = C, N = D, U = Y."""
    QY = orthonormal(seed, n, k + s)
    Q = np.asfortranarray(QY[:, :k])
    Y = np.asfortranarray(QY[:, k:])
    C = np.asfortranarray(rng(seed + 1).standard_normal((k, s)) * c_scale)
    D = bartlett(seed + 2, s, n - k) if d is None else np.asfortranarray(d)
    X = np.asfortranarray(Q @ C + Y @ D)
    return dict(Q=Q, X=X, C=C, D=D, Y=Y)


def stewart(seed: int, n: int, m: int, kappa: float) -> np.ndarray:
    """Stewart matrix: A = U diag(geom 1/kappa..1) V^T from a seeded Gaussian."""
    A = gaussian(seed, n, m)
    u, _ = np.linalg.qr(A, mode="reduced")
    v, _ = np.linalg.qr(gaussian(seed + 1, m, m))
    sig = np.logspace(-math.log10(kappa), 0.0, m)
    return np.asfortranarray((u * sig) @ v.T)


def tiny_inputs(seed: int = CONFIGS["tiny"]["seed"], n: int = 10_000, k: int = 32, s: int = 4):
    """configs[0]: Q = orthonormal factor of seeded N(0,1) n x k; X seeded N(0,1) n x s."""
    return orthonormal(seed, n, k), gaussian(seed + 7, n, s)


def projected_inputs(seed: int, n: int, k: int, s: int, ratio: float = 1e-2):
    """configs[1] shape at any n: X = Q C + E, C ~ N(0,1) (k x s),
    E_ij ~ N(0, (ratio*sqrt(k/n))^2) so ||E||_F / ||Q C||_F ~= ratio (reading R8)."""
    Q = orthonormal(seed, n, k)
    C = rng(seed + 1).standard_normal((k, s))
    E = gaussian(seed + 2, n, s) * (ratio * math.sqrt(max(k, 1) / n))
    return Q, np.asfortranarray(Q @ C + E)


def deflation_inputs(seed: int, n: int, k: int, s: int, dependent=(5, 11), grade: float = 1e-8):
    """configs[3] shape at any n (reading R9): X0 = G diag(grade^(j/(s-1))), then each
    dependent column j := Q c_j + X[:, :j] e_j (earlier columns only).  Expected t = s - len(dependent)."""
    Q = orthonormal(seed, n, k)
    X = gaussian(seed + 1, n, s) * np.array([grade ** (j / max(1, s - 1)) for j in range(s)])
    g = rng(seed + 2)
    for j in dependent:
        if j < s:
            c = g.standard_normal(k)
            e = g.standard_normal(j)
            X[:, j] = Q @ c + X[:, :j] @ e
    return Q, np.asfortranarray(X)


# --------------------------------------------------------------------------
# device (torch) generators, for full-size configs
# --------------------------------------------------------------------------
def _torch():
    import torch

    return torch


def colmajor_empty(n: int, m: int, device, dtype=None):
    """Allocate an n x m column-major (ld = n) float64 tensor."""
    torch = _torch()
    return torch.empty((m, n), device=device, dtype=dtype or torch.float64).t()


def device_gaussian(seed: int, n: int, m: int, device) -> "torch.Tensor":
    torch = _torch()
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    out = colmajor_empty(n, m, device)
    out.t().normal_(generator=g)
    return out


def device_orthonormal(seed: int, n: int, k: int, device, scale: float = 1.0, slab: int = 2 ** 21) -> "torch.Tensor":
    """Orthonormal n x k (column-major) from a seeded Gaussian via cuSOLVER QR (torch.linalg.qr).

    For n > slab the rows are cut into c = ceil(n/slab) slabs, each slab's Gaussian is
    QR-factorised on its own and the stacked factors are scaled by 1/sqrt(c):
    sum_i (Q_i/sqrt(c))^T (Q_i/sqrt(c)) = I, so the result is globally orthonormal
    (cuSOLVER's orgqr fails beyond ~2^31 elements).  ``scale`` multiplies the result
    (1/sqrt(P) makes P independently drawn rank shards globally orthonormal)."""
    torch = _torch()
    out = colmajor_empty(n, k, device)
    if k == 0:
        return out
    c = max(1, -(-n // slab))
    bounds = [(i * n // c, (i + 1) * n // c) for i in range(c)]
    for i, (r0, r1) in enumerate(bounds):
        A = device_gaussian(seed + 7919 * i, r1 - r0, k, device)
        q, _ = torch.linalg.qr(A, mode="reduced")
        del A
        out[r0:r1].copy_(q)
        del q
    f = scale / math.sqrt(c)
    if f != 1.0:
        out.mul_(f)
    return out


def device_weak_inputs(seed: int, n_local: int, k: int, s: int, device, rank: int = 0, world: int = 1):
    """configs[4] per-GPU shard: Q_g = orthonormal(Gaussian shard)/sqrt(P) (globally orthonormal:
    sum_g Q_g^T Q_g = I), X_g seeded N(0,1).  Seeds differ per rank."""
    Q = device_orthonormal(seed + 1000 * rank, n_local, k, device, scale=1.0 / math.sqrt(world))
    X = device_gaussian(seed + 1000 * rank + 1, n_local, s, device)
    return Q, X


def device_projected_inputs(seed: int, n: int, k: int, s: int, device, ratio: float = 1e-2):
    """configs[1] on the device (reading R8)."""
    torch = _torch()
    Q = device_orthonormal(seed, n, k, device)
    g = torch.Generator(device="cpu")
    g.manual_seed(int(seed + 1))
    C = torch.randn((k, s), generator=g, dtype=torch.float64).to(device)
    X = device_gaussian(seed + 2, n, s, device)
    X.mul_(ratio * math.sqrt(max(k, 1) / n))
    X.addmm_(Q, C)
    return Q, X


def device_deflation_inputs(seed: int, n: int, k: int, s: int, device, dependent=(5, 11), grade: float = 1e-8):
    """configs[3] on the device (reading R9)."""
    torch = _torch()
    Q = device_orthonormal(seed, n, k, device)
    X = device_gaussian(seed + 1, n, s, device)
    X.mul_(torch.tensor([grade ** (j / max(1, s - 1)) for j in range(s)], dtype=torch.float64, device=device))
    g = torch.Generator(device="cpu")
    g.manual_seed(int(seed + 2))
    for j in dependent:
        if j < s:
            c = torch.randn((k,), generator=g, dtype=torch.float64).to(device)
            e = torch.randn((j,), generator=g, dtype=torch.float64).to(device)
            X[:, j] = Q @ c + X[:, :j] @ e
    return Q, X


def device_manufactured(seed: int, n: int, k: int, s: int, device, scale: float = 1.0):
    """Manufactured truth at full size on the device: [Q Y] orthonormal (cuSOLVER QR),
    C ~ N(0,1), D = Bartlett; X = Q C + Y D; truth P = C, N = D, U = Y."""
    torch = _torch()
    QY = device_orthonormal(seed, n, k + s, device, scale=scale)
    Q = QY[:, :k]
    Y = QY[:, k:]
    C = torch.from_numpy(rng(seed + 1).standard_normal((k, s))).to(device)
    D = torch.from_numpy(np.ascontiguousarray(bartlett(seed + 2, s, n - k))).to(device)
    X = colmajor_empty(n, s, device)
    X.copy_(Y @ D)
    X.addmm_(Q, C)
    return dict(Q=Q, X=X, C=C, D=D, Y=Y, QY=QY)
