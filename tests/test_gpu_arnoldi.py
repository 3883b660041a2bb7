"""Block Arnoldi (Alg. 1, BASELINE configs[2] shape) driven through the C-ABI, both variants.

Pins: the oracle-driven Arnoldi on a small grid (same seeded start block, same Laplacian
written in numpy) gives the same block-Hessenberg H; properties that hold at any size:
orthonormal basis, the Arnoldi relation A V_m = V_{m+1} H, the Lanczos property of a
symmetric operator (H block tridiagonal up to rounding), Ritz values inside the closed-form
Laplacian spectrum [6 - 6cos(pi/(N+1)), 6 + 6cos(pi/(N+1))]."""
import math

import numpy as np
import pytest

from gpu_util import dev, empty, host, rel
from paper_2204_13393_b200 import inputs

pytestmark = pytest.mark.gpu
VARIANTS = ["cholqr2", "tsqr"]


@pytest.fixture(scope="module")
def P():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2204_13393_b200 import pqr

    pqr.lib()
    return pqr


def lap7_numpy(V, nx, ny, nz):
    """Reference Laplacian (Dirichlet, 6 on the diagonal) on a column-major block."""
    out = np.empty_like(V)
    for c in range(V.shape[1]):
        u = V[:, c].reshape(nz, ny, nx)
        y = 6.0 * u
        y[:, :, 1:] -= u[:, :, :-1]
        y[:, :, :-1] -= u[:, :, 1:]
        y[:, 1:, :] -= u[:, :-1, :]
        y[:, :-1, :] -= u[:, 1:, :]
        y[1:, :, :] -= u[:-1, :, :]
        y[:-1, :, :] -= u[1:, :, :]
        out[:, c] = y.reshape(-1)
    return out


def oracle_arnoldi(orc, R, nx, steps):
    """Alg. 1 with the oracle's PQR (widths follow the oracle's t: a deflated step adds fewer
    columns to H, at the running column offset)."""
    n, s = R.shape
    out = orc.householder_pqr(None, R)
    V = out["U"]
    H = np.zeros(((steps + 1) * s, steps * s))
    k = out["t"]
    w = k
    c0 = 0
    for i in range(steps):
        if w == 0:
            break
        X = lap7_numpy(V[:, k - w:k], nx, nx, nx)
        o = orc.householder_pqr(V, X)
        H[:k, c0:c0 + w] = o["P"]
        H[k:k + o["t"], c0:c0 + w] = o["N"][:o["t"]]
        V = np.hstack([V, o["U"]])
        c0 += w
        k += o["t"]
        w = o["t"]
    return V, H[:k, :c0]


@pytest.mark.parametrize("nx,ny,nz,s", [(9, 9, 9, 4), (37, 11, 23, 3), (64, 48, 40, 4), (1, 1, 5, 1), (33, 9, 300, 2)])
def test_stencil_vs_numpy(P, nx, ny, nz, s):
    """The operator kernel (z-marching lines, ragged x/y tiles, z chunks with halo planes)."""
    import torch

    n = nx * ny * nz
    V = inputs.gaussian(3 + n, n, s)
    Y = empty(n, s)
    P.pqr_laplacian7_apply(nx, ny, nz, s, dev(V), Y)
    torch.cuda.synchronize()
    assert rel(host(Y), lap7_numpy(V, nx, ny, nz)) < 1e-15


@pytest.mark.parametrize("variant", VARIANTS)
def test_arnoldi_vs_oracle_small(P, orc, variant):
    from paper_2204_13393_b200.arnoldi import block_arnoldi

    nx, s, steps = 10, 4, 6
    R = inputs.gaussian(inputs.CONFIGS["arnoldi"]["seed"], nx ** 3, s)
    out = block_arnoldi(nx, nx, nx, dev(R), steps, variant=variant)
    V_ref, H_ref = oracle_arnoldi(orc, R, nx, steps)
    assert out["t_list"] == [s] * (steps + 1)
    assert rel(out["H"], H_ref) < 1e-10
    out["h"].close()


@pytest.mark.parametrize("variant", VARIANTS)
def test_arnoldi_deflated_start_block(P, orc, variant):
    """A rank-deficient start block (column 2 = column 0): t = 3 at every step, so H has 3
    columns per block at the running offset; it must match the oracle's Arnoldi and satisfy
    A V_m = V_{m+1} H."""
    import torch

    from paper_2204_13393_b200.arnoldi import block_arnoldi

    nx, s, steps = 10, 4, 5
    R = inputs.gaussian(7, nx ** 3, s)
    R[:, 2] = R[:, 0]
    out = block_arnoldi(nx, nx, nx, dev(R), steps, variant=variant)
    assert out["t_list"] == [3] * (steps + 1)
    V_ref, H_ref = oracle_arnoldi(orc, R, nx, steps)
    assert out["H"].shape == H_ref.shape == (3 * (steps + 1), 3 * steps)
    assert rel(out["H"], H_ref) < 1e-10
    h, k = out["h"], out["k"]
    V = empty(nx ** 3, k)
    h.apply(dev(np.eye(k)), k, V)
    torch.cuda.synchronize()
    Vh = host(V)
    m = out["H"].shape[1]
    assert np.linalg.norm(lap7_numpy(Vh[:, :m], nx, nx, nx) - Vh @ out["H"]) < 1e-11 * math.sqrt(m) * 12
    h.close()


@pytest.mark.parametrize("variant", VARIANTS)
def test_arnoldi_properties(P, variant):
    import torch

    from paper_2204_13393_b200.arnoldi import block_arnoldi

    nx, s, steps = 24, 4, 12
    n = nx ** 3
    R = inputs.gaussian(inputs.CONFIGS["arnoldi"]["seed"] + 1, n, s)
    out = block_arnoldi(nx, nx, nx, dev(R), steps, variant=variant)
    h, H, k = out["h"], out["H"], out["k"]
    assert k == (steps + 1) * s
    V = empty(n, k)
    h.apply(dev(np.eye(k)), k, V)
    torch.cuda.synchronize()
    Vh = host(V)
    # orthonormal basis
    assert np.linalg.norm(np.eye(k) - Vh.T @ Vh, 2) < 1e-12
    # Arnoldi relation A V_m = V_{m+1} H  (m = steps*s)
    m = steps * s
    AV = lap7_numpy(Vh[:, :m], nx, nx, nx)
    assert np.linalg.norm(AV - Vh @ H) / (12.0 * math.sqrt(m)) < 1e-12
    # Lanczos property: H is block tridiagonal up to rounding
    mask = np.zeros_like(H, dtype=bool)
    for bi in range(steps):
        mask[max(0, (bi - 1) * s):(bi + 2) * s, bi * s:(bi + 1) * s] = True
    assert np.abs(H[~mask]).max() < 1e-10 * np.abs(H).max()
    # Ritz values inside the Laplacian spectrum, largest close to it
    Hm = H[:m, :m]
    ritz = np.linalg.eigvalsh(0.5 * (Hm + Hm.T))
    lo, hi = 6 - 6 * math.cos(math.pi / (nx + 1)), 6 + 6 * math.cos(math.pi / (nx + 1))
    assert ritz.min() > lo - 1e-9 and ritz.max() < hi + 1e-9
    assert ritz.max() > 0.97 * hi
    h.close()


def test_arnoldi_variants_agree(P):
    """H is unique (P = Q^T X, N with positive pivots), so both variants must agree."""
    from paper_2204_13393_b200.arnoldi import block_arnoldi

    nx, s, steps = 20, 4, 10
    R = inputs.gaussian(99, nx ** 3, s)
    a = block_arnoldi(nx, nx, nx, dev(R), steps, variant="cholqr2")
    b = block_arnoldi(nx, nx, nx, dev(R), steps, variant="tsqr")
    assert rel(a["H"], b["H"]) < 1e-9
    a["h"].close()
    b["h"].close()
