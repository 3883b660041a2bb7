"""GPU parity of the CholQR2 (BCGS-PIP+) path against the CPU oracle, per step of
SURVEY.md §8(a) (a1 Gram, a3 factor, a4 update, a5 reiteration) and end to end,
all through the C-ABI (libpqr.so).

Tolerances: BASELINE north_star — relative Frobenius error of
U, P, N <= 1e-10 for kappa <= 1e4 and ||I - [Q U]^T [Q U]||_2 <= 1e-12.  Single steps
that are plain sums (a1) are held tighter (1e-12): the only difference from the
oracle is the summation order, whose error is bounded by ~ n_chunk * eps."""
import numpy as np
import pytest

from gpu_util import dev, empty, host, ortho_loss_2, rel
from paper_2204_13393_b200 import inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2204_13393_b200 import pqr

    pqr.lib()
    return pqr


# ---------------------------------------------------------------------------
# a1: Gram
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("n,k,s", [(10_000, 32, 4), (5003, 17, 3), (4096, 0, 8), (3001, 96, 16),
                                   (2000, 128, 8), (7, 2, 1), (100_003, 64, 8), (65_536, 140, 12)])
def test_step_gram(P, orc, n, k, s):
    Q = inputs.orthonormal(n + k, n, k)
    X = inputs.gaussian(n + s, n, s)
    W = empty(k + s, s)
    P.pqr_step_gram(n, k, s, dev(Q), dev(X), W)
    assert rel(host(W), orc.gram(Q, X)) < 1e-12


# ---------------------------------------------------------------------------
# a3: small factorisation (N, t, pivots) from the oracle's W
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("case", ["random", "duplicate", "span", "k0"])
def test_step_factor(P, orc, case):
    n, k, s = 3000, 24, 8
    Q = inputs.orthonormal(1, n, k)
    X = inputs.gaussian(2, n, s)
    if case == "duplicate":
        X[:, 5] = X[:, 1]
    if case == "span":
        X[:, 3] = Q @ inputs.gaussian(3, k, 1)[:, 0]
    if case == "k0":
        Q = np.zeros((n, 0), order="F")
        k = 0
    W = orc.gram(Q, X)
    tol2, eta = 1e-24, 1e-13
    N_ref, t_ref, piv_ref = orc.cholesky_deflate(W, k, tau_abs2=tol2 * np.trace(W[k:]), eta_rel=eta)
    N = empty(s, s)
    M = empty(k + s, s)
    t, piv = P.pqr_step_factor(k, s, dev(W), N, M, tol2_rel=tol2, eta=eta)
    assert t == t_ref and piv == piv_ref
    assert rel(host(N), N_ref) < 1e-12
    if case in ("duplicate", "span"):
        assert t == s - 1


# ---------------------------------------------------------------------------
# a4: update U = [Q X] M   (M from the GPU factor step) vs the oracle's (X - QP) N^-1
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("n,k,s", [(10_000, 32, 4), (5003, 20, 5), (8192, 0, 16), (2049, 128, 8)])
def test_step_update(P, orc, n, k, s):
    Q = inputs.orthonormal(n, n, k)
    X = inputs.gaussian(n + 1, n, s)
    W = orc.gram(Q, X)
    N_ref, t, piv = orc.cholesky_deflate(W, k)
    U_ref = orc.update(Q, X, W[:k], N_ref, t, piv)
    Nd = empty(s, s)
    M = empty(k + s, s)
    t_gpu, _ = P.pqr_step_factor(k, s, dev(W), Nd, M)
    assert t_gpu == t
    U = empty(n, s)
    P.pqr_step_update(n, k, s, dev(Q), dev(X), M, t, U)
    assert rel(host(U)[:, :t], U_ref) < 1e-12
