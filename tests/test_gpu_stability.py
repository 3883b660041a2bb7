"""Stability suite on the GPU: block column QR (Alg. 2)
of Stewart matrices through the library, against the paper's printed
magnitudes (Table 1a), its qualitative claims (BCGS-PIP+ stable iff
eps*kappa^2 <= 1/2; TSPQR with stable subalgorithms is stable at any kappa,
PAPER.md:L984-996; errors insensitive to the number of subproblems) and
the CPU oracle's own Alg. 2 run on the same matrix.

Setup of experiment E1: n = 2^16 rows, s = 4, local blocks of 256 rows;
the matrix width is read as m = 64 (reading G10)."""
import numpy as np
import pytest

from gpu_util import dev
from paper_2204_13393_b200 import inputs

pytestmark = pytest.mark.gpu

N, M, S = 1 << 16, 64, 4


@pytest.fixture(scope="module")
def P():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2204_13393_b200 import blockqr, pqr

    pqr.lib()
    return blockqr


def run(B, A, variant, **kw):
    out = B.block_column_qr(A, S, variant=variant, **kw)
    return out, B.orthogonality_loss(out["Q"]), B.residual(A, out["Q"], out["R"])


def oracle_eperp(orc, Ah, solve):
    Q = np.zeros((Ah.shape[0], 0), order="F")
    for b in range(0, Ah.shape[1], S):
        out = solve(Q, np.asfortranarray(Ah[:, b:b + S]))
        Q = np.asfortranarray(np.hstack([Q, out["U"]]))
    return np.linalg.norm(np.eye(Q.shape[1]) - Q.T @ Q)


def test_table1a_level0(P, orc):
    """kappa = 1e4: paper prints e_perp 9.97e-10 (BCGS-PIP), 2.33e-15 (BCGS-PIP+), 9.07e-15 (HH)."""
    Ah = inputs.stewart(2204, N, M, 1e4)
    A = dev(Ah)
    _, e_pip, r_pip = run(P, A, "cholqr2", single_pass=True)
    _, e_pp, r_pp = run(P, A, "cholqr2")
    _, e_ts, r_ts = run(P, A, "tsqr", block_rows=256)
    assert 1e-12 < e_pip < 1e-6, e_pip
    assert e_pp < 1e-13 and e_ts < 1e-13, (e_pp, e_ts)
    assert max(r_pip, r_pp, r_ts) < 1e-14, (r_pip, r_pp, r_ts)
    # the oracle's Alg. 2 on the same matrix: same order of magnitude
    o_pip = oracle_eperp(orc, Ah, lambda Q, X: orc.bcgs_pip(Q, X))
    assert 0.1 < e_pip / o_pip < 10.0, (e_pip, o_pip)
    o_hh = oracle_eperp(orc, Ah, lambda Q, X: orc.householder_pqr(Q, X, tau_abs=0.0))
    assert e_ts < 10 * max(o_hh, 1e-15) and e_pp < 10 * max(o_hh, 1e-15), (e_ts, e_pp, o_hh)


@pytest.mark.parametrize("kappa", [1e2, 1e6, 1e10, 1e14])
def test_tsqr_stable_at_any_kappa(P, kappa):
    """TreeTSPQR with Householder local and reduction subalgorithms."""
    A = dev(inputs.stewart(7 + int(np.log10(kappa)), N, M, kappa))
    out, e, r = run(P, A, "tsqr", block_rows=256, defl_tol=1e-300)
    assert out["t_list"] == [S] * (M // S)
    assert e < 1e-13, e
    assert r < 1e-14, r


@pytest.mark.parametrize("kappa", [1e2, 1e5])
def test_cholqr2_stable_below_threshold(P, kappa):
    """BCGS-PIP+ keeps O(eps) orthogonality while eps*kappa^2 <= 1/2."""
    A = dev(inputs.stewart(11 + int(np.log10(kappa)), N, M, kappa))
    out, e, r = run(P, A, "cholqr2")
    assert out["t_list"] == [S] * (M // S)
    assert e < 1e-13 and r < 1e-14, (e, r)


def test_cholqr2_breaks_beyond_threshold(P):
    """kappa = 1e12 (eps*kappa^2 ~ 2e8): BCGS-PIP+ cannot deliver TSQR's result — it either
    loses rank (the Gram-based factor deflates) or loses orthogonality; TSQR does neither."""
    A = dev(inputs.stewart(23, N, M, 1e12))
    out_c, e_c, _ = run(P, A, "cholqr2")
    out_t, e_t, _ = run(P, A, "tsqr", block_rows=256, defl_tol=1e-300)
    assert sum(out_t["t_list"]) == M and e_t < 1e-13
    assert sum(out_c["t_list"]) < M or e_c > 1e-10, (out_c["t_list"], e_c)


def test_pip_error_grows_like_kappa_squared(P):
    """Single-pass BCGS-PIP: e_perp = O(eps kappa^2) (fig:kappa a)."""
    e = {}
    for kappa in (1e3, 1e5):
        A = dev(inputs.stewart(31, N, M, kappa))
        _, e[kappa], _ = run(P, A, "cholqr2", single_pass=True)
    ratio = e[1e5] / e[1e3]
    assert 1e2 < ratio < 1e6, (e, ratio)  # kappa^2 ratio is 1e4


def test_table1b_partition_invariance(P):
    """Errors do not depend on the number of subproblems: leaf blocks of
    256 .. 1536 rows (256 .. 43 leaves, 3 .. 2 tree levels) all give O(eps)."""
    A = dev(inputs.stewart(41, N, M, 1e4))
    errs = []
    for nb in (256, 512, 1024, 1536):
        out, e, r = run(P, A, "tsqr", block_rows=nb)
        assert e < 1e-13 and r < 1e-14, (nb, e, r)
        errs.append(e)
    assert max(errs) / min(errs) < 20.0, errs
