"""Pins of the CPU oracle against things other than itself (CPU-only, -m "not gpu").

Each test names what fixes the expected value: brute force in 50-digit decimal
arithmetic, a closed form of the paper, a library routine for a special case,
a worked example (tests/golden/), a manufactured solution, or the magnitudes
the paper prints (Table 1a).
"""
import json
import math
import os
from decimal import Decimal, getcontext

import numpy as np
import pytest

from paper_2204_13393_b200 import inputs

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def residual(Q, X, U, P, N):
    """||[Q X] - [Q U][I P; 0 N]||_F / ||[Q X]||_F  (Eq. (1))."""
    t = U.shape[1]
    lhs = np.hstack([Q, X])
    rhs = np.hstack([Q, Q @ P + U @ N[:t]])
    return np.linalg.norm(lhs - rhs) / np.linalg.norm(lhs)


# ---------------------------------------------------------------------------
# brute force: 50-digit Gram-Schmidt QR of [Q X] (Python decimal)
# ---------------------------------------------------------------------------
def decimal_qr(A):
    getcontext().prec = 50
    n, m = A.shape
    cols = [[Decimal(float(A[i, j])) for i in range(n)] for j in range(m)]
    qs = []
    R = [[Decimal(0)] * m for _ in range(m)]
    for j in range(m):
        a = cols[j][:]
        for _ in range(2):  # modified Gram-Schmidt, twice
            for i, q in enumerate(qs):
                r = sum(qq * aa for qq, aa in zip(q, a))
                R[i][j] += r
                a = [aa - r * qq for aa, qq in zip(a, q)]
        nrm = sum(aa * aa for aa in a).sqrt()
        R[j][j] = nrm
        qs.append([aa / nrm for aa in a])
    Qd = np.array([[float(q[i]) for q in qs] for i in range(n)])
    Rd = np.array([[float(R[i][j]) for j in range(m)] for i in range(m)])
    return Qd, Rd


@pytest.mark.parametrize("n,k,s,seed", [(6, 2, 2, 1), (9, 3, 2, 2), (12, 1, 4, 3), (7, 0, 3, 4), (12, 4, 1, 5)])
def test_oracle_vs_decimal_bruteforce(orc, n, k, s, seed):
    Q = inputs.orthonormal(seed, n, k)
    X = inputs.gaussian(seed + 100, n, s)
    Qd, Rd = decimal_qr(np.hstack([Q, X]))
    out = orc.householder_pqr(Q, X)
    assert out["t"] == s
    assert np.allclose(out["P"], Rd[:k, k:], rtol=0, atol=1e-14 * max(1, np.abs(X).max()))
    assert np.allclose(out["N"], Rd[k:, k:], rtol=0, atol=1e-14 * max(1, np.abs(X).max()))
    assert np.allclose(out["U"], Qd[:, k:], rtol=0, atol=1e-14)


# ---------------------------------------------------------------------------
# worked examples (tests/golden/spec_examples.json, each with its citation)
# ---------------------------------------------------------------------------
def load_golden():
    with open(os.path.join(GOLDEN, "spec_examples.json")) as f:
        return json.load(f)


def test_golden_345(orc):
    ex = load_golden()["qr_3_4"]
    out = orc.householder_pqr(None, np.array(ex["X"], dtype=float))
    assert out["t"] == 1
    assert np.allclose(out["U"][:, 0], ex["U"], atol=1e-15)
    assert np.allclose(out["N"], ex["N"], atol=1e-15)


def test_golden_cholesky(orc):
    g = load_golden()
    ex = g["cholesky_4_2_5"]
    N, t, piv = orc.cholesky_deflate(np.array(ex["G"], dtype=float), k=0)
    assert t == 2 and piv == [0, 1]
    assert np.array_equal(N, np.array(ex["N"], dtype=float))
    ex = g["cholesky_not_pd"]
    N, t, piv = orc.cholesky_deflate(np.array(ex["G"], dtype=float), k=0)
    assert t == ex["t"] and piv == ex["piv"]
    assert np.allclose(N[0], ex["N_row0"])
    assert np.all(N[1] == 0)


def test_golden_householder_e1(orc):
    ex = load_golden()["hh_e1"]
    A = np.array(ex["X"], dtype=float).reshape(-1, 1)
    V, rd = orc.hh_local(A)
    assert rd[0] == ex["N_paper_sign"]  # sigma = -sgn(1) = -1
    U = orc.hh_apply(V, 1, np.eye(A.shape[0])[:, :1])
    assert np.allclose(U[:, 0], ex["U_paper_sign"], atol=1e-15)
    # canonicalised form used by the PQR outputs
    out = orc.householder_pqr(None, A)
    assert np.allclose(out["N"], [[1.0]]) and np.allclose(out["U"][:, 0], -np.array(ex["U_paper_sign"]))


def test_golden_orthonormal_input_identity(orc):
    # "orthonormal A -> Q = A, R = I": k = 0, X orthonormal
    X = inputs.orthonormal(11, 40, 5)
    out = orc.householder_pqr(None, X)
    assert out["t"] == 5
    assert np.allclose(out["N"], np.eye(5), atol=1e-14)
    assert np.allclose(out["U"], X, atol=1e-14)


# ---------------------------------------------------------------------------
# closed forms of the paper (§3)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("n,k,s", [(500, 12, 4), (2000, 40, 8), (257, 0, 5)])
def test_closed_forms(orc, n, k, s):
    Q = inputs.orthonormal(n + k, n, k)
    X = inputs.gaussian(n + s, n, s)
    out = orc.householder_pqr(Q, X)
    P, N, U = out["P"], out["N"], out["U"]
    # P = Q^T X (unique), via numpy's matmul
    assert rel(P, Q.T @ X) < 1e-13
    # N^T N = X^T X - P^T P, N upper triangular with positive diagonal
    S = X.T @ X - P.T @ P
    assert rel(N.T @ N, S) < 1e-13
    assert np.allclose(np.tril(N, -1), 0) and np.all(np.diag(N) > 0)
    # Cholesky uniqueness: N = chol(S)^T (numpy/LAPACK)
    assert rel(N, np.linalg.cholesky(S).T) < 1e-11
    # U = (X - Q P) N^{-1}
    assert rel(U, np.linalg.solve(N.T, (X - Q @ P).T).T) < 1e-11
    assert residual(Q, X, U, P, N) < 1e-14
    assert np.linalg.norm(Q.T @ U) < 1e-13
    assert np.linalg.norm(np.eye(s) - U.T @ U) < 1e-13


def test_k0_reduces_to_library_qr(orc):
    X = inputs.gaussian(5, 300, 6)
    out = orc.householder_pqr(None, X)
    q, r = np.linalg.qr(X)
    d = np.sign(np.diag(r))
    assert rel(out["N"], d[:, None] * r) < 1e-13
    assert rel(out["U"], q * d) < 1e-13


# ---------------------------------------------------------------------------
# manufactured solutions: X = Q C + Y D  ->  P = C, N = D, U = Y exactly
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("n,k,s", [(1000, 16, 4), (3000, 64, 8), (800, 20, 16)])
def test_manufactured(orc, n, k, s):
    m = inputs.manufactured(77 + s, n, k, s)
    out = orc.householder_pqr(m["Q"], m["X"])
    assert out["t"] == s
    assert rel(out["P"], m["C"]) < 1e-13
    assert rel(out["N"], m["D"]) < 1e-13
    assert rel(out["U"], m["Y"]) < 1e-12
    assert out["diag_q_err"] < 1e-13


def test_special_cases(orc):
    n, k, s = 600, 10, 4
    m = inputs.manufactured(5, n, k, s)
    # X orthogonal to Q -> P = 0
    X = m["Y"] @ m["D"]
    out = orc.householder_pqr(m["Q"], X)
    assert np.linalg.norm(out["P"]) < 1e-12 * np.linalg.norm(X)
    # X orthonormal and orthogonal to Q -> N = I, U = X
    out = orc.householder_pqr(m["Q"], m["Y"])
    assert np.allclose(out["N"], np.eye(s), atol=1e-13) and np.allclose(out["U"], m["Y"], atol=1e-13)
    # X in span(Q) -> t = 0, P = C, N = 0
    X = m["Q"] @ m["C"]
    out = orc.householder_pqr(m["Q"], X)
    assert out["t"] == 0 and rel(out["P"], m["C"]) < 1e-13 and np.all(out["N"] == 0)
    assert all(out["dependent"])


def test_duplicate_column_deflates(orc):
    n, k, s = 500, 6, 4
    Q = inputs.orthonormal(3, n, k)
    X = inputs.gaussian(4, n, s)
    X[:, 2] = X[:, 0]  # duplicated column -> t = s - 1
    out = orc.householder_pqr(Q, X)
    assert out["t"] == s - 1
    assert out["dependent"] == [False, False, True, False]
    t = out["t"]
    N = out["N"]
    # row-echelon: pivots at columns 0, 1, 3; column 2 equals column 0 of N
    assert N[0, 0] > 0 and N[1, 1] > 0 and N[2, 3] > 0 and abs(N[2, 2]) == 0
    assert np.allclose(N[:, 2], N[:, 0], atol=1e-12)
    assert np.all(N[t:] == 0)
    assert residual(Q, X, out["U"], out["P"], N) < 1e-14


def test_deflation_config_small(orc):
    n, k, s = 4000, 24, 16
    Q, X = inputs.deflation_inputs(9, n, k, s)
    out = orc.householder_pqr(Q, X)
    assert out["t"] == 14
    assert [c for c in range(s) if out["dependent"][c]] == [5, 11]
    assert residual(Q, X, out["U"], out["P"], out["N"]) < 1e-14
    assert np.linalg.norm(Q.T @ out["U"], 2) < 1e-13
    assert np.linalg.norm(np.eye(14) - out["U"].T @ out["U"], 2) < 1e-13


# ---------------------------------------------------------------------------
# step functions vs library routines / closed forms
# ---------------------------------------------------------------------------
def test_gram_vs_numpy(orc):
    Q = inputs.orthonormal(1, 3001, 17)
    X = inputs.gaussian(2, 3001, 5)
    W = orc.gram(Q, X)
    assert rel(W, np.hstack([Q, X]).T @ X) < 1e-14


def test_cholesky_vs_lapack(orc):
    Q = inputs.orthonormal(1, 1000, 9)
    X = inputs.gaussian(2, 1000, 6)
    W = np.hstack([Q, X]).T @ X
    N, t, piv = orc.cholesky_deflate(W, k=9)
    S = W[9:] - W[:9].T @ W[:9]
    assert t == 6 and piv == list(range(6))
    assert rel(N, np.linalg.cholesky(S).T) < 1e-13


def test_update_vs_solve(orc):
    Q = inputs.orthonormal(1, 700, 9)
    X = inputs.gaussian(2, 700, 6)
    P = Q.T @ X
    N = np.linalg.cholesky(X.T @ X - P.T @ P).T
    U = orc.update(Q, X, P, N, 6, list(range(6)))
    assert rel(U, np.linalg.solve(N.T, (X - Q @ P).T).T) < 1e-13


def test_matmul_vs_numpy(orc):
    Q = inputs.gaussian(1, 513, 7)
    C = inputs.gaussian(2, 7, 3)
    assert rel(orc.matmul(Q, C), Q @ C) < 1e-15


def test_hh_local_vs_lapack(orc):
    A = inputs.gaussian(3, 200, 12)
    V, rd = orc.hh_local(A)
    _, r = np.linalg.qr(A)
    R = np.triu(V[:12])
    np.fill_diagonal(R, rd)
    assert rel(np.abs(R), np.abs(r)) < 1e-13
    # Q^T A = [R; 0]
    QtA = orc.hh_apply(V, 12, A, trans=True)
    assert rel(QtA[:12], R) < 1e-13 and np.linalg.norm(QtA[12:]) < 1e-12
    # Q (Q^T A) = A
    assert rel(orc.hh_apply(V, 12, QtA), A) < 1e-13


def test_pip_plus_recombination_residual(orc):
    # reading R1: P = P1 + P2 N1, N = N2 N1 satisfies Eq. (1); the printed formula would not
    n, k, s = 2000, 30, 6
    Q, X = inputs.projected_inputs(12, n, k, s, ratio=1e-3)
    out = orc.bcgs_pip_plus(Q, X)
    assert out["t"] == s
    assert residual(Q, X, out["U"], out["P"], out["N"]) < 1e-14
    hh = orc.householder_pqr(Q, X)
    assert rel(out["P"], hh["P"]) < 1e-12 and rel(out["N"], hh["N"]) < 1e-10 and rel(out["U"], hh["U"]) < 1e-10


# ---------------------------------------------------------------------------
# paper-printed magnitudes (Table 1a level 0) via Alg. 2
# ---------------------------------------------------------------------------
def block_column_qr(solve, A, s):
    n, m = A.shape
    Q = np.zeros((n, 0), order="F")
    for b in range(0, m, s):
        out = solve(Q, np.asfortranarray(A[:, b:b + s]))
        Q = np.asfortranarray(np.hstack([Q, out["U"]]))
    return Q


def test_table1a_magnitudes(orc):
    A = inputs.stewart(2022, 4096, 32, 1e4)
    e = {}
    e["pip"] = block_column_qr(lambda Q, X: orc.bcgs_pip(Q, X), A, 4)
    e["pip+"] = block_column_qr(lambda Q, X: orc.bcgs_pip_plus(Q, X), A, 4)
    e["hh"] = block_column_qr(lambda Q, X: orc.householder_pqr(Q, X, tau_abs=0.0), A, 4)
    err = {key: np.linalg.norm(np.eye(q.shape[1]) - q.T @ q) for key, q in e.items()}
    # paper: PIP 9.97e-10, PIP+ 2.33e-15, HH 9.07e-15 (orders of magnitude only)
    assert 1e-12 < err["pip"] < 1e-6, err
    assert err["pip+"] < 1e-13, err
    assert err["hh"] < 1e-13, err


# ---------------------------------------------------------------------------
# the deflation branch in the middle of a block (a column deflates, later columns
# still pivot): orc_cholesky_deflate, orc_update with non-identity pivots and
# orc_bcgs_pip_plus with t1 < s.  Pins: N^T N = S on every column (the
# defining identity of the row-echelon N of P:L119), LAPACK Cholesky of S on the
# pivot columns (uniqueness with positive pivots), numpy solves, Q^T X.
# ---------------------------------------------------------------------------
def _dup_middle(n=900, k=7, s=8, seed=31):
    Q = inputs.orthonormal(seed, n, k)
    X = inputs.gaussian(seed + 1, n, s)
    X[:, 5] = X[:, 1]  # column 5 duplicates column 1: in-order deflation drops column 5 only
    return Q, X


def test_cholesky_deflate_mid_block(orc):
    Q, X = _dup_middle()
    k, s = Q.shape[1], X.shape[1]
    W = np.hstack([Q, X]).T @ X
    S = W[k:] - W[:k].T @ W[:k]
    nx2 = float(np.linalg.norm(X)) ** 2
    N, t, piv = orc.cholesky_deflate(W, k=k, tau_abs2=(1e-12) ** 2 * nx2, eta_rel=1e-13)
    J = [0, 1, 2, 3, 4, 6, 7]
    assert t == 7 and piv == J
    # row echelon: row i is zero left of its pivot column, pivots positive, rows >= t zero
    for i, pc in enumerate(piv):
        assert np.all(N[i, :pc] == 0) and N[i, pc] > 0
    assert np.all(N[t:] == 0)
    # the deflated column is the duplicate's column
    assert np.allclose(N[:, 5], N[:, 1], rtol=0, atol=1e-12 * np.abs(N).max())
    # N^T N = S on all columns (including the deflated one)
    assert rel(N.T @ N, S) < 1e-13
    # N_J = chol(S_JJ)^T (LAPACK), the pivot-column submatrix
    assert rel(N[:t][:, J], np.linalg.cholesky(S[np.ix_(J, J)]).T) < 1e-12


def test_update_nonidentity_pivots(orc):
    Q, X = _dup_middle()
    k = Q.shape[1]
    P = Q.T @ X
    J = [0, 1, 2, 3, 4, 6, 7]
    S = X.T @ X - P.T @ P
    NJ = np.linalg.cholesky(S[np.ix_(J, J)]).T  # t x t on the pivot columns
    N = np.zeros((8, 8))
    N[:7] = np.linalg.solve(NJ.T, S[J])  # full row-echelon N (N_J^T N = S[J, :])
    U = orc.update(Q, X, P, N, 7, J)
    want = np.linalg.solve(NJ.T, (X - Q @ P)[:, J].T).T
    assert rel(U, want) < 1e-12
    assert np.linalg.norm(np.eye(7) - U.T @ U) < 1e-10 and np.linalg.norm(Q.T @ U) < 1e-12
    assert k == 7


def test_bcgs_pip_plus_deflating(orc):
    Q, X = _dup_middle()
    s = X.shape[1]
    nx2 = float(np.linalg.norm(X)) ** 2
    out = orc.bcgs_pip_plus(Q, X, tau_abs2=(1e-12) ** 2 * nx2, eta_rel=1e-13)
    t = out["t"]
    assert t == s - 1 and out["piv"] == [0, 1, 2, 3, 4, 6, 7]
    assert rel(out["P"], Q.T @ X) < 1e-13
    assert residual(Q, X, out["U"], out["P"], out["N"]) < 1e-14
    assert np.linalg.norm(Q.T @ out["U"], 2) < 1e-13
    assert np.linalg.norm(np.eye(t) - out["U"].T @ out["U"], 2) < 1e-13
    N = out["N"]
    for i, pc in enumerate(out["piv"]):
        assert np.all(N[i, :pc] == 0) and N[i, pc] > 0
    assert np.all(N[t:] == 0)
    # agrees with the Householder oracle (the same in-order deflation, reading R3)
    hh = orc.householder_pqr(Q, X)
    assert hh["t"] == t and rel(out["N"], hh["N"]) < 1e-10 and rel(out["U"], hh["U"]) < 1e-10
