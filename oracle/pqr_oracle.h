/*
 * PARITY ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct host implementation (fp64, C) of what the
 * PQR hot path computes, written from the paper (arXiv 2204.13393, PAPER.md).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load it.  It shares no code, header, table or
 * helper with the CUDA library (paper_2204_13393_b200/csrc, include/pqr.h).
 *
 * Storage: every matrix is column-major with an explicit leading dimension
 * (LAPACK convention).  All functions return 0 on success, <0 on error.
 *
 * Readings of the paper used here are listed in DESIGN.md §"Readings".
 */
#ifndef PQR_ORACLE_H
#define PQR_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Definition of the PQR problem (§1 Eq. (1)) solved by the
 * Householder method (§2.2 Eq. (hh), Alg. 6) applied to all
 * k+s columns of A = [Q X], column by column, with in-order deflation:
 * column j >= k is deflated when its remaining norm lambda <= tau_abs
 * (reading R3 in DESIGN.md; callers pass tau_abs = defl_tol * ||X||_F).
 * Outputs are sign-canonicalised so every pivot of R is positive
 * (reading R6), which makes P = Q^T X, and N (t x s row echelon) and U (n x t)
 * unique.  Rows t..s-1 of N are zero-filled.  dependent[c] = 1 when column c
 * of X was deflated (may be NULL).  diag_q_err (may be NULL) receives
 * ||R[0:k,0:k] - I||_F after canonicalisation.  Uses OpenMP over columns. */
int orc_householder_pqr(int64_t n, int k, int s,
                        const double* Q, int64_t ldq,
                        const double* X, int64_t ldx,
                        double tau_abs,
                        double* U, int64_t ldu,
                        double* P, int64_t ldp,
                        double* N, int64_t ldn,
                        int* t, int* dependent, double* diag_q_err);

/* Step a1: W = [Q X]^T X, a (k+s) x s matrix; rows 0..k-1 are P = Q^T X and
 * rows k..k+s-1 are G = X^T X, "computed at once" (Alg. 7).
 * Plain dot products with pairwise summation. */
int orc_gram(int64_t n, int k, int s,
             const double* Q, int64_t ldq, const double* X, int64_t ldx,
             double* W, int64_t ldw);

/* Step a3: S = G - P^T P and the Cholesky factorisation N^T N = S
 * (PAPER.md:L474, L494), written as an in-order (unpivoted) Cholesky that
 * skips a column whose pivot d_j = S_jj - sum_i N_ij^2 satisfies
 * d_j <= max(tau_abs2, eta_rel * G_jj)  (reading R3b).  The result is the
 * t x s row-echelon N of PAPER.md:L119 with positive pivots; piv[i] is the
 * column of row i's pivot (i < t).  W is as returned by orc_gram. */
int orc_cholesky_deflate(int k, int s, const double* W, int64_t ldw,
                         double tau_abs2, double eta_rel,
                         double* N, int64_t ldn, int* t, int* piv);

/* Step a4: U = (X - Q P) N_J^{-1} (Alg. 7 line 3), with
 * N_J the t x t upper-triangular submatrix of N on the pivot columns piv[].
 * Written as: form Y = X - Q P explicitly, then forward substitution per row. */
int orc_update(int64_t n, int k, int s,
               const double* Q, int64_t ldq, const double* X, int64_t ldx,
               const double* P, int64_t ldp, const double* N, int64_t ldn,
               int t, const int* piv, double* U, int64_t ldu);

/* Alg. 7 (BCGS-PIP): orc_gram -> orc_cholesky_deflate ->
 * orc_update, in that order. */
int orc_bcgs_pip(int64_t n, int k, int s,
                 const double* Q, int64_t ldq, const double* X, int64_t ldx,
                 double tau_abs2, double eta_rel,
                 double* U, int64_t ldu, double* P, int64_t ldp,
                 double* N, int64_t ldn, int* t, int* piv);

/* Alg. 8 (BCGS-PIP+): BCGS-PIP on [Q X] giving U1,P1,N1,
 * BCGS-PIP on [Q U1] giving U,P2,N2, then the recombination
 * P = P1 + P2 N1, N = N2 N1 (reading R1: the printed "P = P1 N2 + P2,
 * N = N2 + N1 N2" of PAPER.md:L527 is inconsistent with the two factorisations;
 * the algebra [Q X] = [Q U1][I P1;0 N1] = [Q U][I P2;0 N2][I P1;0 N1] gives this).
 * Deflation is decided in the first pass only: the second pass runs with
 * tau_abs2 = 0 and eta_rel = 0 (it drops a column only if d_j <= 0). */
int orc_bcgs_pip_plus(int64_t n, int k, int s,
                      const double* Q, int64_t ldq, const double* X, int64_t ldx,
                      double tau_abs2, double eta_rel,
                      double* U, int64_t ldu, double* P, int64_t ldp,
                      double* N, int64_t ldn, int* t, int* piv);

/* Y = Q C (n x m), Q n x k, C k x m: the stage-2 product "QC with
 * C in R^{(k+s) x m}".  Plain dot products. */
int orc_matmul(int64_t n, int k, int m, const double* Q, int64_t ldq,
               const double* C, int64_t ldc, double* Y, int64_t ldy);

/* Householder QR of a local block, Alg. 6 restricted to k = 0 on an n x m
 * matrix A (in place): on return A holds the paper's reflectors v_i (unit
 * norm) below/at row i of column i, rdiag[i] = sigma*lambda
 * = N_ii with the paper's sign (sigma = -sgn, sgn(0) = +1; NOT canonicalised),
 * and the strictly upper part of A holds R.  Zero-norm columns get the
 * identity reflector (v = 0) and rdiag = 0 (reading R4).  Used to pin the
 * TSQR local-block kernel (§8(a) a6/a9). */
int orc_hh_local(int64_t n, int m, double* A, int64_t lda, double* rdiag);

/* Apply Q_m = H_0 ... H_{m-1} (reflectors as produced by orc_hh_local) to
 * C (n x c) in place: C <- H_0 (H_1 (... H_{m-1} C)).  trans = 1 applies
 * Q_m^T = H_{m-1} ... H_0 instead. */
int orc_hh_apply(int64_t n, int m, const double* V, int64_t ldv,
                 int trans, int c, double* C, int64_t ldc);

/* Number of OpenMP threads the oracle uses (1 when built without OpenMP). */
int orc_num_threads(void);

#ifdef __cplusplus
}
#endif
#endif
