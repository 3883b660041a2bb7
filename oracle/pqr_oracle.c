/*
 * PARITY ORACLE — TEST INFRASTRUCTURE ONLY (see pqr_oracle.h).
 *
 * Plain fp64 C, compiled with -O2 -fno-fast-math -ffp-contract=off.  Every
 * function follows a passage of PAPER.md (arXiv 2204.13393) step by step; no
 * blocking, fusion or reordering beyond what that passage states.  Sums are
 * pairwise (a fixed, deterministic order).  OpenMP is used only to run
 * independent columns concurrently; each column's arithmetic is serial, so
 * results do not depend on the thread count.
 */
#include "pqr_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define IDX(i, j, ld) ((int64_t)(i) + (int64_t)(j) * (int64_t)(ld))

/* pairwise dot product: plain loop below 64 elements, halves above */
static double pw_dot(const double* a, const double* b, int64_t len) {
  if (len <= 64) {
    double acc = 0.0;
    for (int64_t i = 0; i < len; ++i) acc += a[i] * b[i];
    return acc;
  }
  int64_t h = len / 2;
  return pw_dot(a, b, h) + pw_dot(a + h, b + h, len - h);
}

int orc_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ---------------------------------------------------------------------- */
/* Householder PQR of [Q X]  (Alg. 6; Eq. (1))   */
/* ---------------------------------------------------------------------- */
int orc_householder_pqr(int64_t n, int k, int s,
                        const double* Q, int64_t ldq,
                        const double* X, int64_t ldx,
                        double tau_abs,
                        double* U, int64_t ldu,
                        double* P, int64_t ldp,
                        double* N, int64_t ldn,
                        int* t, int* dependent, double* diag_q_err) {
  if (n < 0 || k < 0 || s < 0 || n < k || !t) return -1;
  if (k > 0 && (!Q || ldq < n)) return -1;
  if (s > 0 && (!X || ldx < n)) return -1;
  const int m = k + s;
  double* A = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1) * (size_t)(m > 0 ? m : 1));
  double* rdiag = (double*)calloc((size_t)(m > 0 ? m : 1), sizeof(double));
  int* pivcol = (int*)malloc(sizeof(int) * (size_t)(m > 0 ? m : 1));
  int* rows_before = (int*)malloc(sizeof(int) * (size_t)(m > 0 ? m : 1)); /* r when column j was visited */
  if (!A || !rdiag || !pivcol || !rows_before) { free(A); free(rdiag); free(pivcol); free(rows_before); return -3; }
  for (int j = 0; j < k; ++j) memcpy(&A[IDX(0, j, n)], &Q[IDX(0, j, ldq)], sizeof(double) * (size_t)n);
  for (int j = 0; j < s; ++j) memcpy(&A[IDX(0, k + j, n)], &X[IDX(0, j, ldx)], sizeof(double) * (size_t)n);
  if (dependent) for (int c = 0; c < s; ++c) dependent[c] = 0;

  int r = 0; /* number of reflectors (accepted rows of R) so far */
  int err = 0;
  for (int j = 0; j < m; ++j) {
    rows_before[j] = r;
    int64_t len = n - r;
    double* u = &A[IDX(r, j, n)];
    /* lambda = ||u~[r:n]||  (Alg. 6 line 5, index reading R2) */
    double lam = len > 0 ? sqrt(pw_dot(u, u, len)) : 0.0;
    if (j >= k && lam <= tau_abs) {           /* deflation (reading R3) */
      if (dependent) dependent[j - k] = 1;
      continue;
    }
    if (lam == 0.0) { err = -4; break; }      /* a Q column of zero norm: Q not orthonormal */
    double sigma = (u[0] >= 0.0) ? -1.0 : 1.0; /* sigma = -sgn(u0), sgn(0) = +1 (line 6) */
    rdiag[r] = sigma * lam;                     /* N_ii = sigma*lambda (line 7) */
    u[0] -= sigma * lam;                        /* v~ = u - sigma*lambda*e1 (line 8) */
    double nv = sqrt(pw_dot(u, u, len));
    for (int64_t i = 0; i < len; ++i) u[i] /= nv; /* v = v~/||v~|| (line 9) */
    pivcol[r] = j;
    /* apply H = I - 2 v v^T to the remaining columns (rows r:n) */
#pragma omp parallel for schedule(dynamic, 1)
    for (int jj = j + 1; jj < m; ++jj) {
      double* a = &A[IDX(r, jj, n)];
      double w = pw_dot(u, a, len);
      for (int64_t i = 0; i < len; ++i) a[i] -= 2.0 * w * u[i];
    }
    ++r;
  }
  if (err) { free(A); free(rdiag); free(pivcol); free(rows_before); return err; }
  const int tt = r - k;
  *t = tt;

  /* sign canonicalisation (reading R6): pivot of every row made positive */
  double* sgn = (double*)malloc(sizeof(double) * (size_t)(r > 0 ? r : 1));
  for (int i = 0; i < r; ++i) sgn[i] = rdiag[i] < 0.0 ? -1.0 : 1.0;

  /* R entry (i, j) for i < r: above the pivot row: A(i,j); at pivot: rdiag;
   * below the rows existing when column j was visited: 0. */
#define R_ENTRY(i, j) ((i) < rows_before[j] ? A[IDX(i, j, n)] : \
                       (((i) == rows_before[j] && (i) < r && pivcol[i] == (j)) ? rdiag[i] : 0.0))
  if (P) for (int c = 0; c < s; ++c) for (int i = 0; i < k; ++i)
    P[IDX(i, c, ldp)] = sgn[i] * R_ENTRY(i, k + c);
  if (N) for (int c = 0; c < s; ++c) for (int i = 0; i < s; ++i)
    N[IDX(i, c, ldn)] = (i < tt) ? sgn[k + i] * R_ENTRY(k + i, k + c) : 0.0;
  if (diag_q_err) {
    double e = 0.0;
    for (int j = 0; j < k; ++j) for (int i = 0; i < k; ++i) {
      double d = sgn[i] * R_ENTRY(i, j) - (i == j ? 1.0 : 0.0);
      e += d * d;
    }
    *diag_q_err = sqrt(e);
  }
#undef R_ENTRY

  /* U = columns k..k+t-1 of Q^ = H_0 ... H_{r-1} I[:,0:r]:
   * y = e_i, then apply H_i, H_{i-1}, ..., H_0 (H_j e_i = e_i for j > i). */
  if (U) {
#pragma omp parallel for schedule(dynamic, 1)
    for (int c = 0; c < tt; ++c) {
      int i = k + c;
      double* y = &U[IDX(0, c, ldu)];
      for (int64_t q = 0; q < n; ++q) y[q] = 0.0;
      y[i] = 1.0;
      for (int jr = i; jr >= 0; --jr) {
        const double* v = &A[IDX(jr, pivcol[jr], n)];
        int64_t len = n - jr;
        double w = pw_dot(v, &y[jr], len);
        for (int64_t q = 0; q < len; ++q) y[jr + q] -= 2.0 * w * v[q];
      }
      for (int64_t q = 0; q < n; ++q) y[q] *= sgn[i];
    }
  }
  free(sgn); free(A); free(rdiag); free(pivcol); free(rows_before);
  return 0;
}

/* ---------------------------------------------------------------------- */
/* Step a1: W = [Q X]^T X                           */
/* ---------------------------------------------------------------------- */
int orc_gram(int64_t n, int k, int s,
             const double* Q, int64_t ldq, const double* X, int64_t ldx,
             double* W, int64_t ldw) {
  if (n < 0 || k < 0 || s < 0 || ldw < k + s) return -1;
#pragma omp parallel for collapse(2) schedule(dynamic, 1)
  for (int c = 0; c < s; ++c)
    for (int j = 0; j < k + s; ++j) {
      const double* a = j < k ? &Q[IDX(0, j, ldq)] : &X[IDX(0, j - k, ldx)];
      W[IDX(j, c, ldw)] = pw_dot(a, &X[IDX(0, c, ldx)], n);
    }
  return 0;
}

/* ---------------------------------------------------------------------- */
/* Step a3: N^T N = G - P^T P, in-order Cholesky with deflation             */
/*                                                */
/* ---------------------------------------------------------------------- */
int orc_cholesky_deflate(int k, int s, const double* W, int64_t ldw,
                         double tau_abs2, double eta_rel,
                         double* N, int64_t ldn, int* t, int* piv) {
  if (k < 0 || s < 0 || ldw < k + s || !t) return -1;
  double* S = (double*)malloc(sizeof(double) * (size_t)(s > 0 ? s * s : 1));
  /* S = G - P^T P */
  for (int b = 0; b < s; ++b)
    for (int a = 0; a < s; ++a) {
      double ptp = 0.0;
      for (int i = 0; i < k; ++i) ptp += W[IDX(i, a, ldw)] * W[IDX(i, b, ldw)];
      S[a + b * s] = W[IDX(k + a, b, ldw)] - ptp;
    }
  for (int b = 0; b < s; ++b) for (int a = 0; a < s; ++a) N[IDX(a, b, ldn)] = 0.0;
  int r = 0;
  for (int j = 0; j < s; ++j) {
    /* entries N[i, j] for existing rows i < r: (S[p_i, j] - sum_{i'<i} N[i',p_i] N[i',j]) / N[i,p_i] */
    for (int i = 0; i < r; ++i) {
      int pc = piv[i];
      double acc = S[pc + j * s];
      for (int i2 = 0; i2 < i; ++i2) acc -= N[IDX(i2, pc, ldn)] * N[IDX(i2, j, ldn)];
      N[IDX(i, j, ldn)] = acc / N[IDX(i, pc, ldn)];
    }
    double d = S[j + j * s];
    for (int i = 0; i < r; ++i) d -= N[IDX(i, j, ldn)] * N[IDX(i, j, ldn)];
    double gjj = W[IDX(k + j, j, ldw)];
    double thr = tau_abs2 > eta_rel * gjj ? tau_abs2 : eta_rel * gjj;
    if (d <= thr) continue;                 /* deflated column: no new row */
    N[IDX(r, j, ldn)] = sqrt(d);
    piv[r] = j;
    ++r;
  }
  *t = r;
  free(S);
  return 0;
}

/* ---------------------------------------------------------------------- */
/* Step a4: U = (X - Q P) N_J^{-1}                   */
/* ---------------------------------------------------------------------- */
int orc_update(int64_t n, int k, int s,
               const double* Q, int64_t ldq, const double* X, int64_t ldx,
               const double* P, int64_t ldp, const double* N, int64_t ldn,
               int t, const int* piv, double* U, int64_t ldu) {
  if (n < 0 || k < 0 || s < 0 || t < 0 || t > s) return -1;
#pragma omp parallel for schedule(static)
  for (int64_t row = 0; row < n; ++row) {
    double y[256];
    /* Y[row, c] = X[row, c] - sum_i Q[row, i] P[i, c] */
    for (int c = 0; c < s; ++c) {
      double acc = X[IDX(row, c, ldx)];
      for (int i = 0; i < k; ++i) acc -= Q[IDX(row, i, ldq)] * P[IDX(i, c, ldp)];
      y[c] = acc;
    }
    /* U[row, :] N_J = Y[row, J]  ->  forward substitution over i */
    for (int i = 0; i < t; ++i) {
      int pc = piv[i];
      double acc = y[pc];
      for (int i2 = 0; i2 < i; ++i2) acc -= U[IDX(row, i2, ldu)] * N[IDX(i2, pc, ldn)];
      U[IDX(row, i, ldu)] = acc / N[IDX(i, pc, ldn)];
    }
  }
  return 0;
}

/* ---------------------------------------------------------------------- */
/* Alg. 7 and Alg. 8                                                         */
/* ---------------------------------------------------------------------- */
int orc_bcgs_pip(int64_t n, int k, int s,
                 const double* Q, int64_t ldq, const double* X, int64_t ldx,
                 double tau_abs2, double eta_rel,
                 double* U, int64_t ldu, double* P, int64_t ldp,
                 double* N, int64_t ldn, int* t, int* piv) {
  if (s > 256) return -1;
  int m = k + s;
  double* W = (double*)malloc(sizeof(double) * (size_t)(m > 0 ? m : 1) * (size_t)(s > 0 ? s : 1));
  int rc = orc_gram(n, k, s, Q, ldq, X, ldx, W, m);
  if (!rc) rc = orc_cholesky_deflate(k, s, W, m, tau_abs2, eta_rel, N, ldn, t, piv);
  if (!rc) for (int c = 0; c < s; ++c) for (int i = 0; i < k; ++i) P[IDX(i, c, ldp)] = W[IDX(i, c, m)];
  if (!rc) rc = orc_update(n, k, s, Q, ldq, X, ldx, P, ldp, N, ldn, *t, piv, U, ldu);
  free(W);
  return rc;
}

int orc_bcgs_pip_plus(int64_t n, int k, int s,
                      const double* Q, int64_t ldq, const double* X, int64_t ldx,
                      double tau_abs2, double eta_rel,
                      double* U, int64_t ldu, double* P, int64_t ldp,
                      double* N, int64_t ldn, int* t, int* piv) {
  if (s > 256) return -1;
  int sp = s > 0 ? s : 1, kp = k > 0 ? k : 1;
  double* U1 = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1) * (size_t)sp);
  double* P1 = (double*)malloc(sizeof(double) * (size_t)kp * (size_t)sp);
  double* N1 = (double*)calloc((size_t)sp * (size_t)sp, sizeof(double));
  double* P2 = (double*)malloc(sizeof(double) * (size_t)kp * (size_t)sp);
  double* N2 = (double*)calloc((size_t)sp * (size_t)sp, sizeof(double));
  int piv1[256], piv2[256], t1 = 0, t2 = 0;
  int64_t ldu1 = n > 0 ? n : 1;
  int rc = orc_bcgs_pip(n, k, s, Q, ldq, X, ldx, tau_abs2, eta_rel, U1, ldu1, P1, kp, N1, sp, &t1, piv1);
  /* second pass on [Q U1] (t1 columns); no new deflation decided here */
  if (!rc) rc = orc_bcgs_pip(n, k, t1, Q, ldq, U1, ldu1, 0.0, 0.0, U, ldu, P2, kp, N2, sp, &t2, piv2);
  if (!rc) {
    /* P = P1 + P2 N1  (k x s);  N = N2 N1 (t2 x s)   (reading R1) */
    for (int c = 0; c < s; ++c) {
      for (int i = 0; i < k; ++i) {
        double acc = P1[IDX(i, c, kp)];
        for (int q = 0; q < t1; ++q) acc += P2[IDX(i, q, kp)] * N1[IDX(q, c, sp)];
        P[IDX(i, c, ldp)] = acc;
      }
      for (int i = 0; i < s; ++i) {
        double acc = 0.0;
        if (i < t2) for (int q = 0; q < t1; ++q) acc += N2[IDX(i, q, sp)] * N1[IDX(q, c, sp)];
        N[IDX(i, c, ldn)] = acc;
      }
    }
    *t = t2;
    /* pivots of N = N2 N1: N2 is t1 x t1 upper triangular with positive diagonal
     * when t2 = t1, so N keeps N1's pivot columns */
    for (int i = 0; i < t2; ++i) piv[i] = piv1[piv2[i]];
  }
  free(U1); free(P1); free(N1); free(P2); free(N2);
  return rc;
}

/* ---------------------------------------------------------------------- */
/* Y = Q C   (stage-2 product)                          */
/* ---------------------------------------------------------------------- */
int orc_matmul(int64_t n, int k, int m, const double* Q, int64_t ldq,
               const double* C, int64_t ldc, double* Y, int64_t ldy) {
  if (n < 0 || k < 0 || m < 0) return -1;
#pragma omp parallel for schedule(static)
  for (int64_t row = 0; row < n; ++row)
    for (int c = 0; c < m; ++c) {
      double acc = 0.0;
      for (int i = 0; i < k; ++i) acc += Q[IDX(row, i, ldq)] * C[IDX(i, c, ldc)];
      Y[IDX(row, c, ldy)] = acc;
    }
  return 0;
}

/* ---------------------------------------------------------------------- */
/* Local Householder QR (Alg. 6 with k = 0) and reflector application        */
/* ---------------------------------------------------------------------- */
int orc_hh_local(int64_t n, int m, double* A, int64_t lda, double* rdiag) {
  if (n < m || m < 0) return -1;
  for (int j = 0; j < m; ++j) {
    int64_t len = n - j;
    double* u = &A[IDX(j, j, lda)];
    double lam = sqrt(pw_dot(u, u, len));
    if (lam == 0.0) {                        /* identity reflector (reading R4) */
      rdiag[j] = 0.0;
      continue;                              /* v = u = 0 already */
    }
    double sigma = (u[0] >= 0.0) ? -1.0 : 1.0;
    rdiag[j] = sigma * lam;
    u[0] -= sigma * lam;
    double nv = sqrt(pw_dot(u, u, len));
    for (int64_t i = 0; i < len; ++i) u[i] /= nv;
    for (int jj = j + 1; jj < m; ++jj) {
      double* a = &A[IDX(j, jj, lda)];
      double w = pw_dot(u, a, len);
      for (int64_t i = 0; i < len; ++i) a[i] -= 2.0 * w * u[i];
    }
  }
  return 0;
}

int orc_hh_apply(int64_t n, int m, const double* V, int64_t ldv,
                 int trans, int c, double* C, int64_t ldc) {
  if (n < m || m < 0 || c < 0) return -1;
  for (int col = 0; col < c; ++col) {
    double* y = &C[IDX(0, col, ldc)];
    for (int step = 0; step < m; ++step) {
      int j = trans ? step : m - 1 - step;   /* Q^T: H_0 first; Q: H_{m-1} first */
      const double* v = &V[IDX(j, j, ldv)];
      int64_t len = n - j;
      double w = pw_dot(v, &y[j], len);
      for (int64_t q = 0; q < len; ++q) y[j + q] -= 2.0 * w * v[q];
    }
  }
  return 0;
}
