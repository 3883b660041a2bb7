/*
 * pqr_steps.h — step-level entry points of libpqr.so, one per row of the hot path
 * (SURVEY.md §8(a)), exported so each step can be checked against its oracle
 * function in isolation.  They launch exactly the kernels pqr_project_normalize
 * launches.  All matrix pointers are DEVICE pointers (column-major, ld >= rows);
 * each call allocates its own scratch, runs on `stream` (cudaStream_t, NULL =
 * default) and synchronises it before returning.  Return codes as in pqr.h.
 */
#ifndef PQR_STEPS_H
#define PQR_STEPS_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* a1: W = [Q X]^T X, (k+s) x s (ldw >= k+s): rows 0..k-1 are P = Q^T X, rows k.. are
 * G = X^T X (Alg. 7 line 1).  1 <= s <= 16, k + s <= 160. */
int pqr_step_gram(int64_t n, int k, int s, const double* Q, int64_t ldq, const double* X, int64_t ldx,
                  double* W, int ldw, void* stream);

/* a3: from W (device, (k+s) x s): S = G - P^T P, in-order Cholesky with deflation
 * (pivot d_j <= max(tol2_rel * trace(G), eta * G_jj) deflates column j; R3b),
 * giving N (s x s, ldn >= s, row echelon, rows >= t zero) and the update operator
 * M = [-P_J N_J^{-1}; E_J N_J^{-1}] ((k+s) x s, ldm >= k+s, columns >= t zero)
 * (PAPER.md:L474, L494-495).  *t_host and piv_host[0..s-1] (pivot columns, -1 past t)
 * are HOST outputs; piv_host may be NULL. */
int pqr_step_factor(int k, int s, const double* W, int ldw, double tol2_rel, double eta,
                    double* N, int ldn, double* M, int ldm, int* t_host, int* piv_host, void* stream);

/* a4: U = [Q X] M (n x s, ldu >= n), columns >= t written as zero
 * ("U = XN^{-1} - QPN^{-1}"). */
int pqr_step_update(int64_t n, int k, int s, const double* Q, int64_t ldq, const double* X, int64_t ldx,
                    const double* M, int ldm, int t, double* U, int64_t ldu, void* stream);

#ifdef __cplusplus
}
#endif
#endif
