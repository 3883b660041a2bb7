/*
 * pqr_support.h — support kernels of libpqr.so that are not part of the PQR hot path but
 * are needed by its consumers (BASELINE configs[2], the block Arnoldi sequence of
 * PAPER.md:L184-208, Alg. 1).  Device pointers, column-major, ordered on `stream`
 * (cudaStream_t, NULL = default); the call does not synchronise.  Return codes as in pqr.h.
 */
#ifndef PQR_SUPPORT_H
#define PQR_SUPPORT_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* Y = A V for the 7-point Laplacian on an nx x ny x nz grid with homogeneous Dirichlet
 * boundaries, unscaled (6 on the diagonal, -1 for every existing neighbour; R10).
 * Row index = i + nx*(j + ny*l).  V, Y: (nx*ny*nz) x s (ldv, ldy >= rows), 1 <= s <= 16;
 * Y must not alias V. */
int pqr_laplacian7_apply(int nx, int ny, int nz, int s, const double* V, int64_t ldv, double* Y, int64_t ldy,
                         void* stream);

#ifdef __cplusplus
}
#endif
#endif
