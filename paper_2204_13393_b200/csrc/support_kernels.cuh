// support_kernels.cuh — operators used by the PQR consumers (not the hot path).
#pragma once
#include "common.cuh"

namespace pqr {

// Y = A V, A = 7-point Dirichlet Laplacian (6 on the diagonal, -1 per existing neighbour).
// One thread per grid point and column; x-neighbours are adjacent in memory so a warp's
// loads are coalesced; the 6 neighbour reads hit L1/L2.
__global__ void __launch_bounds__(256) k_laplacian7(int nx, int ny, int nz, int s, const double* __restrict__ V,
                                                    int64_t ldv, double* __restrict__ Y, int64_t ldy) {
  const int64_t npts = (int64_t)nx * ny * nz;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < npts * s; e += stride) {
    const int c = (int)(e / npts);
    const int64_t p = e - (int64_t)c * npts;
    const int i = (int)(p % nx);
    const int64_t jl = p / nx;
    const int j = (int)(jl % ny);
    const int l = (int)(jl / ny);
    const double* v = V + (int64_t)c * ldv;
    double acc = 6.0 * v[p];
    if (i > 0) acc -= v[p - 1];
    if (i + 1 < nx) acc -= v[p + 1];
    if (j > 0) acc -= v[p - nx];
    if (j + 1 < ny) acc -= v[p + nx];
    if (l > 0) acc -= v[p - (int64_t)nx * ny];
    if (l + 1 < nz) acc -= v[p + (int64_t)nx * ny];
    Y[p + (int64_t)c * ldy] = acc;
  }
}

}  // namespace pqr
