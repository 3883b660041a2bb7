// support_kernels.cuh — operators used by the PQR consumers (not the hot path).
#pragma once
#include "common.cuh"

namespace pqr {

// Y = A V, A = 7-point Dirichlet Laplacian (6 on the diagonal, -1 per existing neighbour), the
// operator of Block Arnoldi (configs[2]).  HBM-bound: each thread owns one
// (x, y) line of one column and marches along z over a chunk of planes with the three z values in
// registers (each point is read from HBM once); the x and y neighbours are loads of values the
// same or a neighbouring warp loads in the same plane (L1 hits).  Blocks of 32 x 8 threads (x
// along a warp: coalesced 256-byte rows); grid (x-tiles * y-tiles, z-chunks, columns).
constexpr int kLapTX = 32, kLapTY = 8;
__global__ void __launch_bounds__(kLapTX * kLapTY) k_laplacian7(int nx, int ny, int nz, int zchunk,
                                                                 const double* __restrict__ V, int64_t ldv,
                                                                 double* __restrict__ Y, int64_t ldy) {
  const int tilesx = (nx + kLapTX - 1) / kLapTX;
  const int i = (blockIdx.x % tilesx) * kLapTX + threadIdx.x;
  const int j = (blockIdx.x / tilesx) * kLapTY + threadIdx.y;
  const int c = blockIdx.z;
  const int l0 = blockIdx.y * zchunk, l1 = min(nz, l0 + zchunk);
  const bool in = i < nx && j < ny;
  const int64_t plane = (int64_t)nx * ny;
  const double* v = V + (int64_t)c * ldv + (int64_t)j * nx + i;
  double* y = Y + (int64_t)c * ldy + (int64_t)j * nx + i;
  double below = (in && l0 > 0) ? v[(int64_t)(l0 - 1) * plane] : 0.0;
  double cur = in && l0 < nz ? v[(int64_t)l0 * plane] : 0.0;
  for (int l = l0; l < l1; ++l) {
    const double* vp = v + (int64_t)l * plane;
    const double above = (in && l + 1 < nz) ? vp[plane] : 0.0;
    if (in) {
      double acc = 6.0 * cur - below - above;
      if (i > 0) acc -= vp[-1];
      if (i + 1 < nx) acc -= vp[1];
      if (j > 0) acc -= vp[-nx];
      if (j + 1 < ny) acc -= vp[nx];
      y[(int64_t)l * plane] = acc;
    }
    below = cur;
    cur = above;
  }
}

}  // namespace pqr
