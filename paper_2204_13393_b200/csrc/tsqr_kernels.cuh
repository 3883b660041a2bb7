// tsqr_kernels.cuh — TreeTSPQR (TSQR variant) kernels, §4.1 Alg. 9.
//
// The basis is kept in a multi-level locally orthogonal representation (LOR,
// PAPER.md:L609-659, applied recursively as L603-607 prescribes):
//   level 0  (leaves)  row blocks of the GPU's rows; block b stores Householder
//                      reflectors v_0..v_{C-1} (unit norm, H = I - 2 v v^T, Eq. (hh))
//                      in the rows of the block, v_j living on block rows j..R-1;
//   level L>0 (nodes)  a node stacks the top-C coordinates of its `arity` children
//                      (child i occupies node rows i*cap .. i*cap+cap-1) and stores
//                      reflectors on those stacked rows — the reduction subalgorithm
//                      (HH) applied to the stacked [R_i P_i; 0 N_i] of L696-720;
//   top                the GPU root's top-C coordinates, where the basis is the
//                      explicit C x k matrix R_top (PAPER.md's stacked "R" at the
//                      final level; orthonormal columns).
// Q = L0 L1 ... L_root [R_top; 0], every L orthogonal.
//
// Level kernels (stage 1 / stage 2 of every leaf and node block) are in tsqr_wy.cuh:
//   k_wy_up      stage 1 (§8(a) a6/a7): X_b <- Q_b^T X_b (apply the committed
//                reflector panels, Alg. 6 line 1), then Householder QR of rows C..R-1
//                with s new reflectors (Alg. 6 lines 2-9, never deflating: reading
//                R4), output [P_b; N_b] ((C+s) x s) into the parent's slot.
//   k_wy_down    stage 2 (§8(a) a7/a8): Y_b = Q_b [coef_b; 0], the assembly
//                "U = [Q_i U_i][P~_i; N~_i]" of PAPER.md:L749-768.
// This file holds the top level:
//   k_tsqr_top   the top-level PQR on the C-dim top coordinates: P = R_top^T B
//                (twice, i.e. BCGS+ projection against the explicit orthonormal
//                R_top), then Householder with in-order deflation (reading R3) of
//                the remainder: N, t and the coefficients U~ of U; sign
//                canonicalisation (reading R6).
#pragma once
#include "common.cuh"

namespace pqr {

constexpr int kTsqrThreads = 256;
constexpr int kTsqrWarps = kTsqrThreads / 32;

// ----------------------------------------------------------------------------
// top-level PQR on the C-dim top coordinates (single CTA)
// ----------------------------------------------------------------------------
struct TsqrTopArgs {
  const double* B; int ldb;      // (C+s) x s  top coefficients of X
  const double* Rt; int ldr;     // C x k explicit basis in top coordinates (rows C.. are zero)
  int C, k, s;
  double tau_rel;                // deflation: lambda_j <= tau_rel * ||B||_F
  int build;                     // 1: LOR build (record B as new R_top columns; no PQR)
  double* P; int ldp;            // k x s
  double* N; int ldn;            // s x s (rows >= t zero, positive pivots)
  double* Ut; int ldu;           // (C+s) x s coefficients of U (columns >= t zero)
  int* t_out; int* deflated;
};

constexpr int kTopMaxRows = 176;  // C + s <= cap <= 160, plus headroom
constexpr int kSMaxTop = 16;

__global__ void __launch_bounds__(256) k_tsqr_top(TsqrTopArgs a) {
  __shared__ double sB[kTopMaxRows * kSMaxTop];
  __shared__ double sV[kTopMaxRows * kSMaxTop];  // reflectors of the top HH
  __shared__ double sdiag[kSMaxTop];
  __shared__ int spiv[kSMaxTop];
  __shared__ int sT;
  __shared__ double snorm;
  const int tid = threadIdx.x;
  const int C = a.C, k = a.k, s = a.s, m = C + s;
  for (int e = tid; e < m * s; e += blockDim.x) {
    const int i = e % m, c = e / m;
    sB[i + c * kTopMaxRows] = a.B[i + (int64_t)c * a.ldb];
  }
  __syncthreads();
  if (a.build) {
    // LOR build: the coefficients themselves are the new basis columns (Q = L [B; 0]).
    for (int e = tid; e < m * s; e += blockDim.x) {
      const int i = e % m, c = e / m;
      a.Ut[i + (int64_t)c * a.ldu] = sB[i + c * kTopMaxRows];
    }
    if (tid == 0) { *a.t_out = s; if (a.deflated) *a.deflated = 0; }
    return;
  }
  if (tid == 0) {
    double acc = 0.0;
    for (int c = 0; c < s; ++c)
      for (int i = 0; i < m; ++i) acc += sB[i + c * kTopMaxRows] * sB[i + c * kTopMaxRows];
    snorm = sqrt(acc);
  }
  for (int e = tid; e < k * s; e += blockDim.x) a.P[(e % k) + (int64_t)(e / k) * a.ldp] = 0.0;
  __syncthreads();
  // ---- P = R_top^T B, B -= R_top P  (twice: BCGS+ against the orthonormal R_top) ----
  for (int pass = 0; pass < 2 && k > 0; ++pass) {
    {  // P_pass = R_top^T B: one warp per column i of R_top, lanes over its rows (coalesced)
      const int warp = tid >> 5, lane = tid & 31, nw = blockDim.x >> 5;
      for (int i = warp; i < k; i += nw) {
        double acc[kSMaxTop];
#pragma unroll
        for (int c = 0; c < kSMaxTop; ++c) acc[c] = 0.0;
        for (int r = lane; r < C; r += 32) {
          const double rv = a.Rt[r + (int64_t)i * a.ldr];
#pragma unroll
          for (int c = 0; c < kSMaxTop; ++c)
            if (c < s) acc[c] = fma(rv, sB[r + c * kTopMaxRows], acc[c]);
        }
#pragma unroll
        for (int c = 0; c < kSMaxTop; ++c) {
          if (c < s) {
            double v = acc[c];
#pragma unroll
            for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == 0) sV[i + c * k] = v;  // scratch
          }
        }
      }
    }
    __syncthreads();
    for (int e = tid; e < C * s; e += blockDim.x) {
      const int r = e % C, c = e / C;
      double acc = 0.0;
      for (int i = 0; i < k; ++i) acc += a.Rt[r + (int64_t)i * a.ldr] * sV[i + c * k];
      sB[r + c * kTopMaxRows] -= acc;
    }
    for (int e = tid; e < k * s; e += blockDim.x) a.P[(e % k) + (int64_t)(e / k) * a.ldp] += sV[e];
    __syncthreads();
  }
  // ---- Householder QR with in-order deflation of B (m x s) (Alg. 6; reading R3) ----
  if (tid < 32) {
    const int lane = tid;
    const double thr = a.tau_rel * snorm;
    int r = 0;
    for (int c = 0; c < s; ++c) {
      double part = 0.0;
      for (int i = r + lane; i < m; i += 32) part += sB[i + c * kTopMaxRows] * sB[i + c * kTopMaxRows];
      for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
      const double lam = sqrt(part);
      if (!(lam > thr)) continue;  // deflated: no reflector, column keeps rows 0..r-1
      const double u0 = sB[r + c * kTopMaxRows];
      const double sigma = (u0 >= 0.0) ? -1.0 : 1.0;
      const double diag = sigma * lam;
      const double inv = rsqrt(2.0 * lam * (lam + fabs(u0)));
      for (int i = lane; i < m; i += 32) {
        const double u = sB[i + c * kTopMaxRows];
        sV[i + r * kTopMaxRows] = i < r ? 0.0 : (i == r ? (u - diag) * inv : u * inv);
      }
      __syncwarp();
      for (int i = r + lane; i < m; i += 32) sB[i + c * kTopMaxRows] = (i == r) ? diag : 0.0;
      if (lane == 0) { spiv[r] = c; sdiag[r] = diag; }
      __syncwarp();
      for (int cc = c + 1; cc < s; ++cc) {
        double d = 0.0;
        for (int i = r + lane; i < m; i += 32) d += sV[i + r * kTopMaxRows] * sB[i + cc * kTopMaxRows];
        for (int o = 16; o; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
        for (int i = r + lane; i < m; i += 32) sB[i + cc * kTopMaxRows] -= 2.0 * d * sV[i + r * kTopMaxRows];
        __syncwarp();
      }
      ++r;
    }
    if (lane == 0) sT = r;
  }
  __syncthreads();
  const int t = sT;
  // ---- outputs: N (sign-canonicalised rows), P, U~ = H_0..H_{t-1} [I_t; 0] ----
  for (int e = tid; e < a.s * a.s; e += blockDim.x) {
    const int i = e % a.s, c = e / a.s;
    double v = 0.0;
    if (i < t) {
      const double sg = sdiag[i] < 0.0 ? -1.0 : 1.0;
      if (c >= spiv[i]) v = sg * sB[i + c * kTopMaxRows];
    }
    a.N[i + (int64_t)c * a.ldn] = v;
  }
  __syncthreads();
  // U~ column c (< t): y = e_c, apply H_c ... H_0 (reverse order), times sign
  for (int c = tid >> 5; c < s; c += blockDim.x >> 5) {
    const int lane = tid & 31;
    double* y = sB + c * kTopMaxRows;  // reuse sB column c as the work vector
    for (int i = lane; i < m; i += 32) y[i] = (i == c && c < t) ? 1.0 : 0.0;
    __syncwarp();
    if (c < t) {
      for (int j = c; j >= 0; --j) {
        double d = 0.0;
        for (int i = j + lane; i < m; i += 32) d += sV[i + j * kTopMaxRows] * y[i];
        for (int o = 16; o; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
        for (int i = j + lane; i < m; i += 32) y[i] -= 2.0 * d * sV[i + j * kTopMaxRows];
        __syncwarp();
      }
    }
    const double sg = (c < t && sdiag[c] < 0.0) ? -1.0 : 1.0;
    for (int i = lane; i < m; i += 32) a.Ut[i + (int64_t)c * a.ldu] = (c < t) ? sg * y[i] : 0.0;
  }
  if (tid == 0) {
    *a.t_out = t;
    if (a.deflated) *a.deflated = s - t;
  }
}

// Cross-GPU level input (a7, §8(e)): the all-gathered GPU-root blocks, rank-major and compact
// (block g = rows x s with ld rows at src + g*rows*s), into the first cross level's stacked
// input: block g at rows g*cap of dst (ld ldd); rows rows..cap-1 of each child slot are
// zeroed (an earlier call with a wider block may have left data there).
__global__ void __launch_bounds__(256) k_unpack_roots(const double* __restrict__ src, int rows, int s, int P,
                                                      double* __restrict__ dst, int64_t ldd, int cap) {
  const int per = cap * s;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < P * per; e += gridDim.x * blockDim.x) {
    const int g = e / per, r = e - g * per, c = r / cap, i = r - c * cap;
    dst[(int64_t)g * cap + i + (int64_t)c * ldd] = i < rows ? src[(int64_t)g * rows * s + c * rows + i] : 0.0;
  }
}

}  // namespace pqr
