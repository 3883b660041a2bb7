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
// Kernels (one CTA of 256 threads per block; the block's rows live in registers,
// RPT rows per thread, S columns):
//   k_tsqr_up    stage 1 (§8(a) a6/a7): X_b <- H_{C-1}...H_0 X_b (apply the C
//                committed reflectors, Alg. 6 line 1), then Householder QR of rows
//                C..R-1 with s new reflectors (Alg. 6 lines 2-9, never deflating:
//                reading R4), output [P_b; N_b] ((C+s) x s) into the parent's slot.
//   k_tsqr_down  stage 2 (§8(a) a7/a8): Y_b = H_0...H_{C+s-1} [coef_b; 0], the
//                assembly "U = [Q_i U_i][P~_i; N~_i]" of PAPER.md:L749-768.
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

// Rows of level block b: q + (b < rem) rows starting at b*q + min(b, rem).
struct TsqrLevel {
  int64_t q, rem;
  int nblocks;
  // up
  const double* X; int64_t ldx;   // stage-1 input, level row index
  double* V; int64_t ldv;         // reflectors, level row index, column j = reflector j
  double* out; int64_t ldo;       // stage-1 output: block b -> rows b*cap .. of out
  // down
  const double* cin; int64_t ldci;  // stage-2 input coefficients: block b -> rows b*cap .. of cin
  double* Y; int64_t ldy;           // stage-2 output, level row index
  int cap;
};

PQR_DEV int64_t blk_start(const TsqrLevel& L, int64_t b) { return b * L.q + (b < L.rem ? b : L.rem); }
PQR_DEV int64_t blk_rows(const TsqrLevel& L, int64_t b) { return L.q + (b < L.rem ? 1 : 0); }

// Warp "reduce-scatter" of S partial sums: afterwards lane l holds the warp total of
// column col_of_lane<S>(l) in v[0].
template <int S>
PQR_DEV void warp_reduce_scatter(double (&v)[S], int lane) {
  int cnt = S;
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) {
    if (cnt > 1) {
      const int half = cnt >> 1;
      const bool upper = (lane & m) != 0;
#pragma unroll
      for (int i = 0; i < S / 2; ++i) {
        if (i < half) {
          const double send = upper ? v[i] : v[i + half];
          const double keep = upper ? v[i + half] : v[i];
          v[i] = keep + __shfl_xor_sync(0xffffffffu, send, m);
        }
      }
      cnt = half;
    } else {
      v[0] += __shfl_xor_sync(0xffffffffu, v[0], m);
    }
  }
}
template <int S>
PQR_DEV int col_of_lane(int lane) {
  // bits consumed from the top: m = 16 (weight S/2), 8 (S/4), ...
  int c = 0, w = S >> 1;
  for (int m = 16; m >= 1 && w >= 1; m >>= 1, w >>= 1)
    if (lane & m) c += w;
  return c;
}
template <int S>
PQR_DEV bool lane_writes(int lane) {
  // one representative lane per column: the low (5 - log2 S) bits are zero
  int lowbits = 0, w = S;
  while (w > 1) { w >>= 1; ++lowbits; }
  const int mask = (1 << (5 - lowbits)) - 1;
  return (lane & mask) == 0;
}

// Block-wide sum of S per-thread partials -> tot[0..S-1] in shared memory (visible to
// all threads on return).  red: kTsqrWarps*S doubles.  Two barriers.
template <int S>
PQR_DEV void block_sum(double (&v)[S], double* red, double* tot) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  warp_reduce_scatter<S>(v, lane);
  if (lane_writes<S>(lane)) red[warp * S + col_of_lane<S>(lane)] = v[0];
  __syncthreads();
  if (threadIdx.x < S) {
    double a = 0.0;
#pragma unroll
    for (int w = 0; w < kTsqrWarps; ++w) a += red[w * S + threadIdx.x];
    tot[threadIdx.x] = a;
  }
  __syncthreads();
}

// ----------------------------------------------------------------------------
// stage 1: apply the committed reflectors, then s new Householder reflectors
// ----------------------------------------------------------------------------
template <int RPT, int S>
__global__ void __launch_bounds__(kTsqrThreads) k_tsqr_up(TsqrLevel L, int C, int s) {
  __shared__ double red[2][kTsqrWarps * S];
  __shared__ double tot[2][S];
  __shared__ double bc[4];
  const int64_t b = blockIdx.x;
  const int64_t r0 = blk_start(L, b);
  const int R = (int)blk_rows(L, b);
  const int tid = threadIdx.x;

  double x[RPT][S];
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    const int row = tid + i * kTsqrThreads;
#pragma unroll
    for (int c = 0; c < S; ++c)
      x[i][c] = (row < R && c < s) ? L.X[r0 + row + (int64_t)c * L.ldx] : 0.0;
  }

  // ---- apply H_{C-1} ... H_0 (H_0 first): x <- H_j x ----
  double vn[RPT];
  if (C > 0) {
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const int row = tid + i * kTsqrThreads;
      vn[i] = (row < R && row >= 0) ? L.V[r0 + row] : 0.0;
    }
  }
  for (int j = 0; j < C; ++j) {
    double v[RPT];
#pragma unroll
    for (int i = 0; i < RPT; ++i) v[i] = vn[i];
    if (j + 1 < C) {  // prefetch reflector j+1
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        const int row = tid + i * kTsqrThreads;
        vn[i] = (row < R && row >= j + 1) ? L.V[r0 + row + (int64_t)(j + 1) * L.ldv] : 0.0;
      }
    }
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const int row = tid + i * kTsqrThreads;
      if (row < j) v[i] = 0.0;
    }
    double w[S];
#pragma unroll
    for (int c = 0; c < S; ++c) {
      double a = 0.0;
#pragma unroll
      for (int i = 0; i < RPT; ++i) a += v[i] * x[i][c];
      w[c] = a;
    }
    block_sum<S>(w, red[j & 1], tot[j & 1]);
#pragma unroll
    for (int c = 0; c < S; ++c) {
      const double f = 2.0 * tot[j & 1][c];
#pragma unroll
      for (int i = 0; i < RPT; ++i) x[i][c] -= f * v[i];
    }
  }

  // ---- Householder QR of rows C..R-1 of the s new columns (Alg. 6 lines 2-9) ----
  double* outb = L.out + b * L.cap;  // rows b*cap .. of the parent's input
  for (int c = 0; c < s; ++c) {
    const int r = C + c;  // pivot row
    // lambda^2 = ||x[r:R, c]||^2 and u0 = x[r, c]
    double part[1] = {0.0};
    double u0 = 0.0;
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const int row = tid + i * kTsqrThreads;
#pragma unroll
      for (int cc = 0; cc < S; ++cc)
        if (cc == c && row >= r && row < R) {
          part[0] += x[i][cc] * x[i][cc];
          if (row == r) u0 = x[i][cc];
        }
    }
    if (tid == (r % kTsqrThreads) ) bc[2] = u0;
    block_sum<1>(part, red[0], tot[0]);
    const double lam = sqrt(tot[0][0]);
    u0 = bc[2];
    const double sigma = (u0 >= 0.0) ? -1.0 : 1.0;  // sigma = -sgn(u0), sgn(0) = +1
    const double diag = sigma * lam;
    // v = (u - sigma*lam*e_r) / ||.||, ||.||^2 = 2 lam (lam + |u0|); identity if lam == 0
    const double nv2 = 2.0 * lam * (lam + fabs(u0));
    const double inv = nv2 > 0.0 ? rsqrt(nv2) : 0.0;
    double v[RPT];
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const int row = tid + i * kTsqrThreads;
      double u = 0.0;
#pragma unroll
      for (int cc = 0; cc < S; ++cc)
        if (cc == c) u = x[i][cc];
      v[i] = (row >= r && row < R) ? (row == r ? (u - diag) * inv : u * inv) : 0.0;
      if (row >= r && row < R) L.V[r0 + row + (int64_t)r * L.ldv] = v[i];
    }
    // column c becomes [x(0:r, c); diag; 0]
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const int row = tid + i * kTsqrThreads;
#pragma unroll
      for (int cc = 0; cc < S; ++cc)
        if (cc == c && row >= r) x[i][cc] = (row == r) ? diag : 0.0;
    }
    // apply H_r to columns c+1..s-1
    if (c + 1 < s) {
      double w[S];
#pragma unroll
      for (int cc = 0; cc < S; ++cc) {
        double a = 0.0;
        if (cc > c) {
#pragma unroll
          for (int i = 0; i < RPT; ++i) a += v[i] * x[i][cc];
        }
        w[cc] = a;
      }
      block_sum<S>(w, red[1], tot[1]);
#pragma unroll
      for (int cc = 0; cc < S; ++cc) {
        if (cc > c) {
          const double f = 2.0 * tot[1][cc];
#pragma unroll
          for (int i = 0; i < RPT; ++i) x[i][cc] -= f * v[i];
        }
      }
    }
  }
  // ---- output [P_b; N_b] = rows 0..C+s-1 of the transformed block ----
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    const int row = tid + i * kTsqrThreads;
    if (row < C + s && row < R) {
#pragma unroll
      for (int c = 0; c < S; ++c)
        if (c < s) outb[row + (int64_t)c * L.ldo] = x[i][c];
    }
  }
}

// ----------------------------------------------------------------------------
// stage 2: Y_b = H_0 ... H_{C-1} [coef; 0]   (C = all reflectors incl. this call's)
// ----------------------------------------------------------------------------
template <int RPT, int S>
__global__ void __launch_bounds__(kTsqrThreads) k_tsqr_down(TsqrLevel L, int C, int t, int ncol) {
  __shared__ double red[2][kTsqrWarps * S];
  __shared__ double tot[2][S];
  const int64_t b = blockIdx.x;
  const int64_t r0 = blk_start(L, b);
  const int R = (int)blk_rows(L, b);
  const int tid = threadIdx.x;
  const double* cb = L.cin + b * L.cap;
  double y[RPT][S];
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    const int row = tid + i * kTsqrThreads;
#pragma unroll
    for (int c = 0; c < S; ++c) y[i][c] = (row < C && row < R && c < t) ? cb[row + (int64_t)c * L.ldci] : 0.0;
  }
  double vn[RPT];
  if (C > 0) {
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const int row = tid + i * kTsqrThreads;
      vn[i] = (row < R && row >= C - 1) ? L.V[r0 + row + (int64_t)(C - 1) * L.ldv] : 0.0;
    }
  }
  for (int j = C - 1; j >= 0; --j) {
    double v[RPT];
#pragma unroll
    for (int i = 0; i < RPT; ++i) v[i] = vn[i];
    if (j > 0) {
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        const int row = tid + i * kTsqrThreads;
        vn[i] = (row < R && row >= j - 1) ? L.V[r0 + row + (int64_t)(j - 1) * L.ldv] : 0.0;
      }
    }
    double w[S];
#pragma unroll
    for (int c = 0; c < S; ++c) {
      double a = 0.0;
#pragma unroll
      for (int i = 0; i < RPT; ++i) a += v[i] * y[i][c];
      w[c] = a;
    }
    block_sum<S>(w, red[j & 1], tot[j & 1]);
#pragma unroll
    for (int c = 0; c < S; ++c) {
      const double f = 2.0 * tot[j & 1][c];
#pragma unroll
      for (int i = 0; i < RPT; ++i) y[i][c] -= f * v[i];
    }
  }
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    const int row = tid + i * kTsqrThreads;
    if (row < R) {
#pragma unroll
      for (int c = 0; c < S; ++c)
        if (c < ncol) L.Y[r0 + row + (int64_t)c * L.ldy] = (c < t) ? y[i][c] : 0.0;
    }
  }
}

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
  __shared__ double sN[kSMaxTop * kSMaxTop];
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
    for (int e = tid; e < k * s; e += blockDim.x) {
      const int i = e % k, c = e / k;
      double acc = 0.0;
      for (int r = 0; r < C; ++r) acc += a.Rt[r + (int64_t)i * a.ldr] * sB[r + c * kTopMaxRows];
      sV[e] = acc;  // scratch
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

}  // namespace pqr
