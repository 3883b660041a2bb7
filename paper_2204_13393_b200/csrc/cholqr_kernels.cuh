// cholqr_kernels.cuh — the BCGS-PIP / BCGS-PIP+ (CholQR2 variant) hot-path kernels.
//
//  k_gram    (§8(a) a1): W = [Q X]^T X, "P = Q^T X and G = X^T X at once"
//                        (Alg. 7 line 1; L521, Alg. 8 line 1).
//  k_factor  (§8(a) a3, a5): S = G - P^T P, N^T N = S by in-order Cholesky with
//                        deflation (R3b),
//                        M = [-P N^{-1}; N^{-1}] and, for the second pass, the
//                        recombination P = P1 + P2 N1, N = N2 N1 (R1).
//  k_update  (§8(a) a4): U = X N^{-1} - Q P N^{-1} = [Q X] M
//                        ("U = XN^{-1} - QPN^{-1}", Alg. 8 lines 3, 6).
//
// Layout: all big operands column-major (ld >= n).  One warp streams slabs of
// rows; both tall operands are read exactly once per pass, with 16-byte
// loads whose 8 (gram) / 4 (update) column segments per instruction are each
// fully-used 32-byte sectors.
#pragma once
#include "common.cuh"

namespace pqr {

// ----------------------------------------------------------------------------
// a1: fused tall-skinny Gram  W = [Q X]^T X
// ----------------------------------------------------------------------------
struct GramArgs {
  const double* Q; int64_t ldq;   // n x k
  const double* X; int64_t ldx;   // n x s (B operand and A columns k..k+s-1)
  int64_t n; int k; int s;        // s: static block width (columns >= s never read)
  int G;                          // column-tile groups per CTA: 1, 2, 4 or 8
  int64_t rows_per_cta;           // multiple of 8
  double* partials;               // [gridDim.x][m*s], element (j,c) at j + c*m
  double* W; int ldw;             // reduced result, element (j,c) at j + c*ldw
  unsigned int* ticket;           // zero-initialised; reset to 0 by the last CTA
};

template <bool VEC>
PQR_DEV double2 ld_pair(const double* p) {
  if constexpr (VEC) return ld2(p);
  else return make_double2(__ldg(p), __ldg(p + 1));
}

// MTW = column tiles (of 8) per warp, NT = column tiles of X (s <= 8*NT).
// Warp w: column group g = w % G (tiles g*MTW .. g*MTW+MTW-1), row lane rw = w / G
// (slabs of 8 rows, every (8/G)-th slab of the CTA's row range).
// Lane l holds rows r0 + 2(l&3) + {0,1} of column 8*tile + (l>>2): the two rows are
// the k-index of two consecutive m8n8k4 steps (any row->k bijection is valid since
// the contraction runs over rows).
template <int MTW, int NT, bool VEC>
__global__ void __launch_bounds__(256) k_gram(GramArgs a) {
  extern __shared__ double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = a.G, RW = 8 / G;
  const int g = warp % G, rw = warp / G;
  const int m = a.k + a.s;
  const int gq = lane >> 2, q = lane & 3;

  const double* acol[MTW];
#pragma unroll
  for (int i = 0; i < MTW; ++i) acol[i] = col_ptr(a.Q, a.ldq, a.X, a.ldx, a.k, m, 8 * (g * MTW + i) + gq);
  const double* bcol[NT];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const int c = 8 * nt + gq;
    bcol[nt] = c < a.s ? a.X + (int64_t)c * a.ldx : nullptr;
  }

  double acc[MTW][NT][2];
#pragma unroll
  for (int i = 0; i < MTW; ++i)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) acc[i][nt][0] = acc[i][nt][1] = 0.0;

  const int64_t rb = (int64_t)blockIdx.x * a.rows_per_cta;
  const int64_t re = min(a.n, rb + a.rows_per_cta);
  const int ro = 2 * q;
  int64_t r0 = rb + 8 * rw;
#pragma unroll 2
  for (; r0 + 8 <= re; r0 += 8 * RW) {
    double2 av[MTW], bv[NT];
#pragma unroll
    for (int i = 0; i < MTW; ++i) av[i] = acol[i] ? ld_pair<VEC>(acol[i] + r0 + ro) : make_double2(0.0, 0.0);
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) bv[nt] = bcol[nt] ? ld_pair<VEC>(bcol[nt] + r0 + ro) : make_double2(0.0, 0.0);
#pragma unroll
    for (int i = 0; i < MTW; ++i)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        dmma884(acc[i][nt][0], acc[i][nt][1], av[i].x, bv[nt].x);
        dmma884(acc[i][nt][0], acc[i][nt][1], av[i].y, bv[nt].y);
      }
  }
  if (r0 < re) {  // ragged last slab of the last CTA
    double2 av[MTW], bv[NT];
#pragma unroll
    for (int i = 0; i < MTW; ++i) av[i] = ld2_guard(acol[i], r0 + ro, re);
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) bv[nt] = ld2_guard(bcol[nt], r0 + ro, re);
#pragma unroll
    for (int i = 0; i < MTW; ++i)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        dmma884(acc[i][nt][0], acc[i][nt][1], av[i].x, bv[nt].x);
        dmma884(acc[i][nt][0], acc[i][nt][1], av[i].y, bv[nt].y);
      }
  }

  // ---- CTA reduction over the RW row lanes (fixed order) ----
  constexpr int FR = MTW * NT * 64;  // doubles per warp
  double* mine = smem + warp * FR;
#pragma unroll
  for (int i = 0; i < MTW; ++i)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      mine[((i * NT + nt) * 32 + lane) * 2 + 0] = acc[i][nt][0];
      mine[((i * NT + nt) * 32 + lane) * 2 + 1] = acc[i][nt][1];
    }
  __syncthreads();
  double* part = a.partials + (size_t)blockIdx.x * m * a.s;
  for (int e = threadIdx.x; e < G * FR; e += blockDim.x) {
    const int v = e & 1, l = (e >> 1) & 31, rest = e >> 6;  // rest = (gg*MTW + i)*NT + nt
    const int nt = rest % NT, gi = rest / NT;
    const int i = gi % MTW, gg = gi / MTW;
    const int j = 8 * (gg * MTW + i) + (l >> 2), c = 8 * nt + 2 * (l & 3) + v;
    if (j < m && c < a.s) {
      double sum = 0.0;
      for (int r = 0; r < RW; ++r) sum += smem[(r * G + gg) * FR + ((i * NT + nt) * 32 + l) * 2 + v];
      part[j + (int64_t)c * m] = sum;
    }
  }

  // ---- grid reduction by the last CTA to finish (fixed order over CTAs) ----
  __threadfence();
  __syncthreads();
  __shared__ unsigned int s_last;
  if (threadIdx.x == 0) s_last = (atomicAdd(a.ticket, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int ms = m * a.s;
  const int nb = gridDim.x;
  grid_sum_partials(a.partials, nb, ms, m, a.W, a.ldw);
  if (threadIdx.x == 0) *a.ticket = 0u;
}

// ----------------------------------------------------------------------------
// a3 / a5: small factorisation (single CTA)
// ----------------------------------------------------------------------------
constexpr int kSMax = 16;
constexpr int kMMax = 160;  // k + s upper bound supported by the small-factor kernel

struct FactorArgs {
  const double* W; int64_t w_stride; int nparts; int ldw;  // sum_r W_r, W_r at W + r*w_stride
  int k; int s;                 // s: static width of this pass's block
  const int* s_dev;             // actual width (pass 2: t1); nullptr -> s
  double tol2;                  // deflation: d_j <= max(tol2 * trace(G), eta * G_jj)
  double eta;
  double* P; int ldp;           // k x s   (this pass's P)
  double* N; int ldn;           // s x s   (this pass's N, rows >= t zero)
  double* M; int ldm;           // (k+s) x s, M = [-P_J N_J^{-1}; E_J N_J^{-1}], cols >= t zero
  int* t_out; int* piv_out; int* deflated;  // t, pivot columns, #deflated columns
  // recombination for the second pass (nullptr in the first pass)
  const double* P1; int ldp1; const double* N1; int ldn1; const int* t1_dev; int s0;
  double* Pf; int ldpf; double* Nf; int ldnf; int* tf;
};

// The whole factorisation by one CTA (any blockDim; callers use 256).  Output pointers may be
// global or shared memory (generic addressing): the small-n persistent kernel runs it in every
// CTA on the same summed Gram, writing to per-CTA shared buffers (identical results).
#ifdef PQR_SMALL_TRACE
__device__ unsigned long long g_factor_trace[8];
#define FB_TR(i)                                                                          \
  if (blockIdx.x == 0 && threadIdx.x == 0) {                                                \
    unsigned long long t_;                                                                \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                \
    g_factor_trace[i] = t_;                                                               \
  }
#else
#define FB_TR(i)
#endif
__device__ __forceinline__ void factor_body(const FactorArgs& a) {
  FB_TR(0);
  __shared__ double sW[kMMax * kSMax];
  __shared__ double sS[kSMax * kSMax];
  __shared__ double sN[kSMax * kSMax];
  __shared__ double sNi[kSMax * kSMax];
  __shared__ int sPiv[kSMax];
  __shared__ int sT;
  __shared__ double sInv[kSMax];  // 1 / N(r, pivot r)
  const int tid = threadIdx.x;
  const int k = a.k;
  const int s = a.s_dev ? min(*a.s_dev, a.s) : a.s;
  const int m = k + s;

  // 1. sum the per-part Gram matrices (ranks, host-buffer chunks, or CTAs) in a fixed order:
  //    part r goes to accumulator r % 4, combined as (a0 + a1) + (a2 + a3); 48 independent
  //    L2 loads in flight per step, the last step guarded (the sum is latency-bound: one step
  //    covers a small-n call's CTA partials)
  for (int e = tid; e < m * s; e += blockDim.x) {
    const int j = e % m, c = e / m;
    const double* w = a.W + j + (int64_t)c * a.ldw;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int r = 0; r < a.nparts; r += 48) {
      double v[48];
#pragma unroll
      for (int u = 0; u < 48; ++u) v[u] = r + u < a.nparts ? __ldcg(w + (size_t)(r + u) * a.w_stride) : 0.0;
#pragma unroll
      for (int u = 0; u < 48; ++u) acc[u & 3] += v[u];
    }
    sW[j + c * m] = (acc[0] + acc[1]) + (acc[2] + acc[3]);
  }
  __syncthreads();
  FB_TR(1);
  // 2. S = G - P^T P: TP threads per entry (a power of two, the entries spread over the CTA),
  //    each a strided partial dot product over the k rows of P, then a fixed xor tree
  {
    const int ss = s * s;
    int TP = 1;
    while (TP < 32 && TP * 2 * ss <= (int)blockDim.x) TP *= 2;
    for (int base = 0; base < ss * TP; base += blockDim.x) {
      const int e = (base + tid) / TP, part = (base + tid) % TP;
      double p0 = 0.0, p1 = 0.0;
      if (e < ss) {
        const int x = e % s, y = e / s;
        const double* px = sW + x * m;
        const double* py = sW + y * m;
        int i = part;
        for (; i + TP < k; i += 2 * TP) {
          p0 = fma(px[i], py[i], p0);
          p1 = fma(px[i + TP], py[i + TP], p1);
        }
        if (i < k) p0 = fma(px[i], py[i], p0);
      }
      double p = p0 + p1;
      for (int mb = 1; mb < TP; mb <<= 1) p += __shfl_xor_sync(0xffffffffu, p, mb);
      if (e < ss && part == 0) {
        const int x = e % s, y = e / s;
        sS[x + y * kSMax] = sW[k + x + y * m] - p;
      }
    }
  }
  for (int e = tid; e < kSMax * kSMax; e += blockDim.x) { sN[e] = 0.0; sNi[e] = 0.0; }
  __syncthreads();
  FB_TR(2);
  // 3. in-order right-looking Cholesky with deflation (warp 0).  Lane x owns row x of the
  //    trailing S (it alone updates it; S is symmetric, so the pivot row's entry S(j, x) is read
  //    as S(x, j) from the lane's own row): one warp synchronisation per column.
  if (tid < 32) {
    const int lane = tid;
    double trace = 0.0;
    for (int c = 0; c < s; ++c) trace += sW[k + c + c * m];
    const double thr_abs = a.tol2 * trace;
    double* Srow = sS + lane;  // row `lane`: Srow[y * kSMax] = S(lane, y)
    int r = 0;
    for (int j = 0; j < s; ++j) {
      const double d = sS[j + j * kSMax];
      const double gjj = sW[k + j + j * m];
      const double thr = fmax(thr_abs, a.eta * gjj);
      if (!(d > thr)) continue;  // deflated column (also catches NaN); uniform across lanes
      // pivot sqrt(d) and its inverse from one reciprocal square root (no fp64 division on
      // the latency-bound critical path)
      const double inv = rsqrt(d);
      const double nx = (lane > j && lane < s) ? Srow[j * kSMax] * inv : 0.0;  // N(r, lane)
      if (lane == 0) { sN[r + j * kSMax] = d * inv; sPiv[r] = j; sInv[r] = inv; }
      if (lane > j && lane < s) sN[r + lane * kSMax] = nx;
      __syncwarp();
      if (lane > j && lane < s)
        for (int y = j + 1; y < s; ++y) Srow[y * kSMax] = fma(-nx, sN[r + y * kSMax], Srow[y * kSMax]);
      __syncwarp();
      ++r;
    }
    if (lane == 0) sT = r;
    __syncwarp();
    // 4. N_J^{-1} (t x t upper triangular), lane c computes column c
    const int t = r;
    if (lane < t) {
      const int c = lane;
      sNi[c + c * kSMax] = sInv[c];
      for (int i = c - 1; i >= 0; --i) {
        double acc = 0.0;
        for (int q = i + 1; q <= c; ++q) acc += sN[i + sPiv[q] * kSMax] * sNi[q + c * kSMax];
        sNi[i + c * kSMax] = -acc * sInv[i];
      }
    }
  }
  __syncthreads();
  FB_TR(3);
  const int t = sT;
  // 5. outputs of this pass: P, N, M, t, pivots
  for (int e = tid; e < k * a.s; e += blockDim.x) {
    const int i = e % k, c = e / k;
    a.P[i + (int64_t)c * a.ldp] = c < s ? sW[i + c * m] : 0.0;
  }
  for (int e = tid; e < a.s * a.s; e += blockDim.x) {
    const int i = e % a.s, c = e / a.s;
    a.N[i + c * a.ldn] = (i < s && c < s) ? sN[i + c * kSMax] : 0.0;
  }
  const int mfull = k + a.s;
  for (int e = tid; e < mfull * a.s; e += blockDim.x) {
    const int i = e % mfull, c = e / mfull;
    double v = 0.0;
    if (c < t) {
      if (i < k) {
        for (int q = 0; q < t; ++q) v -= sW[i + sPiv[q] * m] * sNi[q + c * kSMax];
      } else {
        const int col = i - k;
        for (int q = 0; q < t; ++q)
          if (sPiv[q] == col) v = sNi[q + c * kSMax];
      }
    }
    a.M[i + (int64_t)c * a.ldm] = v;
  }
  if (tid == 0) {
    *a.t_out = t;
    if (a.deflated) *a.deflated = s - t;
  }
  if (tid < kSMax && a.piv_out) a.piv_out[tid] = tid < t ? sPiv[tid] : -1;
  FB_TR(4);
  // 6. recombination (second pass): P = P1 + P2 N1,  N = N2 N1
  if (a.P1) {
    const int t1 = s;  // this pass normalised the t1 columns of U1
    for (int e = tid; e < k * a.s0; e += blockDim.x) {
      const int i = e % k, c = e / k;
      double v = a.P1[i + (int64_t)c * a.ldp1];
      for (int q = 0; q < t1; ++q) v += sW[i + q * m] * a.N1[q + c * a.ldn1];
      a.Pf[i + (int64_t)c * a.ldpf] = v;
    }
    for (int e = tid; e < a.s0 * a.s0; e += blockDim.x) {
      const int i = e % a.s0, c = e / a.s0;
      double v = 0.0;
      if (i < t)
        for (int q = 0; q < t1; ++q) v += sN[i + q * kSMax] * a.N1[q + c * a.ldn1];
      a.Nf[i + c * a.ldnf] = v;
    }
    if (tid == 0) *a.tf = t;
  }
}

__global__ void __launch_bounds__(256) k_factor(FactorArgs a) { factor_body(a); }

// ----------------------------------------------------------------------------
// a4: fused update  U = [Q X] M   (M is m x s, columns >= t zero)
// ----------------------------------------------------------------------------
struct UpdateArgs {
  const double* Q; int64_t ldq;   // n x k
  const double* X; int64_t ldx;   // n x sx
  int64_t n; int k; int sx;       // A = [Q X] has m = k + sx columns
  int sout;                       // output columns (<= 8*NT)
  const double* M; int ldm;       // m x sout
  const int* t_dev;               // valid output columns (nullptr -> sout); columns >= t get 0
  double* U; int64_t ldu;         // n x sout output
  double* U2; int64_t ldu2;       // optional second destination (basis append), columns < t only
};

// U^T = M^T [Q X]^T as m8n8k4 MMAs: M-index = output column c, N-index = row, K = column j
// of [Q X].  Lane l loads rows r0 + 2(l>>2) + {0,1} of column 4*kk + (l&3): the even row
// feeds one MMA, the odd row another, so one 16-byte load serves two MMAs and the D
// fragments give each lane 4 consecutive rows of one output column.
template <int NT, bool VEC>
__global__ void __launch_bounds__(256) k_update(UpdateArgs a) {
  extern __shared__ double sM[];  // [NT][mpad][8]
  const int m = a.k + a.sx;
  const int KS = (m + 3) >> 2, mpad = KS * 4;
  for (int e = threadIdx.x; e < NT * mpad * 8; e += blockDim.x) {
    const int nt = e / (mpad * 8), rem = e % (mpad * 8);
    const int j = rem >> 3, c = 8 * nt + (rem & 7);
    sM[e] = (j < m && c < a.sout) ? a.M[j + (int64_t)c * a.ldm] : 0.0;
  }
  __syncthreads();
  const int t = a.t_dev ? *a.t_dev : a.sout;
  const int lane = threadIdx.x & 31, gq = lane >> 2, q = lane & 3;
  const int64_t nslab = (a.n + 15) >> 4;
  const int64_t wstride = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t sl = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); sl < nslab; sl += wstride) {
    const int64_t r0 = sl << 4;
    const bool full = r0 + 16 <= a.n;
    double d[NT][2][2];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) d[nt][0][0] = d[nt][0][1] = d[nt][1][0] = d[nt][1][1] = 0.0;
    const int64_t rr = r0 + 2 * gq;
#pragma unroll 8
    for (int kk = 0; kk < KS; ++kk) {
      const double* cp = col_ptr(a.Q, a.ldq, a.X, a.ldx, a.k, m, 4 * kk + q);
      double2 av;
      if (full) av = cp ? ld_pair<VEC>(cp + rr) : make_double2(0.0, 0.0);
      else av = ld2_guard(cp, rr, a.n);
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const double mv = sM[(nt * mpad + 4 * kk + q) * 8 + gq];
        dmma884(d[nt][0][0], d[nt][0][1], mv, av.x);
        dmma884(d[nt][1][0], d[nt][1][1], mv, av.y);
      }
    }
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const int c = 8 * nt + gq;
      if (c >= a.sout) continue;
      const bool valid = c < t;
      const double v0 = valid ? d[nt][0][0] : 0.0, v1 = valid ? d[nt][1][0] : 0.0;
      const double v2 = valid ? d[nt][0][1] : 0.0, v3 = valid ? d[nt][1][1] : 0.0;
      const int64_t row = r0 + 4 * q;
      double* up = a.U + (int64_t)c * a.ldu + row;
      if (full && VEC) {
        st2(up, v0, v1);
        st2(up + 2, v2, v3);
      } else {
        if (row + 0 < a.n) up[0] = v0;
        if (row + 1 < a.n) up[1] = v1;
        if (row + 2 < a.n) up[2] = v2;
        if (row + 3 < a.n) up[3] = v3;
      }
      if (a.U2 && valid) {
        double* u2 = a.U2 + (int64_t)c * a.ldu2 + row;
        if (row + 0 < a.n) u2[0] = v0;
        if (row + 1 < a.n) u2[1] = v1;
        if (row + 2 < a.n) u2[2] = v2;
        if (row + 3 < a.n) u2[3] = v3;
      }
    }
  }
}

}  // namespace pqr
