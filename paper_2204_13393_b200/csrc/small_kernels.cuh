// small_kernels.cuh — one-launch CholQR2 (BCGS-PIP+, Alg. 8) for small n
// (latency-bound calls such as configs[0], n = 10,000: PAPER.md:L1488-1511 observes that the
// strong-scaling limit is set by such small per-process row counts).
//
// A cooperative launch of G CTAs (all co-resident); CTA b keeps its rows of [Q X] and of U1
// in shared memory for the whole call, so Q and X are read once and U written once:
//   1. W1_b = [Q X]_b^T X_b            -> partial b in global memory;  grid barrier
//   2. every CTA sums the G partials in CTA order and factors them (factor_body, identical in
//      every CTA: no broadcast needed) -> P1, N1, M1 in its shared memory
//   3. U1_b = [Q X]_b M1 (shared), W2_b = [Q U1]_b^T U1_b -> partial b; grid barrier
//   4. every CTA: factor of W2 with the recombination P = P1 + P2 N1, N = N2 N1 (reading R1)
//   5. U_b = [Q U1]_b M2 -> global U (and the basis' spare columns when appending);
//      CTA 0 writes P, N, t and the pivots (also straight into the caller's P and N and into
//      mapped pinned host memory for t, so a call is this one launch and a stream sync).
// The Gram passes give each warp whole entries (lanes over rows, fixed xor tree) and the products
// with M one thread per row.  The grid barrier is a counter in global memory (0 at launch; the
// last CTA to finish resets it, so no memset precedes the launch);
// the cooperative launch guarantees that the CTAs that wait on one another are resident.
// Sums run in a fixed order, so results are bitwise reproducible (R7).
#pragma once
#include "cholqr_kernels.cuh"
#include "common.cuh"

namespace pqr {

constexpr int kSmallThreads = 256;

struct SmallArgs {
  const double* Q; int64_t ldq;
  const double* X; int64_t ldx;
  int64_t n; int k; int s; int R;    // R = rows per CTA, even (the last CTA may have fewer)
  int vec;                           // Q, X 16-byte aligned with even ld: row-pair copies
  int single;                        // PQR_SINGLE_PASS: Alg. 7 only
  double tol2, eta;                  // deflation of pass 1 (R3b)
  double* U; int64_t ldu;            // n x s output (columns >= t zero)
  double* U2; int64_t ldu2;          // optional copy of the valid columns (basis append)
  double* part1; double* part2;      // [G][m*s] partial Grams
  unsigned int* bar;                 // grid barrier counter: 0 at launch, reset to 0 by the kernel
  // outputs (global): final P (k x s, ld ldp), N (16 x 16 layout, ld kSMax), ints as the handle's
  double* Pf; int ldp; double* Nf; int* ints;
  int* hints;                        // optional: ints[0..7] also written here (mapped pinned host memory)
  double* Pout; int ldpo;            // optional: the caller's P (k x s) and N (s x s), written directly
  double* Nout; int ldno;
};

PQR_DEV void grid_barrier(unsigned int* bar, unsigned int target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
    while (*reinterpret_cast<volatile unsigned int*>(bar) < target) {
    }
    __threadfence();
  }
  __syncthreads();
}

// shared memory: A = [Q X] rows (m x R), U1 (s x R), M (m x s), P1, P2, Pf (k x s),
// N1, N2, Nf (16 x 16), 64 ints
inline size_t small_smem(int R, int k, int s) {
  const int m = k + s, kp = k > 0 ? k : 1;
  return ((size_t)(m + s) * R + (size_t)m * s + 3 * (size_t)kp * s + 3 * kSMax * kSMax) * sizeof(double) +
         (size_t)64 * sizeof(int);
}

#ifdef PQR_SMALL_TRACE
__device__ unsigned long long g_small_trace[16];
#define SM_TR(i)                                                                          \
  if (blockIdx.x == 0 && threadIdx.x == 0) {                                                \
    unsigned long long t_;                                                                \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                \
    g_small_trace[i] = t_;                                                                \
  }
#else
#define SM_TR(i)
#endif

// W_b = A^T B over this CTA's R shared-memory rows for the m*S entries (j, c): column j of A =
// colA(j), column c of B = colB(c), S = s columns (compile time).  Warp w takes the column blocks
// j = 4w', ..., 4w' + 3 (w' = w, w + 8, ...) against all S columns of B: lane l sums rows l,
// l + 32, ... (consecutive lanes read consecutive rows: conflict free; 4 + S loads per 4 S
// FMAs), then the 4 S sums are reduce-scattered over the lanes by a fixed xor tree (bitwise
// reproducible, R7).
template <int S, class FA, class FB>
PQR_DEV void small_gram_t(FA colA, FB colB, int m, int s, int R, double* out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int NW = kSmallThreads / 32, JB = S >= 16 ? 2 : 4, V = JB * S;  // values per warp job
  constexpr int VP = V < 32 ? 32 : V;                          // padded to a power of two >= 32
  static_assert((V & (V - 1)) == 0 || V < 32, "JB * S: power of two or < 32");
  const double* xb[S];
#pragma unroll
  for (int c = 0; c < S; ++c) xb[c] = colB(c);
  for (int j0 = JB * warp; j0 < m; j0 += JB * NW) {
    double acc[VP];
#pragma unroll
    for (int i = 0; i < VP; ++i) acc[i] = 0.0;
    const double* xa[JB];
#pragma unroll
    for (int jj = 0; jj < JB; ++jj) xa[jj] = colA(min(j0 + jj, m - 1));
    for (int r = lane; r < R; r += 32) {
      double bv[S];
#pragma unroll
      for (int c = 0; c < S; ++c) bv[c] = xb[c][r];
#pragma unroll
      for (int jj = 0; jj < JB; ++jj) {
        const double av = xa[jj][r];
#pragma unroll
        for (int c = 0; c < S; ++c) acc[jj * S + c] = fma(av, bv[c], acc[jj * S + c]);
      }
    }
    // reduce-scatter of VP values over 32 lanes: after the halving steps lane l holds value
    // (l >> log2(32 / min(VP, 32)))... i.e. each value ends in 32 / VP' lanes, summed by xor
#pragma unroll
    for (int mb = 16, w = VP; w > 1 && mb >= 1; mb >>= 1, w >>= 1) {
      const bool up = (lane & mb) != 0;
#pragma unroll
      for (int i = 0; i < w / 2; ++i) {
        const double send = up ? acc[i] : acc[i + w / 2];
        const double keep = up ? acc[i + w / 2] : acc[i];
        acc[i] = keep + __shfl_xor_sync(0xffffffffu, send, mb);
      }
    }
    // VP >= 32: after 5 steps lane l holds the sum of value index v(l) = bit-reversed walk;
    // for VP = 32 (one value per lane) and VP = 64 (two: acc[0], acc[1]) the index is
    // v = sum over steps of (bit of lane) * (half width)
    constexpr int PER = VP / 32;  // values per lane after the scatter
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      int v = u;
#pragma unroll
      for (int st = 0, mb = 16, w = VP; st < 5; ++st, mb >>= 1, w >>= 1)
        if (lane & mb) v += w / 2;
      if (v < V) {
        const int jj = v / S, c = v % S, j = j0 + jj;
        if (j < m && c < s) out[j + c * m] = acc[u];
      }
    }
  }
}

template <class FA, class FB>
PQR_DEV void small_gram(FA colA, FB colB, int m, int s, int R, double* out) {
  switch (s) {
#define PQR_SG(S) case S: small_gram_t<S>(colA, colB, m, s, R, out); break;
    PQR_SG(1) PQR_SG(2) PQR_SG(4) PQR_SG(8) PQR_SG(16)
#undef PQR_SG
    default: {  // other widths: columns padded to the next power of two (zero B columns)
      // (B columns >= s read column s - 1; their sums are not written: c < s)
      auto cb = [&](int c) { return colB(min(c, s - 1)); };
      if (s <= 4) small_gram_t<4>(colA, cb, m, s, R, out);
      else if (s <= 8) small_gram_t<8>(colA, cb, m, s, R, out);
      else small_gram_t<16>(colA, cb, m, s, R, out);
    }
  }
}

// rows of out (s columns, ld ldr) = rows of [A1 A2] (k columns of A1, then m - k of A2) times M
// (m x s, ld m): one thread per row, S (compile time) accumulators; columns >= t written as 0
template <int S>
PQR_DEV void small_rows_times_m_t(const double* A1, const double* A2, int k, int m, const double* M, int t,
                                  int R, int ldr, double* out) {
  for (int r = threadIdx.x; r < R; r += kSmallThreads) {
    double acc[S];
#pragma unroll
    for (int c = 0; c < S; ++c) acc[c] = 0.0;
    for (int j = 0; j < k; ++j) {
      const double v = A1[j * ldr + r];
#pragma unroll
      for (int c = 0; c < S; ++c) acc[c] = fma(v, M[j + c * m], acc[c]);
    }
    for (int j = k; j < m; ++j) {
      const double v = A2[(j - k) * ldr + r];
#pragma unroll
      for (int c = 0; c < S; ++c) acc[c] = fma(v, M[j + c * m], acc[c]);
    }
#pragma unroll
    for (int c = 0; c < S; ++c) out[c * ldr + r] = c < t ? acc[c] : 0.0;
  }
}

PQR_DEV void small_rows_times_m(const double* A1, const double* A2, int k, int m, int s, const double* M, int t,
                                int R, int ldr, double* out) {
  switch (s) {
#define PQR_SR(S) case S: small_rows_times_m_t<S>(A1, A2, k, m, M, t, R, ldr, out); break;
    PQR_SR(1) PQR_SR(2) PQR_SR(3) PQR_SR(4) PQR_SR(5) PQR_SR(6) PQR_SR(7) PQR_SR(8)
    PQR_SR(9) PQR_SR(10) PQR_SR(11) PQR_SR(12) PQR_SR(13) PQR_SR(14) PQR_SR(15) PQR_SR(16)
#undef PQR_SR
    default: break;
  }
}

__global__ void __launch_bounds__(kSmallThreads) k_cholqr2_small(SmallArgs a) {
  SM_TR(0);
  extern __shared__ __align__(16) double smd[];
  const int tid = threadIdx.x, G = gridDim.x, b = blockIdx.x;
  const int k = a.k, s = a.s, m = k + s;
  const int64_t r0 = (int64_t)b * a.R;
  const int64_t rem = a.n - r0;
  const int R = rem <= 0 ? 0 : (rem < a.R ? (int)rem : a.R);
  const int ldr = a.R;  // even: 16-byte row pairs; lanes read consecutive rows (conflict free)
  const int kp = k > 0 ? k : 1;
  double* sA = smd;                          // m x ldr: [Q X] rows
  double* sU = sA + (size_t)m * ldr;         // s x ldr: U1 rows
  double* sM = sU + (size_t)s * ldr;         // m x s: M of the current pass
  double* sP1 = sM + (size_t)m * s;          // k x s each (ld k)
  double* sP2 = sP1 + (size_t)kp * s;
  double* sPf = sP2 + (size_t)kp * s;
  double* sN1 = sPf + (size_t)kp * s;        // 16 x 16 each
  double* sN2 = sN1 + kSMax * kSMax;
  double* sNf = sN2 + kSMax * kSMax;
  int* si = reinterpret_cast<int*>(sNf + kSMax * kSMax);
  // si: [0] t1 [1] t2 [2] tf [3] defl1 [4] defl2 [16..31] piv1 [32..47] piv2

  // ---- load this CTA's rows of [Q X] with cp.async (16-byte row pairs when aligned) ----
  if (a.vec) {
    const int RP = (R + 1) >> 1;
    for (int e = tid; e < m * RP; e += kSmallThreads) {
      const int j = e / RP, r = 2 * (e - j * RP);
      const double* src = j < k ? a.Q + r0 + r + (int64_t)j * a.ldq : a.X + r0 + r + (int64_t)(j - k) * a.ldx;
      const uint32_t dst = smem_u32(sA + j * ldr + r);
      if (r + 1 < R)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src) : "memory");
      else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(src) : "memory");
    }
  } else {
    for (int e = tid; e < m * R; e += kSmallThreads) {
      const int j = e / R, r = e - j * R;
      const double* src = j < k ? a.Q + r0 + r + (int64_t)j * a.ldq : a.X + r0 + r + (int64_t)(j - k) * a.ldx;
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(sA + j * ldr + r)), "l"(src)
                   : "memory");
    }
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  SM_TR(1);
  // ---- pass 1: W1_b = [Q X]_b^T X_b ----
  small_gram([&](int j) { return sA + j * ldr; }, [&](int c) { return sA + (k + c) * ldr; }, m, s, R,
             a.part1 + (size_t)b * m * s);
  SM_TR(2);
  grid_barrier(a.bar, G);
  SM_TR(3);
  FactorArgs f{};
  f.W = a.part1; f.w_stride = (int64_t)m * s; f.nparts = G; f.ldw = m; f.k = k; f.s = s; f.s_dev = nullptr;
  f.tol2 = a.tol2; f.eta = a.eta;
  f.P = sP1; f.ldp = max(1, k); f.N = sN1; f.ldn = kSMax; f.M = sM; f.ldm = m;
  f.t_out = si + 0; f.piv_out = si + 16; f.deflated = si + 3;
  factor_body(f);
  __syncthreads();
  SM_TR(4);
  const int t1 = si[0];
  // ---- U1_b = [Q X]_b M1: one thread per row, all s columns in registers ----
  small_rows_times_m(sA, sA + (size_t)k * ldr, k, m, s, sM, t1, R, ldr, sU);
  __syncthreads();
  const double* fin = sU;   // the block whose rows become U
  int tfin = t1;
  if (!a.single) {
    // ---- pass 2: W2_b = [Q U1]_b^T U1_b ----
    small_gram([&](int j) { return j < k ? sA + j * ldr : sU + (j - k) * ldr; },
               [&](int c) { return sU + c * ldr; }, m, s, R, a.part2 + (size_t)b * m * s);
    SM_TR(5);
    grid_barrier(a.bar, 2 * G);
    SM_TR(6);
    FactorArgs f2{};
    f2.W = a.part2; f2.w_stride = (int64_t)m * s; f2.nparts = G; f2.ldw = m; f2.k = k; f2.s = s; f2.s_dev = si + 0;
    f2.tol2 = 0.0; f2.eta = 0.0;
    f2.P = sP2; f2.ldp = max(1, k); f2.N = sN2; f2.ldn = kSMax; f2.M = sM; f2.ldm = m;
    f2.t_out = si + 1; f2.piv_out = si + 32; f2.deflated = si + 4;
    f2.P1 = sP1; f2.ldp1 = max(1, k); f2.N1 = sN1; f2.ldn1 = kSMax; f2.t1_dev = si + 0; f2.s0 = s;
    f2.Pf = sPf; f2.ldpf = max(1, k); f2.Nf = sNf; f2.ldnf = kSMax; f2.tf = si + 2;
    factor_body(f2);
    __syncthreads();
    SM_TR(7);
    tfin = si[1];
    // ---- U_b = [Q U1]_b M2 (into sA's X columns: not read in this phase; thread r owns row r) ----
    double* sOut = sA + (size_t)k * ldr;
    small_rows_times_m(sA, sU, k, m, s, sM, tfin, R, ldr, sOut);
    __syncthreads();
    fin = sOut;
  }
  SM_TR(8);
  // ---- outputs ----
  for (int e = tid; e < s * R; e += kSmallThreads) {
    const int c = e / R, r = e - c * R;
    const double v = fin[c * ldr + r];
    a.U[r0 + r + (int64_t)c * a.ldu] = v;
    if (a.U2 && c < tfin) a.U2[r0 + r + (int64_t)c * a.ldu2] = v;
  }
  if (b == 0) {
    const double* Pfin = a.single ? sP1 : sPf;
    const double* Nfin = a.single ? sN1 : sNf;
    for (int e = tid; e < k * s; e += kSmallThreads) {
      const int i = e % k, c = e / k;
      const double v = Pfin[i + c * max(1, k)];
      a.Pf[i + (int64_t)c * a.ldp] = v;
      if (a.Pout) a.Pout[i + (int64_t)c * a.ldpo] = v;
    }
    for (int e = tid; e < kSMax * kSMax; e += kSmallThreads) {
      a.Nf[e] = Nfin[e];
      const int i = e % kSMax, c = e / kSMax;
      if (a.Nout && i < s && c < s) a.Nout[i + (int64_t)c * a.ldno] = Nfin[e];
    }
    if (tid < 8) {
      const int v = tid == 0 ? si[0]
                    : tid == 1 ? (a.single ? si[0] : si[1])
                    : tid == 2 ? (a.single ? si[0] : si[2])
                    : tid == 3 ? si[3]
                    : tid == 4 ? (a.single ? 0 : si[4])
                               : 0;
      a.ints[tid] = v;
      if (a.hints) a.hints[tid] = v;
    }
    if (tid < kSMax) {
      a.ints[16 + tid] = si[16 + tid];
      a.ints[32 + tid] = a.single ? 0 : si[32 + tid];
    }
  }
  // ---- reset the grid-barrier counter: the CTA that arrives last (every other CTA has passed
  // its last barrier wait) zeroes it for the next launch ----
  if (tid == 0) {
    const unsigned int nbar = a.single ? 1u : 2u;
    if (atomicAdd(a.bar, 1u) == (nbar + 1u) * (unsigned int)G - 1u) atomicExch(a.bar, 0u);
  }
}

}  // namespace pqr
