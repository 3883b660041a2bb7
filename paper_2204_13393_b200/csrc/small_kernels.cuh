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
//      CTA 0 writes P, N, t and the pivots.
// The grid barrier is a counter in global memory (zeroed by the host before the launch);
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
  int64_t n; int k; int s; int R;    // R = rows per CTA (the last CTA may have fewer)
  int single;                        // PQR_SINGLE_PASS: Alg. 7 only
  double tol2, eta;                  // deflation of pass 1 (R3b)
  double* U; int64_t ldu;            // n x s output (columns >= t zero)
  double* U2; int64_t ldu2;          // optional copy of the valid columns (basis append)
  double* part1; double* part2;      // [G][m*s] partial Grams
  unsigned int* bar;                 // grid barrier counter (0 at launch)
  // outputs (global): final P (k x s, ld ldp), N (16 x 16 layout, ld kSMax), ints as the handle's
  double* Pf; int ldp; double* Nf; int* ints;
};

// x . y over R shared-memory entries: four accumulators (independent chains), fixed order
PQR_DEV double sdot(const double* x, const double* y, int R) {
  double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
  int r = 0;
  for (; r + 4 <= R; r += 4) {
    c0 += x[r] * y[r];
    c1 += x[r + 1] * y[r + 1];
    c2 += x[r + 2] * y[r + 2];
    c3 += x[r + 3] * y[r + 3];
  }
  for (; r < R; ++r) c0 += x[r] * y[r];
  return (c0 + c1) + (c2 + c3);
}

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

// shared memory: A = [Q X] rows (m x ldr), U1 (s x ldr), M (m x s), P1, P2, Pf (k x s),
// N1, N2, Nf (16 x 16), 64 ints
inline size_t small_smem(int R, int k, int s) {
  const int ldr = R | 1;
  const int m = k + s, kp = k > 0 ? k : 1;
  return ((size_t)(m + s) * ldr + (size_t)m * s + 3 * (size_t)kp * s + 3 * kSMax * kSMax) * sizeof(double) +
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

__global__ void __launch_bounds__(kSmallThreads) k_cholqr2_small(SmallArgs a) {
  SM_TR(0);
  extern __shared__ __align__(16) double smd[];
  const int tid = threadIdx.x, G = gridDim.x, b = blockIdx.x;
  const int k = a.k, s = a.s, m = k + s;
  const int64_t r0 = (int64_t)b * a.R;
  const int64_t rem = a.n - r0;
  const int R = rem <= 0 ? 0 : (rem < a.R ? (int)rem : a.R);
  const int ldr = a.R | 1;  // odd leading dimension: strided column reads are conflict free
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

  // ---- load this CTA's rows of [Q X]: 8-byte cp.async, all of a thread's copies in flight ----
  for (int e = tid; e < m * R; e += kSmallThreads) {
    const int j = e / R, r = e - j * R;
    const double* src = j < k ? a.Q + r0 + r + (int64_t)j * a.ldq : a.X + r0 + r + (int64_t)(j - k) * a.ldx;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(sA + j * ldr + r)), "l"(src) : "memory");
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  SM_TR(1);
  // ---- pass 1: W1_b = [Q X]_b^T X_b ----
  for (int e = tid; e < m * s; e += kSmallThreads) {
    const int j = e % m, c = e / m;
    a.part1[(size_t)b * m * s + e] = sdot(sA + j * ldr, sA + (k + c) * ldr, R);
  }
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
  // ---- U1_b = [Q X]_b M1 ----
  for (int e = tid; e < s * R; e += kSmallThreads) {
    const int c = e / R, r = e - c * R;
    double acc = 0.0;
    if (c < t1)
      for (int j = 0; j < m; ++j) acc += sA[j * ldr + r] * sM[j + c * m];
    sU[c * ldr + r] = acc;
  }
  __syncthreads();
  const double* fin = sU;   // the block whose rows become U
  const double* Mfin = sM;
  int tfin = t1;
  if (!a.single) {
    // ---- pass 2: W2_b = [Q U1]_b^T U1_b ----
    for (int e = tid; e < m * s; e += kSmallThreads) {
      const int j = e % m, c = e / m;
      a.part2[(size_t)b * m * s + e] = sdot(j < k ? sA + j * ldr : sU + (j - k) * ldr, sU + c * ldr, R);
    }
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
    // ---- U_b = [Q U1]_b M2 (into sA's X columns: no longer needed) ----
    double* sOut = sA + (size_t)k * ldr;
    for (int e = tid; e < s * R; e += kSmallThreads) {
      const int c = e / R, r = e - c * R;
      double acc = 0.0;
      if (c < tfin) {
        for (int j = 0; j < k; ++j) acc += sA[j * ldr + r] * sM[j + c * m];
        for (int j = 0; j < s; ++j) acc += sU[j * ldr + r] * sM[k + j + c * m];
      }
      sOut[c * ldr + r] = acc;
    }
    __syncthreads();
    fin = sOut;
    (void)Mfin;
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
      a.Pf[i + (int64_t)c * a.ldp] = Pfin[i + c * max(1, k)];
    }
    for (int e = tid; e < kSMax * kSMax; e += kSmallThreads) a.Nf[e] = Nfin[e];
    if (tid == 0) {
      a.ints[0] = si[0];
      a.ints[1] = a.single ? si[0] : si[1];
      a.ints[2] = a.single ? si[0] : si[2];
      a.ints[3] = si[3];
      a.ints[4] = a.single ? 0 : si[4];
    }
    if (tid < kSMax) {
      a.ints[16 + tid] = si[16 + tid];
      a.ints[32 + tid] = a.single ? 0 : si[32 + tid];
    }
  }
}

}  // namespace pqr
