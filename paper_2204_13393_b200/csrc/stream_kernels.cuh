// stream_kernels.cuh — pipelined CholQR2 passes (§8(a) a1 Gram, a4 update).
//
// Design (measured, see DESIGN.md §6 and profiles/r01_*):
//  * A memory-bound fp64 stream needs ~100-200 KB of loads in flight per SM.  The
//    kernels keep NS-1 shared-memory stages in flight with cp.async (LDGSTS, 16 B per
//    thread, zero-fill past n); each stage's arrival is tracked by an mbarrier that
//    every thread arms with cp.async.mbarrier.arrive.noinc, and one barrier per stage
//    protects stage reuse.  One persistent 256-thread CTA per SM.  The per-thread copy
//    tasks are fixed across stages (shifts only, no divisions in the loop).
//  * TMA tensor copies were measured and rejected for this layout: on B200 the TMA
//    unit moves about one box line per ~8 SM cycles, and a line is one column's run
//    of rows (column-major data): 64/128/256/512-byte lines stream at 2.3/4.6/6.6/7.2
//    TB/s (tools/tma_bench.cu), and long lines cannot be swizzled, so the MMA fragment
//    reads (8 columns x 4 row pairs, or 4 columns x 8 row pairs) would hit 2-4-way
//    bank conflicts.  cp.async lets each stage use a padded column stride that makes
//    both fragment patterns conflict-free.
//  * Compute: fp64 mma.sync m8n8k4 (DMMA.8x8x4), fragments read with LDS.128.
//
// k_gram_cpa    W = [Q X]^T X.  Stage = 32 rows x all m columns;
//               warp w handles 8-row sub-slab (w & 3) of every stage for half
//               (w >> 2) of the column tiles; sub-slab warps are summed in fixed order.
// k_update_cpa  U = [Q X] M.  Stage = 128 rows x 16 columns;
//               warp w owns the 16-row unit w of a row block and accumulates U^T over
//               the column chunks in registers.
#pragma once
#include "cholqr_kernels.cuh"
#include "common.cuh"

namespace pqr {

constexpr int kCpaThreads = 256;
constexpr int kCpaWarps = kCpaThreads / 32;

// 16-byte chunk of rows (row, row+1) of a column, zero-filled past n (or for a missing
// column: colp == nullptr).  `safe` is any valid global address (not read when 0 bytes).
PQR_DEV void cp_rows(double* dst, const double* colp, int64_t row, int64_t n, const double* safe) {
  const int bytes = colp ? (row + 1 < n ? 16 : (row < n ? 8 : 0)) : 0;
  cp_async16(dst, bytes ? (const void*)(colp + row) : (const void*)safe, bytes);
}

// ----------------------------------------------------------------------------
// a1: W = [Q X]^T X
// ----------------------------------------------------------------------------
// rows per stage = kGramRB (template: 16 or 32); column stride kGramRB + 8 doubles, i.e.
// 192 B or 320 B = 64 (mod 128): an LDS.128 phase (2 columns x 4 row pairs) touches both
// bank halves once.

struct GramCpaArgs {
  const double* Q; int64_t ldq;
  const double* X; int64_t ldx;
  int64_t n; int k; int s; int NS;
  double* partials;               // [gridDim.x][m*s]
  double* W; int ldw;
  unsigned int* ticket;
};

template <int MTH, int NT, int kGramRB>
__global__ void __launch_bounds__(kCpaThreads, 2) k_gram_cpa(GramCpaArgs a) {
  constexpr int kGramRBP = kGramRB + 8;
  constexpr int SUBS = kGramRB / 8;           // 8-row sub-slabs per stage
  constexpr int GROUPS = kCpaWarps / SUBS;    // column-tile groups
  extern __shared__ __align__(16) double sm[];
  const int k = a.k, s = a.s, m = k + s, MT = (m + 7) >> 3, mp = MT * 8;
  const int NS = a.NS;
  const int stage_dbl = mp * kGramRBP;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gq = lane >> 2, q = lane & 3;
  const int sub = warp % SUBS, half = warp / SUBS;

  // columns m..mp-1 of every stage are never copied: zero them once
  for (int e = tid; e < NS * (mp - m) * kGramRBP; e += kCpaThreads) {
    const int st = e / ((mp - m) * kGramRBP), rem = e % ((mp - m) * kGramRBP);
    sm[(size_t)st * stage_dbl + m * kGramRBP + rem] = 0.0;
  }

  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)NS * stage_dbl);
  uint64_t* empty = full + NS;
  if (tid == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&full[i], kCpaThreads);
      mbar_init(&empty[i], kCpaWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int64_t nrb = (a.n + kGramRB - 1) / kGramRB;
  const int cnt = blockIdx.x < nrb ? (int)((nrb - 1 - blockIdx.x) / gridDim.x + 1) : 0;
  // this thread's copy tasks (fixed across stages): chunk e = tid + 256 t -> column
  // e / (RB/2), row pair e % (RB/2); global pointer and smem offset precomputed once
  constexpr int RP = kGramRB / 2;
  constexpr int TMAX = (kMMax * RP + kCpaThreads - 1) / kCpaThreads;
  const double* tsrc[TMAX];
  int tdst[TMAX];
  int ntask = 0;
#pragma unroll
  for (int t = 0; t < TMAX; ++t) {
    const int e = tid + t * kCpaThreads;
    const int j = e / RP, p = e % RP;
    const bool ok = j < m;
    tsrc[t] = ok ? col_ptr(a.Q, a.ldq, a.X, a.ldx, k, m, j) + 2 * p : a.X;
    tdst[t] = ok ? j * kGramRBP + 2 * p : 0;
    ntask += ok ? 1 : 0;
  }
  int64_t r0_p = (int64_t)blockIdx.x * kGramRB;       // producer row cursor
  const int64_t r0_step = (int64_t)gridDim.x * kGramRB;
  auto issue = [&](int it, int st) {
    if (it < cnt) {
      double* buf = sm + (size_t)st * stage_dbl;
      if (r0_p + kGramRB <= a.n) {
#pragma unroll
        for (int t = 0; t < TMAX; ++t)
          if (t < ntask) cp_async16(buf + tdst[t], tsrc[t] + r0_p, 16);
      } else {
#pragma unroll
        for (int t = 0; t < TMAX; ++t)
          if (t < ntask) {
            const int64_t row = r0_p + ((tid + t * kCpaThreads) % RP) * 2;
            const int bytes = row + 1 < a.n ? 16 : (row < a.n ? 8 : 0);
            cp_async16(buf + tdst[t], bytes ? (const void*)(tsrc[t] + r0_p) : (const void*)a.X, bytes);
          }
      }
      cp_async_mbar_arrive(&full[st]);
      r0_p += r0_step;
    }
  };

  double acc[MTH][NT][2];
#pragma unroll
  for (int i = 0; i < MTH; ++i)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) acc[i][nt][0] = acc[i][nt][1] = 0.0;

  for (int it = 0; it < NS - 1; ++it) issue(it, it);
  const int ro = sub * 8 + 2 * q;
  int st = 0, ph = 0, stp = NS - 1;
  // tiles past MT read the zeroed padding columns (or a valid column) and are discarded
  int aoff[MTH];
#pragma unroll
  for (int i = 0; i < MTH; ++i) {
    const int mt = half * MTH + i;
    aoff[i] = (mt < MT ? 8 * mt + gq : 0) * kGramRBP + ro;
  }
  int boff[NT];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) boff[nt] = (8 * nt + gq < s ? k + 8 * nt + gq : mp - 1) * kGramRBP + ro;
  for (int it = 0; it < cnt; ++it) {
    // stage `stp` last held item it-1: wait until every warp has released it
    if (it >= 1) mbar_wait(&empty[stp], (uint32_t)(((it - 1) / NS) & 1));
    issue(it + NS - 1, stp);
    stp = stp + 1 == NS ? 0 : stp + 1;
    mbar_wait(&full[st], (uint32_t)ph);
    const double* buf = sm + (size_t)st * stage_dbl;
    double2 bv[NT], av[MTH];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) bv[nt] = lds2(buf + boff[nt]);
#pragma unroll
    for (int i = 0; i < MTH; ++i) av[i] = lds2(buf + aoff[i]);
#pragma unroll
    for (int i = 0; i < MTH; ++i)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) dmma884(acc[i][nt][0], acc[i][nt][1], av[i].x, bv[nt].x);
#pragma unroll
    for (int i = 0; i < MTH; ++i)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) dmma884(acc[i][nt][0], acc[i][nt][1], av[i].y, bv[nt].y);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
    if (++st == NS) { st = 0; ph ^= 1; }
  }
  __syncthreads();
  // ---- CTA reduction over the SUBS sub-slab warps of each tile group (fixed order) ----
  const int per_warp = MTH * NT * 64;
  double* red = sm;  // [8 warps][MTH][NT][32][2]
#pragma unroll
  for (int i = 0; i < MTH; ++i)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      red[warp * per_warp + ((i * NT + nt) * 32 + lane) * 2 + 0] = acc[i][nt][0];
      red[warp * per_warp + ((i * NT + nt) * 32 + lane) * 2 + 1] = acc[i][nt][1];
    }
  __syncthreads();
  double* part = a.partials + (size_t)blockIdx.x * m * s;
  for (int e = tid; e < GROUPS * per_warp; e += kCpaThreads) {
    const int hf = e / per_warp, r = e % per_warp;
    const int v = r & 1, l = (r >> 1) & 31, rest = r >> 6;  // rest = i*NT + nt
    const int nt = rest % NT, i = rest / NT;
    const int mt = hf * MTH + i;
    const int jj = 8 * mt + (l >> 2), c = 8 * nt + 2 * (l & 3) + v;
    if (mt < MT && jj < m && c < s) {
      double sum = 0.0;
      for (int sb = 0; sb < SUBS; ++sb) sum += red[(hf * SUBS + sb) * per_warp + r];
      part[jj + (int64_t)c * m] = sum;
    }
  }
  // ---- grid reduction by the last CTA to finish (fixed order over CTAs) ----
  __threadfence();
  __syncthreads();
  __shared__ unsigned int s_last;
  if (tid == 0) s_last = (atomicAdd(a.ticket, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int ms = m * s;
  const int nb = gridDim.x;
  grid_sum_partials(a.partials, nb, ms, m, a.W, a.ldw);
  if (tid == 0) *a.ticket = 0u;
}

// ----------------------------------------------------------------------------
// a4 + a1 fused (second CholQR pass): U1 = [Q X] M1 and W2 = [Q U1]^T U1 in one pass
// ----------------------------------------------------------------------------
// Stage = 32 rows x all m columns of [Q X] (as k_gram_cpa).  Per stage:
//   (U) U1^T = M1^T [Q X]^T for the 32 rows: warp w takes 16-row unit (w & 1) and a
//       quarter (w >> 1) of the k-steps; the 4 partials per unit are summed in fixed
//       order into a shared-memory U1 tile, which is also written to HBM (pass 3 reads it);
//   (G) W2 += [Q U1]^T U1 over the same rows, Q from the stage, U1 from the tile.
// Q and X are read once for both — the second pass of BCGS-PIP+ (PAPER.md:L521-525,
// Alg. 8 lines 3-4) costs one read of [Q X] instead of two.
struct UpdGramArgs {
  const double* Q; int64_t ldq;
  const double* X; int64_t ldx;
  int64_t n; int k; int s; int NS;
  const double* M; int ldm;       // (k+s) x s: U1 = [Q X] M
  const int* t_dev;               // valid U1 columns (t1); columns >= t1 are written as zero
  double* U1; int64_t ldu;        // n x s output
  double* partials;
  double* W; int ldw;
  unsigned int* ticket;
};

constexpr int kFuseRB = 32;
constexpr int kFuseRBP = 40;

template <int MTH, int NT>
__global__ void __launch_bounds__(kCpaThreads, NT == 1 ? 2 : 1) k_update_gram_cpa(UpdGramArgs a) {
  constexpr int SUBS = kFuseRB / 8, GROUPS = kCpaWarps / SUBS;
  extern __shared__ __align__(16) double sm[];
  const int k = a.k, s = a.s, m = k + s, MT = (m + 7) >> 3, mp = MT * 8;
  const int KS = (m + 3) >> 2, mpad = KS * 4, KQ = (KS + 3) / 4;
  const int NS = a.NS;
  const int stage_dbl = mp * kFuseRBP;
  double* sMm = sm + (size_t)NS * stage_dbl;          // [NT][mpad][8]
  double* u1t = sMm + (size_t)NT * mpad * 8;          // U1 tile: [8*NT cols][kFuseRBP]
  double* redU = u1t + 8 * NT * kFuseRBP;             // [8 warps][NT][32 lanes][4]
  uint64_t* full = reinterpret_cast<uint64_t*>(redU + kCpaWarps * NT * 128);
  uint64_t* empty = full + NS;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gq = lane >> 2, q = lane & 3;
  const int sub = warp % SUBS, half = warp / SUBS;
  const int t1 = a.t_dev ? *a.t_dev : s;

  for (int e = tid; e < NS * (mp - m) * kFuseRBP; e += kCpaThreads) {
    const int st = e / ((mp - m) * kFuseRBP), rem = e % ((mp - m) * kFuseRBP);
    sm[(size_t)st * stage_dbl + m * kFuseRBP + rem] = 0.0;
  }
  for (int e = tid; e < NT * mpad * 8; e += kCpaThreads) {
    const int nt = e / (mpad * 8), rem = e % (mpad * 8);
    const int j = rem >> 3, c = 8 * nt + (rem & 7);
    sMm[e] = (j < m && c < s) ? a.M[j + (int64_t)c * a.ldm] : 0.0;
  }
  for (int e = tid; e < 8 * NT * kFuseRBP; e += kCpaThreads) u1t[e] = 0.0;
  if (tid == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&full[i], kCpaThreads);
      mbar_init(&empty[i], kCpaWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int64_t nrb = (a.n + kFuseRB - 1) / kFuseRB;
  const int cnt = blockIdx.x < nrb ? (int)((nrb - 1 - blockIdx.x) / gridDim.x + 1) : 0;
  constexpr int RP = kFuseRB / 2;
  constexpr int TMAX = (kMMax * RP + kCpaThreads - 1) / kCpaThreads;
  const double* tsrc[TMAX];
  int tdst[TMAX];
  int ntask = 0;
#pragma unroll
  for (int t = 0; t < TMAX; ++t) {
    const int e = tid + t * kCpaThreads;
    const int j = e / RP, p = e % RP;
    const bool ok = j < m;
    tsrc[t] = ok ? col_ptr(a.Q, a.ldq, a.X, a.ldx, k, m, j) + 2 * p : a.X;
    tdst[t] = ok ? j * kFuseRBP + 2 * p : 0;
    ntask += ok ? 1 : 0;
  }
  int64_t r0_p = (int64_t)blockIdx.x * kFuseRB;
  const int64_t r0_step = (int64_t)gridDim.x * kFuseRB;
  auto issue = [&](int it, int st) {
    if (it < cnt) {
      double* buf = sm + (size_t)st * stage_dbl;
      if (r0_p + kFuseRB <= a.n) {
#pragma unroll
        for (int t = 0; t < TMAX; ++t)
          if (t < ntask) cp_async16(buf + tdst[t], tsrc[t] + r0_p, 16);
      } else {
#pragma unroll
        for (int t = 0; t < TMAX; ++t)
          if (t < ntask) {
            const int64_t row = r0_p + ((tid + t * kCpaThreads) % RP) * 2;
            const int bytes = row + 1 < a.n ? 16 : (row < a.n ? 8 : 0);
            cp_async16(buf + tdst[t], bytes ? (const void*)(tsrc[t] + r0_p) : (const void*)a.X, bytes);
          }
      }
      cp_async_mbar_arrive(&full[st]);
      r0_p += r0_step;
    }
  };

  double acc[MTH][NT][2];
#pragma unroll
  for (int i = 0; i < MTH; ++i)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) acc[i][nt][0] = acc[i][nt][1] = 0.0;
  for (int it = 0; it < NS - 1; ++it) issue(it, it);
  const int ro = sub * 8 + 2 * q;
  // Gram tiles of [Q U1]: lanes whose column is < k read the stage, the others the U1 tile
  int aoff[MTH];
  bool ain_u[MTH];
#pragma unroll
  for (int i = 0; i < MTH; ++i) {
    const int mt = half * MTH + i;
    const int j = mt < MT ? 8 * mt + gq : 0;
    ain_u[i] = j >= k;
    aoff[i] = (j >= k ? j - k : j) * kFuseRBP + ro;
  }
  int boff[NT];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) boff[nt] = (8 * nt + gq) * kFuseRBP + ro;
  const int uu = warp & 1, kq = warp >> 1;       // update: unit, k-step quarter
  const int kk0 = kq * KQ, kk1 = min(KS, kk0 + KQ);
  // M1^T fragments of this warp's k-steps, held for the whole kernel (KQ <= MTH)
  double mreg[MTH][NT];
#pragma unroll
  for (int i = 0; i < MTH; ++i)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) mreg[i][nt] = kk0 + i < kk1 ? sMm[(nt * mpad + 4 * (kk0 + i) + q) * 8 + gq] : 0.0;
  int st = 0, ph = 0, stp = NS - 1;
  int64_t r0 = (int64_t)blockIdx.x * kFuseRB;
  for (int it = 0; it < cnt; ++it) {
    if (it >= 1) mbar_wait(&empty[stp], (uint32_t)(((it - 1) / NS) & 1));
    issue(it + NS - 1, stp);
    stp = stp + 1 == NS ? 0 : stp + 1;
    mbar_wait(&full[st], (uint32_t)ph);
    const double* buf = sm + (size_t)st * stage_dbl;
    // ---- (U) partial U1^T over this warp's k-steps ----
    double d[NT][2][2];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) d[nt][0][0] = d[nt][0][1] = d[nt][1][0] = d[nt][1][1] = 0.0;
    // k-steps past this warp's quarter have zero M fragments (mreg) and read a clamped, valid
    // column of the stage (finite data), so no predicate is needed
#pragma unroll
    for (int i = 0; i < MTH; ++i) {
      {
        const int kc = min(kk0 + i, KS - 1);
        const double2 av = lds2(buf + (4 * kc + q) * kFuseRBP + 16 * uu + 2 * gq);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          dmma884(d[nt][0][0], d[nt][0][1], mreg[i][nt], av.x);
          dmma884(d[nt][1][0], d[nt][1][1], mreg[i][nt], av.y);
        }
      }
    }
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      double* rp = redU + ((warp * NT + nt) * 32 + lane) * 4;
      rp[0] = d[nt][0][0]; rp[1] = d[nt][0][1]; rp[2] = d[nt][1][0]; rp[3] = d[nt][1][1];
    }
    __syncthreads();
    // combine the 4 k-quarters of each unit (fixed order) into the U1 tile and HBM
    for (int e = tid; e < 2 * NT * 128; e += kCpaThreads) {
      const int u = e / (NT * 128), rest = e % (NT * 128);
      const int nt = rest / 128, l = (rest % 128) >> 2, v = rest & 3;
      double val = 0.0;
#pragma unroll
      for (int qq = 0; qq < 4; ++qq) val += redU[(((qq * 2 + u) * NT + nt) * 32 + l) * 4 + v];
      // v: 0 = even MMA c0 (row 4q), 1 = even c1 (row 4q+2), 2 = odd c0 (4q+1), 3 = odd c1 (4q+3)
      const int lq = l & 3, lg = l >> 2;
      const int row = 16 * u + 4 * lq + ((v & 1) ? 2 : 0) + (v >> 1);
      const int col = 8 * nt + lg;
      const double w = col < t1 ? val : 0.0;
      u1t[col * kFuseRBP + row] = w;
      const int64_t grow = r0 + row;
      if (col < s && grow < a.n) a.U1[grow + (int64_t)col * a.ldu] = w;
    }
    __syncthreads();
    // ---- (G) W2 += [Q U1]^T U1 over the stage's rows ----
    double2 bv[NT], avv[MTH];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) bv[nt] = lds2(u1t + boff[nt]);
#pragma unroll
    for (int i = 0; i < MTH; ++i) avv[i] = lds2((ain_u[i] ? u1t : buf) + aoff[i]);
#pragma unroll
    for (int i = 0; i < MTH; ++i)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) dmma884(acc[i][nt][0], acc[i][nt][1], avv[i].x, bv[nt].x);
#pragma unroll
    for (int i = 0; i < MTH; ++i)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) dmma884(acc[i][nt][0], acc[i][nt][1], avv[i].y, bv[nt].y);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
    if (++st == NS) { st = 0; ph ^= 1; }
    r0 += r0_step;
  }
  __syncthreads();
  // ---- CTA reduction over the SUBS sub-slab warps of each tile group (fixed order) ----
  const int per_warp = MTH * NT * 64;
  double* red = sm;
#pragma unroll
  for (int i = 0; i < MTH; ++i)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      red[warp * per_warp + ((i * NT + nt) * 32 + lane) * 2 + 0] = acc[i][nt][0];
      red[warp * per_warp + ((i * NT + nt) * 32 + lane) * 2 + 1] = acc[i][nt][1];
    }
  __syncthreads();
  double* part = a.partials + (size_t)blockIdx.x * m * s;
  for (int e = tid; e < GROUPS * per_warp; e += kCpaThreads) {
    const int hf = e / per_warp, r = e % per_warp;
    const int v = r & 1, l = (r >> 1) & 31, rest = r >> 6;
    const int nt = rest % NT, i = rest / NT;
    const int mt = hf * MTH + i;
    const int jj = 8 * mt + (l >> 2), c = 8 * nt + 2 * (l & 3) + v;
    if (mt < MT && jj < m && c < s) {
      double sum = 0.0;
      for (int sb = 0; sb < SUBS; ++sb) sum += red[(hf * SUBS + sb) * per_warp + r];
      part[jj + (int64_t)c * m] = sum;
    }
  }
  __threadfence();
  __syncthreads();
  __shared__ unsigned int s_last;
  if (tid == 0) s_last = (atomicAdd(a.ticket, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int ms = m * s;
  const int nb = gridDim.x;
  grid_sum_partials(a.partials, nb, ms, m, a.W, a.ldw);
  if (tid == 0) *a.ticket = 0u;
}

// ----------------------------------------------------------------------------
// a4: U = [Q X] M
// ----------------------------------------------------------------------------
constexpr int kUpdRB = 128;   // rows per row block (8 warps x 16)
constexpr int kUpdRBP = 132;  // column stride (doubles): 1056 B = 32 (mod 128) -> an LDS.128
                              // phase (4 columns x 2 row pairs) hits 4 disjoint bank octets

struct UpdCpaArgs {
  const double* Q; int64_t ldq;
  const double* X; int64_t ldx;
  int64_t n; int k; int sx; int sout;
  const double* M; int ldm;       // (k+sx) x sout
  const int* t_dev;
  double* U; int64_t ldu;
  double* U2; int64_t ldu2;
  int NS;
};

// U^T = M^T [Q X]^T as m8n8k4 MMAs: M-index = output column c, N-index = row, K = column j
// of [Q X].  Lane l reads rows 2(l>>2), 2(l>>2)+1 of column 4kk+(l&3): the even row feeds
// one MMA, the odd row another; the D fragments give each lane 4 consecutive rows.
template <int NT, int kUpdCW>
__global__ void __launch_bounds__(kCpaThreads, 2) k_update_cpa(UpdCpaArgs a) {
  extern __shared__ __align__(16) double sm[];
  const int k = a.k, m = k + a.sx;
  const int NCH = (m + kUpdCW - 1) / kUpdCW, mpad = NCH * kUpdCW;
  const int NS = a.NS;
  constexpr int stage_dbl = kUpdCW * kUpdRBP;
  double* sM = sm;                                  // [NT][mpad][8]
  double* stages = sm + (size_t)NT * mpad * 8;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gq = lane >> 2, q = lane & 3;
  for (int e = tid; e < NT * mpad * 8; e += kCpaThreads) {
    const int nt = e / (mpad * 8), rem = e % (mpad * 8);
    const int j = rem >> 3, c = 8 * nt + (rem & 7);
    sM[e] = (j < m && c < a.sout) ? a.M[j + (int64_t)c * a.ldm] : 0.0;
  }
  uint64_t* full = reinterpret_cast<uint64_t*>(stages + (size_t)NS * stage_dbl);
  uint64_t* empty = full + NS;
  if (tid == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&full[i], kCpaThreads);
      mbar_init(&empty[i], kCpaWarps);
    }
    fence_mbar_init();
  }
  const int t = a.t_dev ? *a.t_dev : a.sout;
  const int64_t nrb = (a.n + kUpdRB - 1) / kUpdRB;
  const int cnt_rb = blockIdx.x < nrb ? (int)((nrb - 1 - blockIdx.x) / gridDim.x + 1) : 0;
  const int cnt = cnt_rb * NCH;
  const double* safe = a.k > 0 ? a.Q : a.X;
  // producer cursor (item = (row block, chunk)); this thread's 4 chunks per stage:
  // e = tid + 256 t -> column (e >> 6) of the chunk, row pair e & 63
  constexpr int TU = kUpdCW * (kUpdRB / 2) / kCpaThreads;
  int ch_p = 0;
  int64_t r0_p = (int64_t)blockIdx.x * kUpdRB;
  const int64_t r0_step = (int64_t)gridDim.x * kUpdRB;
  auto issue = [&](int it, int st) {
    if (it < cnt) {
      double* buf = stages + (size_t)st * stage_dbl;
      const int j0 = ch_p * kUpdCW;
      const bool full_rows = r0_p + kUpdRB <= a.n;
#pragma unroll
      for (int t = 0; t < TU; ++t) {
        const int e = tid + t * kCpaThreads;
        const int jl = e >> 6, p = e & 63;
        const double* cp = col_ptr(a.Q, a.ldq, a.X, a.ldx, k, m, j0 + jl);
        const int64_t row = r0_p + 2 * p;
        const int bytes = !cp ? 0 : (full_rows || row + 1 < a.n ? 16 : (row < a.n ? 8 : 0));
        cp_async16(buf + jl * kUpdRBP + 2 * p, bytes ? (const void*)(cp + row) : (const void*)safe, bytes);
      }
      cp_async_mbar_arrive(&full[st]);
      if (++ch_p == NCH) {
        ch_p = 0;
        r0_p += r0_step;
      }
    }
  };
  __syncthreads();  // sM and barriers ready
  for (int it = 0; it < NS - 1; ++it) issue(it, it);
  double d[NT][2][2], e2[NT][2][2];  // two accumulator sets (even / odd k-steps) for ILP
  const int so = 16 * warp + 2 * gq;
  int st = 0, ph = 0, stp = NS - 1, ch = 0;
  int64_t r0 = (int64_t)blockIdx.x * kUpdRB;
  for (int it = 0; it < cnt; ++it) {
    if (ch == 0) {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int x = 0; x < 2; ++x) d[nt][x][0] = d[nt][x][1] = e2[nt][x][0] = e2[nt][x][1] = 0.0;
    }
    if (it >= 1) mbar_wait(&empty[stp], (uint32_t)(((it - 1) / NS) & 1));
    issue(it + NS - 1, stp);
    stp = stp + 1 == NS ? 0 : stp + 1;
    mbar_wait(&full[st], (uint32_t)ph);
    const double* buf = stages + (size_t)st * stage_dbl;
    const double* mrow = sM + (ch * kUpdCW) * 8 + gq;
    double2 av[kUpdCW / 4];
#pragma unroll
    for (int kk = 0; kk < kUpdCW / 4; ++kk) av[kk] = lds2(buf + (4 * kk + q) * kUpdRBP + so);
#pragma unroll
    for (int kk = 0; kk < kUpdCW / 4; ++kk) {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const double mv = mrow[(nt * mpad + 4 * kk + q) * 8];
        double (&acc)[2][2] = (kk & 1) ? e2[nt] : d[nt];
        dmma884(acc[0][0], acc[0][1], mv, av[kk].x);
        dmma884(acc[1][0], acc[1][1], mv, av[kk].y);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
    if (++st == NS) { st = 0; ph ^= 1; }
    if (++ch == NCH) {
      ch = 0;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int x = 0; x < 2; ++x) {
          d[nt][x][0] += e2[nt][x][0];
          d[nt][x][1] += e2[nt][x][1];
        }
      const int64_t row = r0 + 16 * warp + 4 * q;
      r0 += (int64_t)gridDim.x * kUpdRB;
      const bool full_rows = row + 3 < a.n;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int c = 8 * nt + gq;
        if (c >= a.sout) continue;
        const bool valid = c < t;
        const double v0 = valid ? d[nt][0][0] : 0.0, v1 = valid ? d[nt][1][0] : 0.0;
        const double v2 = valid ? d[nt][0][1] : 0.0, v3 = valid ? d[nt][1][1] : 0.0;
        double* up = a.U + (int64_t)c * a.ldu + row;
        if (full_rows) {
          st2(up, v0, v1);
          st2(up + 2, v2, v3);
        } else {
          if (row + 0 < a.n) up[0] = v0;
          if (row + 1 < a.n) up[1] = v1;
          if (row + 2 < a.n) up[2] = v2;
        }
        if (a.U2 && valid) {
          double* u2 = a.U2 + (int64_t)c * a.ldu2 + row;
          if (full_rows) {
            st2(u2, v0, v1);
            st2(u2 + 2, v2, v3);
          } else {
            if (row + 0 < a.n) u2[0] = v0;
            if (row + 1 < a.n) u2[1] = v1;
            if (row + 2 < a.n) u2[2] = v2;
          }
        }
      }
    }
  }
}

}  // namespace pqr
