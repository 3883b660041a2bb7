// stream2_kernels.cuh — CholQR2 streaming passes with a producer warp and warp-private
// 16-row units (§8(a) a1 Gram, a4 update, and the fused a4 + a1 second pass).
//
// One persistent CTA of 8 warps per SM, no CTA barrier in the stream.  The CTA owns a
// contiguous range of 16-row units; unit i lives in shared-memory slot i % NSL and is computed
// by warp i % 8 alone, with all its column steps, so no partial result is ever reduced across
// warps in the stream.  The rows of all m = k + sx columns of [Q X] of a unit (16 rows = 128 B
// per column) are copied with 16-byte cp.async (LDGSTS) and complete the slot's mbarrier (32
// no-increment arrivals).  The warp that has just consumed unit i refills its slot with unit
// i + NSL, so a slot is never overwritten before it is consumed and no `empty` barrier is
// needed; NSL - 8 units are in flight per SM.  Warps drift apart, so the consumer of unit i
// may arrive before fill i / NSL of its slot has been issued (the mbarrier's parity would then
// alias the previous fill): a per-slot count of issued fills, written after the copies are
// issued, is checked first.  (A separate producer warp would put three
// warps on one SM sub-partition and cap the registers at 168 per thread: spills.)
//
// Slot layout: column j occupies 128 B (8 chunks of two rows); chunk (j, row pair p) sits at
// chunk j*8 + (p ^ f(j)), f(j) = 3*(j&1) + 4*((j>>1)&1).  Both fragment read patterns are
// then bank-conflict free without padding (LDS.128 phases of 8 lanes, lane = 4g + q):
//   U phase: column 4kk+q, pair g            -> chunk bits (g0^q0, g1^q0, g2^q1): distinct
//   G phase: column 8mt+g, pair 2q+jj        -> chunk bits (jj^g0, q0^g0, q1^g1): distinct
//
// Per unit (fp64 mma.sync m8n8k4, SASS DMMA):
//   (U) U^T = M^T [Q X]^T: A = M^T fragments held in registers for the whole kernel, B = the
//       slot (rows 2g, 2g+1 of column 4kk+q feed two MMAs), four accumulator chains.  The D
//       fragments leave lane (g, q) holding rows 4q..4q+3 of column g of U.
//   (G) W += [Q U]^T U (fused) or [Q X]^T X (Gram): K = the unit's rows with lane q <-> rows
//       4q..4q+3, so the fused pass's B operand (and the A operand of the U tiles) are the U
//       phase's D fragments as they are — only the tile straddling column k (k % 8 != 0)
//       needs shuffles.  A operand of the Q tiles: two LDS.128 per tile.
// The per-warp W partials are summed over the 8 warps in fixed order at the end, then over the
// CTAs by the last CTA (grid_sum_partials): bitwise reproducible (R7).
#pragma once
#include <algorithm>

#include "common.cuh"

namespace pqr {

#ifndef PQR_S2_UCH
#define PQR_S2_UCH 2  // U-phase accumulator chains per row half (2 or 4)
#endif
#ifndef PQR_S2_CPUNROLL
#define PQR_S2_CPUNROLL 0  // unroll factor of the slot-copy issue loop (0: the compiler's choice; A/B: tools/cpunroll_ab.sh)
#endif
#ifndef PQR_S2_PF
#define PQR_S2_PF 0  // 1: compile the L2 prefetch of later rounds in (S2Args::pf_rounds; measured: no gain)
#endif
#ifndef PQR_S2_GBAR
// what separates the G phase's tile groups when the interleaved refill is compiled out (MT > 12):
// 0 nothing (one basic block), 1 a compiler-level memory barrier, 2 the run-time refill test as
// below 12 tiles (a never-taken-path branch per group).  Measured equal (with PQR_S2_KTEST = 0);
// 2 keeps the code closest to the tuned build
#define PQR_S2_GBAR 2
#endif
#ifndef PQR_S2_KTEST
// 1: every G-phase tile selects its A operand at run time (slot column, or U column through
// shuffles, by 8 mt + 8 <= k); 0: tiles below MT - NT - 1, Q columns for every k, skip the test
// and its shuffles.  Measured (tools/gbar_ab.sh, profiles/r02m_gbar_ab.txt): 0 drops 120 SHFL per
// unit but the weak config's fused pass goes 7.6-7.7 -> 9.1-9.2 ms (ptxas then schedules the tile
// loads differently); configs[1] is the same either way.  So 1.
#define PQR_S2_KTEST 1
#endif
#ifndef PQR_S2_LOOP
#define PQR_S2_LOOP 1  // slot copies issued by a loop over the lane's columns (0: fully unrolled, fresh addresses)
#endif
#ifndef PQR_S2_TG
#define PQR_S2_TG 2  // G-phase tile group (1: each tile's four k-steps back to back; measured best: 2)
#endif
constexpr int kS2Consumers = 8;
constexpr int kS2Threads = 32 * kS2Consumers;
// warp-specialised form (S2Args::ws): + one producer warpgroup that issues every slot copy;
// setmaxnreg splits the launch allocation (384 x 168): 256 x 216 + 128 x 72 <= 384 x 168
constexpr int kS2WsThreads = kS2Threads + 128;
constexpr int kS2WsConsumerRegs = 216, kS2WsProducerRegs = 72;
constexpr int kS2Rows = 16;
constexpr int kS2Gram = 1, kS2Update = 2, kS2Fused = 3;
constexpr int kS2InterleaveMaxMT = 12;  // S2Args::interleave is honoured up to this many column tiles

struct S2Args {
  const double* Q; int64_t ldq;
  const double* X; int64_t ldx;
  int64_t n; int k; int sx;         // slot columns: [Q X], m = k + sx
  int sout;                         // U columns (update / fused; fused: sout = sx)
  const double* M; int ldm;         // m x sout: U = [Q X] M
  const int* t_dev;                 // valid U columns (nullptr: sout); columns >= t are written as zero
  double* U; int64_t ldu;           // n x sout
  double* U2; int64_t ldu2;         // optional second copy of the valid columns (update)
  double* partials;                 // [grid][m * sx]
  double* W; int ldw;               // m x sx
  unsigned int* ticket;
  int nslot;
  int interleave;                   // fused: refill copies interleaved with the G phase (else after it)
  int pf_rounds;                    // L2 prefetch distance in rounds of 8 units (0: off)
  int ws;                           // warp-specialised launch (k_stream2<..., true>, kS2WsThreads)
};

PQR_HOST_DEV int s2_swz(int j) { return 3 * (j & 1) + 4 * ((j >> 1) & 1); }

// WS: the copies are issued by a producer warpgroup (warps 8..11, slot sl by producer warp sl % 4)
// instead of the consuming warp; a consumer releases its slot through the slot's `empty` mbarrier
// (one arrival), and the producer waits on it before the slot's next fill.  The consumer warps
// then issue only their LDS / DMMA / store stream.
template <int MT, int NT, int MODE, bool WS = false>
__global__ void __launch_bounds__(WS ? kS2WsThreads : kS2Threads, 1) k_stream2(S2Args a) {
  constexpr bool DO_U = (MODE & kS2Update) != 0, DO_G = (MODE & kS2Gram) != 0;
  constexpr int MP = MT * 8, SLOT = MP * kS2Rows;  // doubles per slot
  // two output tiles (NT = 2): the M fragments live in shared memory (in registers they would
  // push the kernel past 255 registers: spills); one LDS.64 per k-step and tile
  constexpr bool MSMEM = NT == 2 && DO_U;
  constexpr int MFS = MSMEM ? 2 * MT * NT * 32 : 0;
  extern __shared__ __align__(128) double sm[];
  const int k = a.k, m = k + a.sx, NSL = a.nslot;
  double* sMf = sm + (size_t)NSL * SLOT;  // [2MT][NT][32 lanes] (MSMEM)
  uint64_t* full = reinterpret_cast<uint64_t*>(sMf + MFS);
  uint64_t* empty = full + NSL;  // WS: slot released by its consumer (one arrival)
  volatile int* fills = reinterpret_cast<volatile int*>(full + (WS ? 2 : 1) * NSL);  // fills issued per slot
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, q = lane & 3;

  // slot columns m..MP-1 are never copied: zero them once (finite operands, zero products)
  for (int e = tid; e < NSL * (MP - m) * kS2Rows; e += (WS ? kS2WsThreads : kS2Threads)) {
    const int sl = e / ((MP - m) * kS2Rows), r = e % ((MP - m) * kS2Rows);
    sm[(size_t)sl * SLOT + m * kS2Rows + r] = 0.0;
  }
  if (tid == 0) {
    for (int i = 0; i < NSL; ++i) {
      mbar_init(&full[i], 32);
      if constexpr (WS) mbar_init(&empty[i], 1);
      fills[i] = 0;
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int64_t nunits = (a.n + kS2Rows - 1) / kS2Rows;
  const int64_t ub = nunits * blockIdx.x / gridDim.x;
  const int nu = (int)(nunits * (blockIdx.x + 1) / gridDim.x - ub);

  double acc[DO_G ? MT : 1][NT][2];
#pragma unroll
  for (int i = 0; i < (DO_G ? MT : 1); ++i)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) acc[i][nt][0] = acc[i][nt][1] = 0.0;

  // copies of unit i into its slot: lane (jl, p) copies row pair p of columns jl + 4t
  const int cp_p = lane & 7, cp_jl = lane >> 3;
  const int dsto = cp_jl * kS2Rows + 2 * (cp_p ^ s2_swz(cp_jl));  // f(j) depends on j & 3 = jl only
  const uint32_t sm0 = smem_u32(sm) + 8u * (uint32_t)dsto;
  const double* safe = k > 0 ? a.Q : a.X;
  // unit i (fill f of slot sl): copies, then the slot's arrival, then the issued-fill count.
  // Fully unrolled with immediate shared-memory offsets and a fresh source address per copy:
  // an LDGSTS keeps its address registers until the LSU takes it, so updating one register in
  // a loop stalls on the long scoreboard (measured: 8 % of all stall samples).
  // copy t of unit i (columns jl + 4t, i.e. tile t/2) into the slot at dst; branch-free:
  // columns m..MP-1 are zero-filled (they are the slot's zero padding)
  auto copy_t = [&](uint32_t dst, int64_t row, int bytes, int t) {
    const int j = cp_jl + 4 * t;
    const int nb = j < m ? bytes : 0;
    const double* src = j < k ? a.Q + (int64_t)j * a.ldq : a.X + (int64_t)(j - k) * a.ldx;
    cp_async16_s(dst + 512u * t, nb ? src + row : safe, nb);
  };
  auto unit_row = [&](int64_t i) { return (ub + i) * kS2Rows + 2 * cp_p; };
  auto row_bytes = [&](int64_t row) { return row + 1 < a.n ? 16 : (row < a.n ? 8 : 0); };
  auto publish = [&](int sl, int f) {
    cp_async_mbar_arrive(&full[sl]);
    __syncwarp();
    if (lane == 0) fills[sl] = f + 1;
  };
  const int nq = k > cp_jl ? (k - cp_jl + 3) / 4 : 0;       // this lane's Q columns
  const int nx = m > cp_jl ? (m - cp_jl + 3) / 4 - nq : 0;  // ... and X columns
  auto issue = [&](int64_t i, int sl, int f) {
    const uint32_t dst = sm0 + 8u * (uint32_t)(sl * SLOT);
    const int64_t row = unit_row(i);
    const int bytes = row_bytes(row);
    if constexpr (PQR_S2_LOOP != 0) {
      double* d = sm + (size_t)sl * SLOT + dsto;
      const double* src = a.Q + (int64_t)cp_jl * a.ldq + row;
      int t = 0;
#if PQR_S2_CPUNROLL > 0
      constexpr int kCpUnroll = PQR_S2_CPUNROLL;
#pragma unroll kCpUnroll
#endif
      for (; t < nq; ++t, src += 4 * a.ldq) cp_async16(d + t * 64, bytes ? src : safe, bytes);
      src = a.X + (int64_t)(cp_jl + 4 * nq - k) * a.ldx + row;
      for (int e = 0; e < nx; ++e, ++t, src += 4 * a.ldx) cp_async16(d + t * 64, bytes ? src : safe, bytes);
    } else {
#pragma unroll
      for (int t = 0; t < 2 * MT; ++t) copy_t(dst, row, bytes, t);
    }
    publish(sl, f);
  };
  // consumer-side CTA barrier (WS: the producer warps have left; named barrier 1 over the consumers)
  auto csync = [&]() {
    if constexpr (WS) asm volatile("bar.sync 1, %0;\n" ::"n"(kS2Threads) : "memory");
    else __syncthreads();
  };
  if constexpr (WS) {
    if (warp >= kS2Consumers) {
      // ---------------- producer warps: every fill of every slot, in unit order ----------------
      asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(kS2WsProducerRegs));
      // producer warp pw owns slots pw, pw + 4, ...: all fills of a slot come from one warp, in
      // order, so the empty barrier's phase is never more than one behind (no parity aliasing)
      bool done = false;
      for (int f = 0; !done; ++f)
        for (int sl = warp - kS2Consumers; sl < NSL; sl += 4) {
          const int i = f * NSL + sl;
          if (i >= nu) {
            done = true;
            break;
          }
          if (f > 0) mbar_wait(&empty[sl], (uint32_t)((f - 1) & 1));
          const int64_t row = unit_row(i);
          const int bytes = row_bytes(row);
          double* d = sm + (size_t)sl * SLOT + dsto;
          const double* src = a.Q + (int64_t)cp_jl * a.ldq + row;
          int t = 0;
          for (; t < nq; ++t, src += 4 * a.ldq) cp_async16(d + t * 64, bytes ? src : safe, bytes);
          src = a.X + (int64_t)(cp_jl + 4 * nq - k) * a.ldx + row;
          for (int e = 0; e < nx; ++e, ++t, src += 4 * a.ldx) cp_async16(d + t * 64, bytes ? src : safe, bytes);
          publish(sl, f);
        }
      return;
    }
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(kS2WsConsumerRegs));
  } else {
    for (int i = warp; i < nu && i < NSL; i += kS2Consumers) issue(i, i, 0);
  }
  {
    // ---------------- consumer warps ----------------
    double mreg[(DO_U && !MSMEM) ? 2 * MT : 1][NT];
#pragma unroll
    for (int kk = 0; kk < (DO_U ? 2 * MT : 1); ++kk)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int j = 4 * kk + q, c = 8 * nt + g;
        const double v = (DO_U && j < m && c < a.sout) ? a.M[j + (int64_t)c * a.ldm] : 0.0;
        if constexpr (MSMEM) {
          if (warp == 0) sMf[(kk * NT + nt) * 32 + lane] = v;
        } else {
          mreg[kk][nt] = v;
        }
      }
    if constexpr (MSMEM) csync();
    const int tv = a.t_dev ? *a.t_dev : a.sout;
    const int offU = q * kS2Rows + 2 * (g ^ s2_swz(q));  // column 4kk+q, pair g (+ kk*64)
    const int sg = s2_swz(g & 3);
    const int offG0 = g * kS2Rows + 2 * ((2 * q) ^ sg), offG1 = g * kS2Rows + 2 * ((2 * q + 1) ^ sg);  // + mt*128
    // Gram mode: B operand = X column 8nt + g (slot column k + 8nt + g), rows 4q..4q+3
    int offB0[NT], offB1[NT];
    bool bval[NT];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const int j = k + 8 * nt + g;
      bval[nt] = 8 * nt + g < a.sx;
      const int jc = bval[nt] ? j : 0;
      offB0[nt] = jc * kS2Rows + 2 * ((2 * q) ^ s2_swz(jc));
      offB1[nt] = jc * kS2Rows + 2 * ((2 * q + 1) ^ s2_swz(jc));
    }
    int sl = warp, f = 0;  // slot and fill of unit i (i = f * NSL + sl)
    // L2 prefetch: round r = units 8r..8r+7 of this CTA (128 contiguous rows); warp (r % 8)
    // prefetches round r + pf_rounds when it starts its unit of round r (one bulk L2 prefetch of
    // the round's rows per column, spread over the lanes): the slot copies then hit L2
    const int pfr = PQR_S2_PF != 0 ? a.pf_rounds : 0;
    if (pfr > 0) {
      // rounds 0..pfr-1 up front: warp w takes round w (if < pfr)
      for (int r = warp; r < pfr; r += kS2Consumers) {
        const int64_t r0 = (ub + (int64_t)r * kS2Consumers) * kS2Rows;
        const int64_t rr = min((int64_t)kS2Consumers * kS2Rows, a.n - r0);
        if (rr > 0)
          for (int j = lane; j < m; j += 32) {
            const double* c = (j < k ? a.Q + (int64_t)j * a.ldq : a.X + (int64_t)(j - k) * a.ldx) + r0;
            prefetch_l2(c, (uint32_t)(((rr * 8) + 15) & ~15));
          }
      }
    }
    for (int i = warp; i < nu; i += kS2Consumers) {
      if (pfr > 0) {
        const int r = i / kS2Consumers + pfr;  // i = 8 * round + warp
        if ((i / kS2Consumers) % kS2Consumers == warp) {
          const int64_t r0 = (ub + (int64_t)r * kS2Consumers) * kS2Rows;
          const int64_t rr = min(min((int64_t)kS2Consumers * kS2Rows, a.n - r0), (ub + nu) * kS2Rows - r0);
          if (rr > 0)
            for (int j = lane; j < m; j += 32) {
              const double* c = (j < k ? a.Q + (int64_t)j * a.ldq : a.X + (int64_t)(j - k) * a.ldx) + r0;
              prefetch_l2(c, (uint32_t)(((rr * 8) + 15) & ~15));
            }
        }
      }
      while (fills[sl] <= f) {
      }
      mbar_wait(&full[sl], (uint32_t)(f & 1));
      const double* slot = sm + (size_t)sl * SLOT;
      double u[NT][4];
      if constexpr (DO_U) {
        constexpr int UC = PQR_S2_UCH;
        double dx[NT][UC][2], dy[NT][UC][2];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int e = 0; e < UC; ++e) dx[nt][e][0] = dx[nt][e][1] = dy[nt][e][0] = dy[nt][e][1] = 0.0;
#pragma unroll
        for (int kk = 0; kk < 2 * MT; ++kk) {
          const double2 b = lds2(slot + offU + kk * 64);
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            double mv;
            if constexpr (MSMEM) mv = sMf[(kk * NT + nt) * 32 + lane];
            else mv = mreg[kk][nt];
            dmma884(dx[nt][kk % UC][0], dx[nt][kk % UC][1], mv, b.x);
            dmma884(dy[nt][kk % UC][0], dy[nt][kk % UC][1], mv, b.y);
          }
        }
        const int64_t row = (ub + i) * kS2Rows + 4 * q;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const int c = 8 * nt + g;
          const bool valid = c < tv;
          double sx0 = dx[nt][0][0] + dx[nt][1][0], sx1 = dx[nt][0][1] + dx[nt][1][1];
          double sy0 = dy[nt][0][0] + dy[nt][1][0], sy1 = dy[nt][0][1] + dy[nt][1][1];
          if constexpr (UC == 4) {
            sx0 += dx[nt][2][0] + dx[nt][3][0];
            sx1 += dx[nt][2][1] + dx[nt][3][1];
            sy0 += dy[nt][2][0] + dy[nt][3][0];
            sy1 += dy[nt][2][1] + dy[nt][3][1];
          }
          u[nt][0] = valid ? sx0 : 0.0;  // row 4q
          u[nt][1] = valid ? sy0 : 0.0;  // row 4q + 1
          u[nt][2] = valid ? sx1 : 0.0;  // row 4q + 2
          u[nt][3] = valid ? sy1 : 0.0;  // row 4q + 3
          if (c < a.sout) {
            double* up = a.U + (int64_t)c * a.ldu + row;
            if (row + 3 < a.n) {
              st2(up, u[nt][0], u[nt][1]);
              st2(up + 2, u[nt][2], u[nt][3]);
            } else {
#pragma unroll
              for (int e = 0; e < 3; ++e)
                if (row + e < a.n) up[e] = u[nt][e];
            }
            if (MODE == kS2Update && a.U2 && valid) {
              double* u2 = a.U2 + (int64_t)c * a.ldu2 + row;
              if (row + 3 < a.n) {
                st2(u2, u[nt][0], u[nt][1]);
                st2(u2 + 2, u[nt][2], u[nt][3]);
              } else {
#pragma unroll
                for (int e = 0; e < 3; ++e)
                  if (row + e < a.n) u2[e] = u[nt][e];
              }
            }
          }
        }
      }
      // fused pass: the refill of this slot with unit i + NSL is interleaved with the G phase,
      // tile by tile, each tile's copies behind the MMAs that consumed its last reads
      // (compile-time off past 12 tiles, where it is slower: the skipped copy blocks would
      // otherwise leave a taken branch per tile group in the MMA stream — instruction-fetch stalls)
      constexpr bool IL_OK = !WS && MODE == kS2Fused && (MT <= kS2InterleaveMaxMT || PQR_S2_GBAR == 2);
      const bool refill = IL_OK && a.interleave && i + NSL < nu;
      const uint32_t rdst = sm0 + 8u * (uint32_t)(sl * SLOT);
      const int64_t rrow = unit_row(i + NSL);
      const int rbytes = row_bytes(rrow);
      if constexpr (DO_G) {
        double bq[NT][4];
        if constexpr (MODE == kS2Fused) {
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int e = 0; e < 4; ++e) bq[nt][e] = u[nt][e];
        } else {
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            const double2 b0 = lds2(slot + offB0[nt]), b1 = lds2(slot + offB1[nt]);
            bq[nt][0] = bval[nt] ? b0.x : 0.0;
            bq[nt][1] = bval[nt] ? b0.y : 0.0;
            bq[nt][2] = bval[nt] ? b1.x : 0.0;
            bq[nt][3] = bval[nt] ? b1.y : 0.0;
          }
        }
        // tiles in groups of TG: the group's A operands first, then its MMAs tile-innermost, so
        // consecutive MMAs of the (in-order) asm stream do not feed each other
        constexpr int TG = PQR_S2_TG;
#pragma unroll
        for (int m0 = 0; m0 < MT; m0 += TG) {
          double av[TG][4];
#pragma unroll
          for (int tg = 0; tg < TG; ++tg) {
            const int mt = m0 + tg;
            if (mt >= MT) break;
            // tiles below MT - NT - 1 are Q columns for every k (k >= 8 (MT - 1 - NT) + 1): no
            // run-time test, so the unrolled tile loop keeps no branch over the shuffle path
            if (MODE != kS2Fused || (PQR_S2_KTEST == 0 && mt < MT - NT - 1) || 8 * mt + 8 <= k) {
              const double2 a0 = lds2(slot + offG0 + mt * 128), a1 = lds2(slot + offG1 + mt * 128);
              av[tg][0] = a0.x; av[tg][1] = a0.y; av[tg][2] = a1.x; av[tg][3] = a1.y;
            } else {
              // fused: column j = 8mt + g of [Q U]: j < k from the slot, j >= k is U column j - k,
              // held by lane ((j - k) & 7, q) in its D fragments
              const int j = 8 * mt + g, c = j - k;
              double2 a0 = make_double2(0.0, 0.0), a1 = a0;
              if (8 * mt < k) {
                a0 = lds2(slot + offG0 + mt * 128);
                a1 = lds2(slot + offG1 + mt * 128);
              }
              const double sv[4] = {a0.x, a0.y, a1.x, a1.y};
              const int src = ((c & 7) << 2) | q;
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const double v0 = __shfl_sync(0xffffffffu, u[0][e], src);
                const double v1 = NT > 1 ? __shfl_sync(0xffffffffu, u[NT - 1][e], src) : 0.0;
                av[tg][e] = c < 0 ? sv[e] : (c < a.sx ? (c < 8 ? v0 : v1) : 0.0);
              }
            }
          }
#pragma unroll
          for (int e = 0; e < 4; ++e)
#pragma unroll
            for (int tg = 0; tg < TG; ++tg)
#pragma unroll
              for (int nt = 0; nt < NT; ++nt)
                if (m0 + tg < MT) dmma884(acc[m0 + tg][nt][0], acc[m0 + tg][nt][1], av[tg][e], bq[nt][e]);
          if constexpr (!IL_OK && PQR_S2_GBAR == 1) asm volatile("" ::: "memory");
          if constexpr (IL_OK) {
            if (refill) {
#pragma unroll
              for (int t = 2 * m0; t < 2 * (m0 + TG); ++t)
                if (t < 2 * MT) copy_t(rdst, rrow, rbytes, t);
            }
          }
        }
      }
      if constexpr (WS) {
        // every lane's reads of the slot have completed (their MMAs have issued): release it
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[sl]);
      } else if (refill) {
        publish(sl, f + 1);
      } else if (!(MODE == kS2Fused && a.interleave) && i + NSL < nu) {
        // every lane's reads of the slot have completed (their MMAs have issued): refill it
        issue(i + NSL, sl, f + 1);
      }
      sl += kS2Consumers;
      if (sl >= NSL) {
        sl -= NSL;
        ++f;
      }
    }
  }
  if constexpr (DO_G) {
    // ---- CTA reduction over the 8 warps (fixed order), then over the CTAs ----
    csync();
    constexpr int PW = MT * NT * 64;  // doubles per warp
    double* red = sm;
    {
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          red[warp * PW + ((mt * NT + nt) * 32 + lane) * 2 + 0] = acc[mt][nt][0];
          red[warp * PW + ((mt * NT + nt) * 32 + lane) * 2 + 1] = acc[mt][nt][1];
        }
    }
    csync();
    double* part = a.partials + (size_t)blockIdx.x * m * a.sx;
    for (int e = tid; e < PW; e += kS2Threads) {
      const int v = e & 1, l = (e >> 1) & 31, rest = e >> 6;
      const int nt = rest % NT, mt = rest / NT;
      const int jj = 8 * mt + (l >> 2), c = 8 * nt + 2 * (l & 3) + v;
      if (jj < m && c < a.sx) {
        double sum = 0.0;
#pragma unroll
        for (int w = 0; w < kS2Consumers; ++w) sum += red[w * PW + e];
        part[jj + (int64_t)c * m] = sum;
      }
    }
    __threadfence();
    csync();
    __shared__ unsigned int s_last;
    if (tid == 0) s_last = (atomicAdd(a.ticket, 1u) == gridDim.x - 1);
    csync();
    if (!s_last) return;
    __threadfence();
    grid_sum_partials(a.partials, gridDim.x, m * a.sx, m, a.W, a.ldw, tid, kS2Threads);
    if (tid == 0) *a.ticket = 0u;
  }
}

// host: shared-memory slots for MT tiles of 8 columns (>= 9: every warp holds one while
// another is in flight), and the launch.  Defined in stream2_*.cu (one translation unit
// per mode, compiled in parallel).
inline size_t s2_mfs(int MT, int NT, int mode) {
  return (NT == 2 && (mode & kS2Update)) ? (size_t)2 * MT * NT * 32 * sizeof(double) : 0;
}
inline int s2_nslot(int MT, int NT, int mode, size_t budget, bool ws = false) {
  const size_t slot = (size_t)MT * 8 * kS2Rows * sizeof(double) + (ws ? 2 : 1) * sizeof(uint64_t) + sizeof(int);
  return (int)std::min<size_t>(24, (budget - 1024 - s2_mfs(MT, NT, mode)) / slot);
}
inline size_t s2_smem(int MT, int NT, int mode, int nslot, bool ws = false) {
  return (size_t)nslot * MT * 8 * kS2Rows * sizeof(double) + s2_mfs(MT, NT, mode) +
         (size_t)nslot * ((ws ? 2 : 1) * sizeof(uint64_t) + sizeof(int));
}

}  // namespace pqr

// launchers (one translation unit per mode): cudaSuccess, or cudaErrorNotSupported when no
// instantiation fits (the caller falls back)
cudaError_t pqr_launch_s2_fused(const pqr::S2Args& a, int grid, cudaStream_t st);
cudaError_t pqr_launch_s2_gram(const pqr::S2Args& a, int grid, cudaStream_t st);
cudaError_t pqr_launch_s2_update(const pqr::S2Args& a, int grid, cudaStream_t st);
