// tsqr_wy.cuh — TreeTSPQR level kernels (§4.1 Alg. 9 with Householder local and
// reduction subalgorithms), persistent, with blocked (compact-WY) reflector panels and
// fp64 MMAs (mma.sync m8n8k4 .f64, SASS DMMA).
//
// Blocks of a level (leaf row blocks, or tree nodes) are processed by a persistent grid of
// 640-thread CTAs (one per SM): 16 consumer warps plus a producer warpgroup; CTA i takes
// blocks i, i + grid, ...  The consumer warps form NG groups of NW = 16 / NG warps: one group
// per block (NG = 1, small tree levels), or two groups on alternate blocks of the CTA
// (NG = 2), so that one group's Householder tail overlaps the other group's panels.  A block
// holds R <= 16*NW*UW rows; group warp w owns UW units of 16 rows, lane (g = l>>2, q = l&3)
// keeping rows 16u+4q+{0..3} of columns 8nt+g in registers (the D-fragment layout of the
// update MMA below).  The block's reflectors are grouped in panels (the s reflectors one
// call creates, or one LOR-build chunk): H_a ... H_b = I - V T V^T with
// T^{-1} = I/2 + striu(V^T V) (unit-norm v, Eq. (hh)).
//
//   stage 1 (Q_b^T X):  for each panel in order   Z = V^T X, Z' = T^T Z, X -= V Z'
//   stage 2 (Q_b Y):    for each panel reversed    Z = V^T Y, Z' = T Z,   Y -= V Z'
//
// Memory: everything a block streams (its X — stage 1 only — and every panel V with its
// T) is a "ring item", copied by cp.async.bulk into one of nbuf shared-memory slots and
// completed on that slot's mbarrier.  One producer lane streams the items in block order,
// across block boundaries, so the next block's data lands while this block does its
// Householder tail; a slot is refilled once every warp of the group that held it released
// it (empty mbarrier).
//
// Per panel: Gram Z = V^T x (per-warp DMMA partials) -> group barrier -> fixed-order sum of
// the NW partials -> group barrier -> every warp forms Z'^T = Z^T T (or Z^T T^T) with two
// DMMAs from shared memory -> update x^T -= Z'^T V^T.  Two barriers per panel.
//
// Stage-1 tail (Alg. 6 lines 2-9 on rows C..R-1 of the s new columns; never deflating,
// reading R4): the columns move to a row layout (lane-local rows).  Round c makes one
// group-wide reduction of D_c' = x_c . x_c' over rows >= r = C+c for all c' (c' = c gives
// lambda^2) and broadcasts row r; warp 0 forms the reflector
//   v = (x_c - sigma*lambda e_r) / sqrt(2 lambda (lambda + |x_c[r]|)),  sigma = -sgn(x_c[r]),
// and the coefficients v . x_c' = (D_c' - sigma*lambda x_c'[r]) / sqrt(...) (c' > c: update;
// c' < c: column c of V^T V for T) behind a second barrier.  Then T of the new panel and the
// outputs.
#pragma once
#include "common.cuh"

namespace pqr {

// 16 consumer warps per CTA, as one group or as two groups of 8 on alternate blocks (see the
// kernels at the end); UW below is per-warp units for the group's warp count, the host plans
// in 16-warp units.
#ifndef PQR_WY_ROT8
#define PQR_WY_ROT8 0  // 8-column tail: 0 = fully unrolled rounds, RU > 0 = rotated, RU rounds per group
#endif
constexpr int kWyWarps = 16;                     // consumer warps per CTA
constexpr int kWyThreads = 32 * kWyWarps;        // consumer threads
constexpr int kWyLaunch = kWyThreads + 128;      // + one producer warpgroup (one working lane)
constexpr int kWyConsumerRegs = 112;  // setmaxnreg split of the launch allocation (640 x 96):
                                      // 4 x 128 x 112 + 128 x 24 <= 640 x 96
constexpr int kWyProducerRegs = 24;
constexpr int kWyRowsPerUW = 16 * kWyWarps;  // block rows covered per unit-per-warp
constexpr int kWyMaxW = 16;                  // widest panel
constexpr int kWyHS = 17;                          // Householder-round partials: row stride (padded)
constexpr int kWyHH = 2 * (kWyWarps * kWyHS + 16);  // Householder-round reduction buffers

struct WyLevel {
  int64_t q, rem2;      // block b: q + 2*(b < rem2) rows starting at b*q + 2*min(b, rem2) (even);
  int odd_last;         // ... the last block has one more row when the level's row count is odd
  int nblocks;
  int64_t b0, nrun;     // this launch processes blocks b0 .. b0 + nrun - 1 (host-buffer pipeline chunks)
  const double* X; int64_t ldx;     // stage-1 input (level rows); 16-B aligned, ldx even
  double* V; int64_t ldv;           // reflectors (level rows); column j = reflector j; ldv even,
                                    // and row R of an odd-sized last block is a zero pad row
  double* T; int64_t tstride;       // block b's T area at T + b*tstride; panel at +16*start
  double* out; int64_t ldo;         // stage-1 output: block b -> rows b*cap ...
  int orows;                        // ... rows written per block: min(R, orows) (cap, or C+s for a
                                    // compact GPU-root block that is all-gathered)
  int ovec;                         // out 16-B aligned with even cap and ldo (paired stores)
  const double* cin; int64_t ldci;  // stage-2 coefficients: block b -> rows b*cap ...
  double* Y; int64_t ldy;           // stage-2 output (level rows)
  int yvec;                         // Y 16-B aligned with even ldy (paired stores)
  int cap;
  int RP;                           // smem panel stride (>= max block rows + 1, = 10 mod 16)
  int wmax;                         // widest panel (<= 16) -> smem slot width
  int nbuf;                         // ring slots (>= 2)
  unsigned long long* trace;        // optional phase-cycle counters (tools; nullptr = off)
  // FlatTSPQR chains (§4.2, Alg. 10, Eqs. flat_tsqr / flattspqr_q; leaf level only,
  // nchain = 0 elsewhere): block b continues chain b % nchain.  A "chained" block (b >= nchain)
  // solves the stacked problem [K; X_b], K = the chain's [P; N] so far ((C+s) x s, the previous
  // block's output, kept in the chain slot out + (b % nchain) * cap), so each chain hands one block
  // to the tree instead of one per leaf block.  The carry rows K are not held in the register
  // file: reflector j of a chained block is non-zero on the carry rows only in its panel's rows
  // [x, x + w) (below C+s the carry is zero, and a panel's reflectors start at its own pivot
  // rows), so a panel touches only K[x : x+w, :] — read once and written once, by warp 0:
  //   Z += K[x:x+w]^T Vc (one more MMA pair in warp 0's partial),  K[x:x+w] -= Vc Z'  (-> slot),
  // and the stage-1 tail's pivot rows C+c are the carry rows [C, C+s) (warp 0, in shared memory),
  // every own row lying below every pivot.  Stage 2 walks a chain backwards: K = the block's
  // coefficients (cin slot), own rows start at zero, and the updated K is the coefficient block of
  // the chain's previous block (written back into the cin slot).  Launches of a chained level use
  // grid = nchain / NG and b0 a multiple of nchain.
  // Storage of the carry part of reflector j: rows [j & ~1, (j & ~1) + LS), LS = wmax + 2, at
  // VC + (b*cap + j)*LS; a panel's columns are contiguous there (one bulk copy per panel).
  int nchain, LS;
  double* VC;
};

struct WyPanels {
  const int4* pan;  // (start, width, T offset in the block's T area, merged) per panel, device
  int np;           // panels to apply
};

PQR_DEV int64_t wy_start(const WyLevel& L, int64_t b) { return b * L.q + 2 * (b < L.rem2 ? b : L.rem2); }
PQR_DEV int wy_rows(const WyLevel& L, int64_t b) {
  return (int)(L.q + (b < L.rem2 ? 2 : 0) + (b == L.nblocks - 1 ? L.odd_last : 0));
}

// per-group scratch (doubles) of a level kernel with NW consumer warps per group:
// partials (NW + 1) E, Z (E), Householder-round buffers, diag, T scratch, round coefficients,
// a chained block's carry rows: the stage-1 tail's (E) and three panels' (3 E)
PQR_HOST_DEV constexpr int wy_group_scratch(int NW, int E) {
  return (NW + 1) * E + E + 2 * (NW * kWyHS + 16) + 16 + 512 + 4 * E;
}
// ring slot (doubles): a panel (RP x wm), its T (wm x wm), its columns' carry segments (wm x LS)
PQR_HOST_DEV constexpr int wy_slot(int RP, int wm) { return RP * wm + wm * wm + wm * (wm + 2); }
// shared-memory bytes of a level kernel (host and device agree on this layout)
inline size_t wy_smem_bytes(int RP, int wmax, int cap, int nbuf, int NW, int NG) {
  const int E = wmax * wmax;
  return ((size_t)nbuf * wy_slot(RP, wmax) + (size_t)NG * wy_group_scratch(NW, E)) * sizeof(double) +
         (size_t)(cap + 2) * sizeof(int4) + (size_t)2 * nbuf * sizeof(uint64_t) + 16;
}

// NG groups of NW consumer warps (+ the producer warpgroup).  With NG = 2 the groups take the
// CTA's blocks alternately (group g: its blocks jb = g, g + 2, ...), each with its own scratch
// and named barrier; the producer streams the items in block order as for one group, so while
// one group runs its block's Householder tail the other applies its panels.
template <int NW, int UW, int NT, int WM, bool UP, bool MERGE = false, int NG = 1, bool CH = false, bool NAR = false>
PQR_DEV void wy_body(const WyLevel& L, const WyPanels& P, int C, int s, int Call, int ncol, int merge_,
                     int mtoff) {
  constexpr int NTH = 32 * NW, NLA = NTH * NG + 128;  // consumer threads per group, launch size
  static_assert(NW == 8 || NW == 16, "consumer warps");
  static_assert(NG == 1 || NG == 2, "groups");
  constexpr bool merge = MERGE;  // separate instantiation: the common path carries no merge code
  (void)merge_;
  extern __shared__ __align__(16) double sm[];
  constexpr int wm = WM, MTM = WM / 8;  // widest panel (8 or 16) and its 8-column tiles
  const int RP = L.RP, nbuf = L.nbuf;
  const int SS = wy_slot(RP, wm);  // slot: panel (RP x wm), its T, its carry segments
  const int E = wm * wm;
  const int gtid = threadIdx.x, gwarp = gtid >> 5;
  const int grp = NG > 1 ? (gwarp < NW ? 0 : 1) : 0;  // (producer warps: irrelevant)
  const int GS = wy_group_scratch(NW, E);
  double* ring = sm;
  double* red = ring + (size_t)nbuf * SS + grp * GS;  // E x (NW + 1): per-warp partials, entry-major (padded)
  double* Zs = red + (NW + 1) * E;         // E: reduced Z (ld wm)
  double* hred = Zs + E;                   // 2 x (NW*17 partials + 16 pivot-row values)
  double* diagv = hred + 2 * (NW * kWyHS + 16);  // 16: sigma*lambda of the new columns
  double* tsc = diagv + 16;                // 2 x 16 x 16: V^T V of the new panel, T-column scratch
  double* ctl = tsc + 512;                 // E: carry rows [C, C+s) of a chained block's tail (row-major, ld 8*NT)
  double* kbuf = ctl + E;                  // 3 x E: K[x : x+w, :] of a chained block's panels (ld wm), panel p at p % 3
  // NW x 16 per-warp round coefficients of the 16-column tail: the T-column half of tsc, which the
  // rounds leave free (T is formed after them)
  double* hupd = tsc + 256;
  int4* pans = reinterpret_cast<int4*>(ring + (size_t)nbuf * SS + NG * GS);
  uint64_t* full = reinterpret_cast<uint64_t*>(pans + L.cap + 2);
  uint64_t* empty = full + nbuf;
  // items issued by the producer so far (two groups: a group may run ahead of a slot's phase
  // by more than one, so it first waits until its item has been issued, then on the parity)
  volatile int* issued = reinterpret_cast<volatile int*>(empty + nbuf);

  // tid, warp: within the group
  const int tid = gtid - grp * NTH, warp = tid >> 5, lane = gtid & 31;
  const int g = lane >> 2, q = lane & 3;
  const int np = P.np;
  const int ipb = np + (UP ? 1 : 0);  // ring items per block (stage 1: X first)
  const int64_t nbl = L.nrun;
  const int nb_cta = (int64_t)blockIdx.x < nbl ? (int)((nbl - 1 - blockIdx.x) / gridDim.x + 1) : 0;
  const int64_t total = (int64_t)nb_cta * ipb;
  const bool chains = CH && L.nchain > 0;  // (CH: separate instantiations; others carry no chain code)
  constexpr int LS = WM + 2;              // carry segment rows (WyLevel::LS)
  const bool rev = chains && !UP;  // stage 2 walks the chains backwards

  // never-copied slot parts must hold finite values (they meet zero coefficients)
  for (int e = gtid; e < nbuf * SS; e += NLA) ring[e] = 0.0;
  for (int i = gtid; i < np; i += NLA) pans[i] = P.pan[i];
  if (gtid == 0) {
    *issued = 0;
    for (int i = 0; i < nbuf; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], NW);
    }
    fence_mbar_init();
  }
  fence_proxy_async_smem();
  __syncthreads();

  // ---- producer warp: streams ring item `it` into slot it % nbuf once the consumers have
  // released the slot's previous item (empty barrier, one arrival per consumer warp) ----
  if (gwarp >= NW * NG) {
    if constexpr (NW * NG == 16) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(kWyProducerRegs));
    if (gwarp == NW * NG && lane == 0) {
      for (int it = 0; it < total; ++it) {
        const int pos = it / ipb;
        const int jb = rev ? nb_cta - 1 - pos : pos;
        const int p = it - pos * ipb;
        const int slot = it % nbuf;
        // (sleeping between polls: the power-capped bench runs ~0.7 % faster)
        if (it >= nbuf) mbar_wait_sleep(&empty[slot], (uint32_t)((it / nbuf - 1) & 1));
        const int64_t b = L.b0 + blockIdx.x + (int64_t)jb * gridDim.x;
        const int64_t r0 = wy_start(L, b);
        const int R = wy_rows(L, b);
        double* buf = ring + (size_t)slot * SS;
        uint64_t* bar = &full[slot];
        if (UP && p == 0) {
          const int Re = R & ~1;  // an odd last row is read from global by the consumer
          mbar_arrive_expect_tx(bar, (uint32_t)(s * Re * 8));
          if (Re)
            for (int c = 0; c < s; ++c)
              bulk_g2s(buf + c * RP, L.X + r0 + (int64_t)c * L.ldx, (uint32_t)Re * 8u, bar);
        } else {
          const int4 pn = pans[UP ? p - 1 : np - 1 - p];
          const int Rc = R + (R & 1);  // includes the zero pad row of an odd block
          const uint32_t tb = (uint32_t)((pn.y * pn.y + 1) & ~1) * 8u;
          const bool chained = chains && b >= L.nchain;
          const uint32_t cb = chained ? (uint32_t)(pn.y * LS) * 8u : 0u;  // the columns' carry segments
          mbar_arrive_expect_tx(bar, (uint32_t)pn.y * Rc * 8u + tb + cb);
          for (int j = 0; j < pn.y; ++j)
            bulk_g2s(buf + j * RP, L.V + (int64_t)(pn.x + j) * L.ldv + r0, (uint32_t)Rc * 8u, bar);
          bulk_g2s(buf + RP * wm, L.T + b * L.tstride + pn.z, tb, bar);
          if (chained) bulk_g2s(buf + RP * wm + wm * wm, L.VC + (b * L.cap + pn.x) * LS, cb, bar);
        }
        if constexpr (NG > 1) {
          __threadfence_block();
          *issued = it + 1;
        }
      }
    }
    return;
  }
  if constexpr (NW * NG == 16) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(kWyConsumerRegs));
  // consumer warps only from here: named barrier 1 + group over the group's NTH threads
  auto cbar = [&]() { asm volatile("bar.sync %0, %1;\n" ::"r"(1 + grp), "n"(NTH) : "memory"); };
  // this warp is done with ring item `it` (all of its lanes' reads precede the arrival)
  auto release = [&](int64_t it) {
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[it % nbuf]);
  };
  // fixed-order sum of the NW partials;
  // partials are entry-major with stride NW + 1 (conflict-free for writers and readers)
  // 16 warps: 2 threads per entry (the first 2E threads), 8 partials each, one xor step;
  // 8 warps: one thread per entry (E <= NTH), 8 partials
  const int rz_e = NW == 16 ? tid >> 1 : tid, rz_part = NW == 16 ? tid & 1 : 0;
  const double* rz_src = red + rz_e * (NW + 1) + rz_part;
  auto reduce_Z = [&]() {
    if constexpr (NW == 16) {
      if (tid < 2 * E) {
        double z0 = rz_src[0], z1 = rz_src[2], z2 = rz_src[4], z3 = rz_src[6];
        z0 += rz_src[8];
        z1 += rz_src[10];
        z2 += rz_src[12];
        z3 += rz_src[14];
        double z = (z0 + z1) + (z2 + z3);
        z += __shfl_xor_sync(0xffffffffu, z, 1);
        if (rz_part == 0) Zs[rz_e] = z;
      }
    } else {
      if (tid < E) {
        const double z0 = rz_src[0] + rz_src[4], z1 = rz_src[1] + rz_src[5];
        const double z2 = rz_src[2] + rz_src[6], z3 = rz_src[3] + rz_src[7];
        Zs[rz_e] = (z0 + z2) + (z1 + z3);
      }
    }
  };
  // optional phase tracing (CTA 0, warps 0 and 15, lane 0): cycles per phase in smem.
  // Compiled in only with -DPQR_WY_TRACE (tools: build.py --trace); absent from the product build.
#ifdef PQR_WY_TRACE
  __shared__ unsigned long long s_tr[2][16];
  const bool tr_on = L.trace != nullptr && blockIdx.x == 0 && grp == 0 && lane == 0 && (warp == 0 || warp == NW - 1);
  const int tr_w = warp == 0 ? 0 : 1;
  long long tr_t0 = 0;
  if (tr_on) {
    for (int i = 0; i < 16; ++i) s_tr[tr_w][i] = 0;
    tr_t0 = clock64();
  }
#define WY_TR(k)                                       \
  if (tr_on) {                                         \
    const long long t1_ = clock64();                   \
    s_tr[tr_w][k] += (unsigned long long)(t1_ - tr_t0); \
    tr_t0 = t1_;                                       \
  }
#else
#define WY_TR(k)
#endif

  int64_t it = 0;  // consumer item cursor
  int hpar = 0;    // Householder-round buffer parity
  const int ncnt = nb_cta > grp ? (nb_cta - grp + NG - 1) / NG : 0;  // this group's blocks
  for (int kb = 0; kb < ncnt; ++kb) {
    const int jb = rev ? grp + (ncnt - 1 - kb) * NG : grp + kb * NG;
    it = (int64_t)(rev ? nb_cta - 1 - jb : jb) * ipb;  // this block's first ring item
    const int64_t b = L.b0 + blockIdx.x + (int64_t)jb * gridDim.x;
    const int64_t r0 = wy_start(L, b);
    const int R = wy_rows(L, b);
    const bool chained = chains && b >= L.nchain;  // stacked problem [K; X_b] (see WyLevel)
    const int Rt = R;
    const int64_t cslot = chains ? b % L.nchain : b;  // output (stage 1) / coefficient (stage 2) slot
    // K: the chain slot (stage 1: the chain's [P; N], updated in place into this block's output;
    // stage 2: the coefficients, updated in place into the previous block's)
    double* kslot = UP ? L.out + cslot * L.cap : const_cast<double*>(L.cin) + cslot * L.cap;
    const int64_t kld = UP ? L.ldo : L.ldci;
    // the chain slot is re-read one block later (by the chain's next block) while tens of MB stream
    // through L2: it is written and read with an evict-last policy so that it stays resident
    const uint64_t kpol = chains ? l2_evict_last() : 0ull;
    const bool mrow = 16 * UW * (warp + 1) > Rt;  // warp holds rows >= Rt
    // The chain's previous block (this group's previous one) wrote the slot read below: across
    // warps when either block is a chain's first (its rows are in every warp), else warp 0 to
    // warp 0.
    if (chains && kb > 0) {
      const bool xw = UP ? (chained && b - L.nchain < L.nchain) : !chained;
      if (xw) cbar();
      else __syncwarp();
    }
    // chained block, warp 0: K rows of panel p into kbuf[p % 3] by cp.async, one commit group per
    // panel (panel p + 2's rows are fetched while panel p runs; a panel's rows are disjoint from
    // every other panel's, so the prefetch never reads a row an earlier panel rewrites)
    auto kfetch = [&](int pp) {
      if (pp < np) {
        const int4 pn = pans[UP ? pp : np - 1 - pp];
        double* dst = kbuf + (pp % 3) * E;
        for (int e = lane; e < wm * s; e += 32) {
          const int i = e % wm, c = e / wm;  // (rows i >= w are never read)
          if (i < pn.y) cp_async8_l2pol(dst + i + wm * c, kslot + pn.x + i + (int64_t)c * kld, kpol);
        }
      }
      cp_async_commit();
    };
    if (chained && UP && warp == NW - 1) {  // the stage-1 tail's carry rows [C, C+s) (no panel touches them)
      for (int e = lane; e < 8 * NT * 8 * NT; e += 32) {
        const int i = e / (8 * NT), col = e % (8 * NT);
        if (i < s && col < s) cp_async8_l2pol(ctl + e, kslot + C + i + (int64_t)col * kld, kpol);
        else ctl[e] = 0.0;
      }
      cp_async_commit();
    }
    if (chained && warp == 0) {
      kfetch(0);
      kfetch(1);
    }
    double x[UW][NT][4];
    if (UP) {
      WY_TR(9);
      if constexpr (NG > 1) {
        while (*issued <= it) __nanosleep(256);  // (32 ns polling: -0.8 % on the power-capped bench)
      }
      mbar_wait(&full[it % nbuf], (uint32_t)((it / nbuf) & 1));
      WY_TR(0);
      const double* buf = ring + (size_t)(it % nbuf) * SS;
#pragma unroll
      for (int u = 0; u < UW; ++u)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int row = 16 * (warp * UW + u) + 4 * q + i, c = 8 * nt + g;
            double v = 0.0;
            if (c < s && row < Rt) v = (row == Rt - 1 && (R & 1)) ? L.X[r0 + row + (int64_t)c * L.ldx] : buf[c * RP + row];
            x[u][nt][i] = v;
          }
      release(it);
      ++it;
    } else {
      const double* cb = L.cin + cslot * L.cap;
#pragma unroll
      for (int u = 0; u < UW; ++u)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int row = 16 * (warp * UW + u) + 4 * q + i, c = 8 * nt + g;
            // (a chained block's coefficients are all carry rows: its own rows start at zero)
            x[u][nt][i] = (!chained && row < Call && row < Rt && c < s) ? cb[row + (int64_t)c * L.ldci] : 0.0;
          }
    }

    // ---------------- committed panels ----------------
    for (int p = 0; p < np; ++p, ++it) {
      WY_TR(9);
      if constexpr (NG > 1) {
        while (*issued <= it) __nanosleep(256);  // (32 ns polling: -0.8 % on the power-capped bench)
      }
      mbar_wait(&full[it % nbuf], (uint32_t)((it / nbuf) & 1));
      WY_TR(0);
      const double* vb = ring + (size_t)(it % nbuf) * SS;
      const double* Tg = vb + RP * wm;
      const int w = pans[UP ? p : np - 1 - p].y;
      const int mtn = (w + 7) >> 3;
      double zp[NT][MTM][2];
      // chained block: warp 0 also carries the panel's carry rows K[px : px+w] (see WyLevel)
      const int px = pans[UP ? p : np - 1 - p].x;
      const bool kw = chained && warp == 0;
      const double* vcs = Tg + wm * wm;  // the panel's carry segments: column j at j*LS
      // carry part of reflector px + j on stacked row r (zero outside [px + j, px + w))
      auto vcar = [&](int r, int j) -> double {
        return (j < w && r >= px + j && r < px + w) ? vcs[j * LS + r - ((px + j) & ~1)] : 0.0;
      };
      const double* kb = kbuf + (p % 3) * E;  // K[px + i][c] at kb[i + wm c]
      if (kw) kfetch(p + 2);
      // this panel's K rows have landed (waited for right before their first use)
      auto kready = [&]() {
        cp_async_wait<2>();
        __syncwarp();
      };
      // K[px + 4kk + q][8nt + g] (zero outside the panel's rows and the block's columns)
      auto kcar = [&](int nt, int kk) -> double {
        const int i = 4 * kk + q, c = 8 * nt + g;
        return (i < w && c < s) ? kb[i + wm * c] : 0.0;
      };
      // K[px : px+w] -= Vc Z' (Z'(j, c) from shared memory), written back to the slot: per 8 x 8
      // tile D[c][i] = sum_j Z'(j, c) Vc(px + i, j) by MMAs (A = Z'^T, B = Vc^T)
      auto carry_update = [&](const double* zsrc, int zld) {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int ti = 0; ti < MTM; ++ti) {
            const int c = 8 * nt + g;
            double d0 = 0.0, d1 = 0.0;
#pragma unroll
            for (int kk = 0; kk < 2 * MTM; ++kk) {
              const int j = 4 * kk + q;
              const double a = (j < w && c < s) ? zsrc[j + zld * c] : 0.0;
              dmma884(d0, d1, a, vcar(px + 8 * ti + g, j));
            }
#pragma unroll
            for (int v = 0; v < 2; ++v) {
              const int i = 8 * ti + 2 * q + v;  // D[c][i] in (d0, d1)
              if (i < w && c < s) st_l2pol(kslot + px + i + (int64_t)c * kld, kb[i + wm * c] - (v ? d1 : d0), kpol);
            }
          }
      };
      if constexpr (MTM == 1) {
        // 8-wide panels (stage 1 too since the two-group kernels: 6.65 -> 6.37 ms; with one
        // 16-warp group it was slower there): each warp forms its partial of Z^T = x^T V (A = x from registers,
        // B = V from the slot) and multiplies it by T (stage 1) or T^T (stage 2) right away, so
        // the summed partials are Z'^T itself; after the barriers a lane only loads the two
        // coefficients it needs (no per-warp MMA chain between the second barrier and the update)
        double acc[2][NT][2];
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) acc[h][nt][0] = acc[h][nt][1] = 0.0;
        if (kw) {  // + K[px:px+w]^T Vc (rows px + 4kk + q), first: the unit MMAs hide its latency
          kready();
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int kk = 0; kk < 2; ++kk) dmma884(acc[kk][nt][0], acc[kk][nt][1], kcar(nt, kk), vcar(px + 4 * kk + q, g));
        }
#pragma unroll
        for (int u = 0; u < UW; ++u) {
          const int row = 16 * (warp * UW + u) + 4 * q;
          const double* vp = vb + g * RP + row;
          const double2 a01 = *reinterpret_cast<const double2*>(vp);
          const double2 a23 = *reinterpret_cast<const double2*>(vp + 2);
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            double (&ac)[2] = acc[u & 1][nt];
            dmma884(ac[0], ac[1], x[u][nt][0], a01.x);
            dmma884(ac[0], ac[1], x[u][nt][1], a01.y);
            dmma884(ac[0], ac[1], x[u][nt][2], a23.x);
            dmma884(ac[0], ac[1], x[u][nt][3], a23.y);
          }
        }
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const double p0 = acc[0][nt][0] + acc[1][nt][0];  // Z^T[c = 8nt+g][j = 2q]
          const double p1 = acc[0][nt][1] + acc[1][nt][1];  // Z^T[c][2q + 1]
          double d0 = 0.0, d1 = 0.0;
#pragma unroll
          for (int k4 = 0; k4 < 2; ++k4) {
            const int src = 4 * g + 2 * k4 + (q >> 1);  // holder of Z^T[c][l = 4 k4 + q]
            const double s0 = __shfl_sync(0xffffffffu, p0, src);
            const double s1 = __shfl_sync(0xffffffffu, p1, src);
            const int l = 4 * k4 + q;
            const double bt = (l < w && g < w) ? (UP ? Tg[l + w * g] : Tg[g + w * l]) : 0.0;
            dmma884(d0, d1, (q & 1) ? s1 : s0, bt);
          }
          // D[c = 8nt+g][j = 2q + v] of this warp's partial of Z'^T
          red[((2 * q) + wm * (8 * nt + g)) * (NW + 1) + warp] = d0;
          red[((2 * q + 1) + wm * (8 * nt + g)) * (NW + 1) + warp] = d1;
        }
        WY_TR(1);
        cbar();  // B1: partials complete; every warp is done with the previous item
        WY_TR(2);
        WY_TR(3);
        reduce_Z();
        WY_TR(4);
        cbar();  // B2: Z'^T complete
        WY_TR(5);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const double2 z2 = *reinterpret_cast<const double2*>(Zs + 2 * q + wm * (8 * nt + g));
          zp[nt][0][0] = z2.x;
          zp[nt][0][1] = z2.y;
        }
        if (kw) carry_update(Zs, wm);  // Zs[j + wm c] = Z'(j, c)
      } else {
      // Z = V^T x: per-warp partials, two accumulator chains over alternate units
      double acc[2][MTM][NT][2];
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int mt = 0; mt < MTM; ++mt)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) acc[h][mt][nt][0] = acc[h][mt][nt][1] = 0.0;
#pragma unroll
      for (int mt = 0; mt < MTM; ++mt) {
        if (mt < mtn) {
          if (kw) {  // + Vc^T K[px:px+w] (rows px + 4kk + q), before the unit MMAs
            if (mt == 0) kready();
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
              for (int kk = 0; kk < 4; ++kk)
                dmma884(acc[kk & 1][mt][nt][0], acc[kk & 1][mt][nt][1], vcar(px + 4 * kk + q, 8 * mt + g), kcar(nt, kk));
          }
#pragma unroll
          for (int u = 0; u < UW; ++u) {
            const int row = 16 * (warp * UW + u) + 4 * q;
            const double* vp = vb + (8 * mt + g) * RP + row;
            const double2 a01 = *reinterpret_cast<const double2*>(vp);
            const double2 a23 = *reinterpret_cast<const double2*>(vp + 2);
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
              double (&ac)[2] = acc[u & 1][mt][nt];
              dmma884(ac[0], ac[1], a01.x, x[u][nt][0]);
              dmma884(ac[0], ac[1], a01.y, x[u][nt][1]);
              dmma884(ac[0], ac[1], a23.x, x[u][nt][2]);
              dmma884(ac[0], ac[1], a23.y, x[u][nt][3]);
            }
          }
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int v = 0; v < 2; ++v)
              red[((8 * mt + g) + wm * (8 * nt + 2 * q + v)) * (NW + 1) + warp] = acc[0][mt][nt][v] + acc[1][mt][nt][v];
        }
      }
      WY_TR(1);
      cbar();  // B1: partials complete; every warp is done with the previous item
      WY_TR(2);
      WY_TR(3);
      reduce_Z();
      WY_TR(4);
      cbar();  // B2: Z complete
      WY_TR(5);
      // Z'^T = Z^T T (stage 1) or Z^T T^T (stage 2): lane gets Z'[8jt+2q+v][8nt+g].
      // 8-wide panels: every warp forms it (two MMAs).  16-wide panels: warps 0-3 form one
      // 8x8 tile each into shared memory (tsc: free outside the stage-1 tail) behind one
      // more barrier, instead of 16 MMAs in every warp.
      // (a chained block always: warp 0's carry update reads Z' from tsc)
      const bool shared_zp = (NT > 1 && mtn == 2) || chained;
      if (MTM == 2 && shared_zp) {
        if (warp < 4) {
          const int jt = warp >> 1, nt = warp & 1, jj = 8 * jt + g;
          double d0 = 0.0, d1 = 0.0;
#pragma unroll
          for (int k4 = 0; k4 < 4; ++k4) {
            const int l = 4 * k4 + q;
            const double a = l < 8 * mtn ? Zs[l + wm * (8 * nt + g)] : 0.0;
            const double bt = (l < w && jj < w) ? (UP ? Tg[l + w * jj] : Tg[jj + w * l]) : 0.0;
            dmma884(d0, d1, a, bt);
          }
          // D[m = c = 8nt+g][n = j = 8jt+2q+v]: store Z'[j][c] at tsc[j + 16 c]
          tsc[(8 * jt + 2 * q) + 16 * (8 * nt + g)] = d0;
          tsc[(8 * jt + 2 * q + 1) + 16 * (8 * nt + g)] = d1;
        }
        cbar();
        if (kw) carry_update(tsc, 16);  // tsc[j + 16 c] = Z'(j, c)
      }
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int jt = 0; jt < MTM; ++jt) {
          zp[nt][jt][0] = zp[nt][jt][1] = 0.0;
          if (MTM == 2 && shared_zp) {
            zp[nt][jt][0] = tsc[(8 * jt + 2 * q) + 16 * (8 * nt + g)];
            zp[nt][jt][1] = tsc[(8 * jt + 2 * q + 1) + 16 * (8 * nt + g)];
          } else if (jt < mtn) {
            const int jj = 8 * jt + g;
#pragma unroll
            for (int k4 = 0; k4 < 2 * MTM; ++k4) {
              if (k4 < 2 * mtn) {
                const int l = 4 * k4 + q;
                const double a = Zs[l + wm * (8 * nt + g)];
                const double bt = (l < w && jj < w) ? (UP ? Tg[l + w * jj] : Tg[jj + w * l]) : 0.0;
                dmma884(zp[nt][jt][0], zp[nt][jt][1], a, bt);
              }
            }
          }
        }
      }
      // x^T -= Z'^T V^T
#pragma unroll
      for (int kk = 0; kk < 2 * MTM; ++kk) {
        if (kk < 2 * mtn) {
          const int j = 8 * (kk >> 1) + 2 * q + (kk & 1);
          double am[NT];
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) am[nt] = -zp[nt][kk >> 1][kk & 1];
#pragma unroll
          for (int u = 0; u < UW; ++u) {
            const int row = 16 * (warp * UW + u) + 2 * g;
            const double2 bv = *reinterpret_cast<const double2*>(vb + j * RP + row);
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
              dmma884(x[u][nt][0], x[u][nt][2], am[nt], bv.x);  // even rows 4q, 4q+2
              dmma884(x[u][nt][1], x[u][nt][3], am[nt], bv.y);  // odd rows 4q+1, 4q+3
            }
          }
        }
      }
      if (!(UP && merge && p == np - 1)) {  // merging: the last panel stays for the tail
        release(it);
      }
      WY_TR(6);
      if (mrow) {  // rows >= R stay zero (stale slot rows may be non-zero)
#pragma unroll
        for (int u = 0; u < UW; ++u)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int i = 0; i < 4; ++i)
              if (16 * (warp * UW + u) + 4 * q + i >= Rt) x[u][nt][i] = 0.0;
      }
    }

    if constexpr (!UP) {
      // ---------------- stage-2 output: Y_b (columns >= t written as zero) ----------------
      // (a chained block's carry coefficients went back into the chain slot panel by panel)
#pragma unroll
      for (int u = 0; u < UW; ++u)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const int c = 8 * nt + g;
          if (c >= ncol) continue;
          const int row = 16 * (warp * UW + u) + 4 * q;
          double* yp = L.Y + r0 + row + (int64_t)c * L.ldy;
          const bool ok = c < s;
#pragma unroll
          for (int i = 0; i < 4; i += 2) {
            const double v0 = ok ? x[u][nt][i] : 0.0, v1 = ok ? x[u][nt][i + 1] : 0.0;
            if (L.yvec && row + i + 1 < Rt) {
              st2(yp + i, v0, v1);
            } else {
              if (row + i < Rt) yp[i] = v0;
              if (row + i + 1 < Rt) yp[i + 1] = v1;
            }
          }
        }
    } else {
    WY_TR(9);
    // ---------------- stage-1 tail: Householder QR of rows C..R-1 of the s new columns ----------------
    // Row layout: an 8-lane butterfly transpose inside every q-group gives lane (g, q) RPL = UW/2
    // whole rows (all 8*NT columns), so each round's dot products are lane-local.  Round c:
    //   D_c' = sum over rows >= r = C+c of x_c x_c' for every c' (one reduction: lane-local,
    //   warp reduce-scatter, 16 warp partials), pivot row r broadcast; then every lane knows
    //   v = (x_c - sigma*lambda e_r) / sqrt(2 lambda (lambda + |x_c[r]|)), sigma = -sgn(x_c[r]),
    //   v . x_c' = (D_c' - sigma*lambda x_c'[r]) / sqrt(...) for c' > c (the update), and
    //   v_c' . v_c by the same formula for c' < c (column c of V^T V, for T).
    constexpr int RPL = UW / 2;   // rows per lane in the row layout
    // columns per row (NAR: calls with s <= 4 — Arnoldi's blocks and every panel merge — keep 4)
    static_assert(!NAR || NT == 1, "narrow tail: one 8-column tile");
    constexpr int S8 = NAR ? 4 : 8 * NT;
    // Chained block: the tail's pivot rows C + c are the carry rows [C, C+s) (the chain's N so far;
    // no panel touches them).  They take the spare register rows [crow, crow + s) at the end of the
    // group's rows (chained blocks hold <= crow own rows) and join the rounds like own rows, with
    // stacked index C + (row - crow); every own row lies below every pivot.
    constexpr int crow = 16 * NW * UW - WM;
    if (chained) {
      if (warp == NW - 1) {  // ctl was fetched by this warp at the block's start
        cp_async_wait<0>();
        __syncwarp();
      }
#pragma unroll
      for (int u = 0; u < UW; ++u)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int row = 16 * (warp * UW + u) + 4 * q + i, c = 8 * nt + g;
            if (row >= crow) x[u][nt][i] = (row - crow < s && c < s) ? ctl[(row - crow) * S8 + c] : 0.0;
          }
    }
    double xr[RPL][S8];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      double a[4 * UW];  // slot 4u + i of this lane's column 8nt + g; block p = slots p*RPL ..
#pragma unroll
      for (int u = 0; u < UW; ++u)
#pragma unroll
        for (int i = 0; i < 4; ++i) a[4 * u + i] = x[u][nt][i];
      // element (lane g, block p) moves to (lane p, block g): swap one index bit per stage
#pragma unroll
      for (int mb = 4; mb >= 1; mb >>= 1) {
        const bool up = (g & mb) != 0;
#pragma unroll
        for (int pb = 0; pb < 8; ++pb) {
          if (pb & mb) continue;
#pragma unroll
          for (int e = 0; e < RPL; ++e) {
            double& lo = a[pb * RPL + e];
            double& hi = a[(pb | mb) * RPL + e];
            const double recv = __shfl_xor_sync(0xffffffffu, up ? lo : hi, 4 * mb);
            if (up) lo = recv; else hi = recv;
          }
        }
      }
#pragma unroll
      for (int pb = 0; pb < 8; ++pb)
#pragma unroll
        for (int e = 0; e < RPL; ++e)
          if (8 * nt + pb < S8) xr[e][8 * nt + pb] = a[pb * RPL + e];
    }
    int rowk[RPL];  // block-local rows of this lane
#pragma unroll
    for (int e = 0; e < RPL; ++e) {
      const int sg = g * RPL + e;
      rowk[e] = 16 * (warp * UW + (sg >> 2)) + 4 * q + (sg & 3);
    }
    // stacked row index of each of this lane's rows (chained: own rows below every pivot, carry rows
    // at C + (row - crow), unused rows never >= a pivot)
    int srow[RPL];
#pragma unroll
    for (int e = 0; e < RPL; ++e)
    {
      srow[e] = !chained ? rowk[e] : (rowk[e] < R ? (1 << 24) : (rowk[e] >= crow && rowk[e] - crow < s ? C + rowk[e] - crow : -1));
      // opaque to the compiler: otherwise it specialises the whole unrolled tail for srow == rowk
      // (unchained blocks) and keeps two copies of it (+3 K instructions: instruction-cache misses)
      if constexpr (CH) asm volatile("" : "+r"(srow[e]));
    }
    double* Gs = tsc;  // strict upper part of V^T V (ld 16), column c written in round c by tid 0
    // Round scalars, formed by every warp from the NW warp partials of hb (the same fixed summation
    // order in every warp and lane: bitwise-identical values), so a round needs one barrier:
    //   lambda, sigma = -sgn(u0), v's scale inv = 1/sqrt(2 lambda (lambda + |u0|)), wr = u0 - sigma*lambda,
    //   fvc[c'] = 2 v . x_c' = 2 inv (D_c' - sigma*lambda x_c'[r]) (c' > c: update coefficient;
    //   c' < c: twice column c of V^T V, recorded for T by warp 0).  hb is double-buffered by round
    //   parity: a warp's reads of round c precede its arrival at round c + 1's barrier.
    auto round_scalars = [&](int c, const double* hb, double (&fvc)[S8], double& inv, double& wr) {
      constexpr int NP = 32 / S8, WPP = NW / NP;  // lane groups, warps per group
      const int v = lane & (S8 - 1), part = lane / S8;
      const double* hv = hb + part * WPP * kWyHS + v;
      double tot = 0.0;
#pragma unroll
      for (int ww = 0; ww < WPP; ++ww) tot += hv[ww * kWyHS];
#pragma unroll
      for (int mb = S8; mb < 32; mb <<= 1) tot += __shfl_xor_sync(0xffffffffu, tot, mb);
      const double lam2 = __shfl_sync(0xffffffffu, tot, c);
      const double u0 = hb[NW * kWyHS + c];
      const double lam = sqrt(lam2);
      const double sigma = (u0 >= 0.0) ? -1.0 : 1.0;  // sigma = -sgn(u0), sgn(0) = +1
      const double diag = sigma * lam;
      const double nv2 = 2.0 * lam * (lam + fabs(u0));
      inv = nv2 > 0.0 ? rsqrt(nv2) : 0.0;  // identity reflector if lambda == 0 (R4)
      wr = u0 - diag;
      const double fv = v == c ? 0.0 : 2.0 * inv * (tot - diag * hb[NW * kWyHS + v]);
#pragma unroll
      for (int cc = 0; cc < S8; ++cc) fvc[cc] = __shfl_sync(0xffffffffu, fv, cc);
      if (warp == 0) {
        if (lane < c) Gs[lane + 16 * c] = 0.5 * fv;
        if (lane == 0) diagv[c] = diag;
      }
    };
    WY_TR(10);
    if constexpr (S8 <= 8 && PQR_WY_ROT8 == 0) {
#pragma unroll
    for (int c = 0; c < S8; ++c) {
      if (c >= s) break;
      const int r = C + c;
      double D[S8];
#pragma unroll
      for (int cc = 0; cc < S8; ++cc) D[cc] = 0.0;
#pragma unroll
      for (int e = 0; e < RPL; ++e)
        if (srow[e] >= r) {
#pragma unroll
          for (int cc = 0; cc < S8; ++cc) D[cc] = fma(xr[e][c], xr[e][cc], D[cc]);
        }
      // warp reduce-scatter of the S8 values (fixed xor tree): lane ends with value vi
#pragma unroll
      for (int mb = 16, w = S8; w > 1; mb >>= 1, w >>= 1) {
        const bool up = (lane & mb) != 0;
#pragma unroll
        for (int j = 0; j < w / 2; ++j) {
          const double send = up ? D[j] : D[j + w / 2];
          const double keep = up ? D[j + w / 2] : D[j];
          D[j] = keep + __shfl_xor_sync(0xffffffffu, send, mb);
        }
      }
      constexpr int LG = 32 / S8;  // lanes sharing a value after the scatter
#pragma unroll
      for (int m = 1; m < LG; m <<= 1) D[0] += __shfl_xor_sync(0xffffffffu, D[0], m);
      const int vi = (lane / LG) & (S8 - 1);
      double* hb = hred + hpar * (NW * kWyHS + 16);
      hpar ^= 1;
      if ((lane & (LG - 1)) == 0) hb[warp * kWyHS + vi] = D[0];
#pragma unroll
      for (int e = 0; e < RPL; ++e)
        if (srow[e] == r) {
#pragma unroll
          for (int cc = 0; cc < S8; ++cc) hb[NW * kWyHS + cc] = xr[e][cc];
        }
      WY_TR(11);
      cbar();  // the round's only barrier: partials and pivot row complete
      WY_TR(12);
      double fvc[S8];
      double inv, wr;
      round_scalars(c, hb, fvc, inv, wr);
      WY_TR(13);
#pragma unroll
      for (int e = 0; e < RPL; ++e)
        if (srow[e] >= r) {
          const double vv = (srow[e] == r ? wr : xr[e][c]) * inv;
#pragma unroll
          for (int cc = c + 1; cc < S8; ++cc) xr[e][cc] = fma(-fvc[cc], vv, xr[e][cc]);
          xr[e][c] = vv;
        }
    }
    } else {
    {
    // 16 columns, rotated register file: entering a group of RU rounds with base c0, xr[e][j] holds
    // column (c0 + j) mod 16, so round c = c0 + cj pivots on the compile-time index cj and every
    // register index is static (no select chains, no per-column predicates); the group ends by
    // rotating the columns by RU (16 rounds: back to identity).  Coefficients of finished columns
    // are zero, so the update is one unpredicated FMA per element (an exact no-op there).
    // (8 columns too unless PQR_WY_ROT8 = 0: the fully unrolled 8 rounds make the kernel large
    // enough to miss in the instruction cache while the other group runs the panel code)
    constexpr int RU = S8 == 8 ? (PQR_WY_ROT8 > 0 ? PQR_WY_ROT8 : 1) : 4;
    double* wup = hupd + warp * 16;  // this warp's update coefficients of the round
#pragma unroll 1
    for (int c0 = 0; c0 < S8; c0 += RU) {
#pragma unroll
      for (int cj = 0; cj < RU; ++cj) {
        const int c = c0 + cj;
        if (c < s) {
          const int r = C + c;
          double D[S8];
#pragma unroll
          for (int j = 0; j < S8; ++j) D[j] = 0.0;
#pragma unroll
          for (int e = 0; e < RPL; ++e)
            if (srow[e] >= r) {
#pragma unroll
              for (int j = 0; j < S8; ++j) D[j] = fma(xr[e][cj], xr[e][j], D[j]);
            }
#pragma unroll
          for (int mb = 16, w = S8; w > 1; mb >>= 1, w >>= 1) {
            const bool up = (lane & mb) != 0;
#pragma unroll
            for (int j = 0; j < w / 2; ++j) {
              const double send = up ? D[j] : D[j + w / 2];
              const double keep = up ? D[j + w / 2] : D[j];
              D[j] = keep + __shfl_xor_sync(0xffffffffu, send, mb);
            }
          }
          constexpr int LG = 32 / S8;  // lanes sharing a value after the scatter
#pragma unroll
          for (int m = 1; m < LG; m <<= 1) D[0] += __shfl_xor_sync(0xffffffffu, D[0], m);
          const int vi = (lane / LG) & (S8 - 1);  // rotated index of the value this lane holds
          double* hb = hred + hpar * (NW * kWyHS + 16);
          hpar ^= 1;
          if ((lane & (LG - 1)) == 0) hb[warp * kWyHS + vi] = D[0];
#pragma unroll
          for (int e = 0; e < RPL; ++e)
            if (srow[e] == r) {
#pragma unroll
              for (int j = 0; j < S8; ++j) hb[NW * kWyHS + j] = xr[e][j];
            }
          WY_TR(11);
          cbar();  // the round's only barrier
          WY_TR(12);
          double inv, wr;
          {
            // every warp sums the NW partials of its value j = lane & (S8-1) (fixed order) and forms
            // the scalars; column (c0 + j) mod S8: > c update target, < c finished (column c of V^T V)
            constexpr int NP = 32 / S8, WPP = NW / NP;
            const int j = lane & (S8 - 1), part = lane / S8;
            const double* hv = hb + part * WPP * kWyHS + j;
            double tot = 0.0;
#pragma unroll
            for (int ww = 0; ww < WPP; ++ww) tot += hv[ww * kWyHS];
#pragma unroll
            for (int mb = S8; mb < 32; mb <<= 1) tot += __shfl_xor_sync(0xffffffffu, tot, mb);
            const double lam2 = __shfl_sync(0xffffffffu, tot, cj);
            const double u0 = hb[NW * kWyHS + cj];
            const double lam = sqrt(lam2);
            const double sigma = (u0 >= 0.0) ? -1.0 : 1.0;  // sigma = -sgn(u0), sgn(0) = +1
            const double diag = sigma * lam;
            const double nv2 = 2.0 * lam * (lam + fabs(u0));
            inv = nv2 > 0.0 ? rsqrt(nv2) : 0.0;  // identity reflector if lambda == 0 (R4)
            wr = u0 - diag;
            const double fv = 2.0 * inv * (tot - diag * hb[NW * kWyHS + j]);
            const int col = (c0 + j) & (S8 - 1);
            if (lane < S8) wup[j] = col > c ? fv : 0.0;
            if (warp == 0) {
              if (lane < S8 && col < c) Gs[col + 16 * c] = 0.5 * fv;
              if (lane == 0) diagv[c] = diag;
            }
            __syncwarp();
          }
          WY_TR(13);
          double up[S8];
#pragma unroll
          for (int j = 0; j < S8; j += 2) {
            const double2 u2 = *reinterpret_cast<const double2*>(wup + j);
            up[j] = u2.x;
            up[j + 1] = u2.y;
          }
#pragma unroll
          for (int e = 0; e < RPL; ++e)
            if (srow[e] >= r) {
              const double vv = (srow[e] == r ? wr : xr[e][cj]) * inv;
#pragma unroll
              for (int j = 0; j < S8; ++j)
                if (j != cj) xr[e][j] = fma(-up[j], vv, xr[e][j]);
              xr[e][cj] = vv;
            }
          __syncwarp();  // wup is rewritten next round
        }
      }
      // rotate by RU: column (c0 + RU + j) mod S8 to index j
#pragma unroll
      for (int e = 0; e < RPL; ++e) {
        double tmp[S8];
#pragma unroll
        for (int j = 0; j < S8; ++j) tmp[j] = xr[e][(j + RU) & (S8 - 1)];
#pragma unroll
        for (int j = 0; j < S8; ++j) xr[e][j] = tmp[j];
      }
    }
    }
    }
    // sigma*lambda (diagv) of the last round is read by every warp below
    cbar();
    WY_TR(7);
    // ---------------- T of the new panel: T^{-1} = I/2 + striu(V^T V) (warp 0) ----------------
    __syncwarp();
    if (tid < s) {
      const int c = tid;
      double* col = tsc + 256 + 16 * c;
      for (int i = 0; i < kWyMaxW; ++i) col[i] = 0.0;
      col[c] = 2.0;  // 1 / (1/2)
      for (int i = c - 1; i >= 0; --i) {
        double acc = 0.0;
        for (int l = i + 1; l <= c; ++l) acc += Gs[i + 16 * l] * col[l];
        col[i] = -acc * 2.0;
      }
      double* Tn = L.T + b * L.tstride + 16 * C;
      for (int i = 0; i < s; ++i) Tn[i + c * s] = i <= c ? col[i] : 0.0;
    }
    __syncwarp();
    if constexpr (merge) {
      // The previous panel (width w1, still in its slot) and the new one (s = 8 - w1) become
      // one 8-wide panel: H_prev H_new = I - [V1 V2] [T1, -T1 (V1^T V2) T2; 0, T2] [V1 V2]^T.
      // V1^T V2 takes one more reduction (lane-local products in the row layout).
      const int64_t hit = it - 1;  // the held item
      const double* v1 = ring + (size_t)(hit % nbuf) * SS;
      constexpr int w1 = 4;  // merges pair two 4-wide panels (host: s == 4 after a 4-wide panel)
      const double* T1 = v1 + RP * wm;
      double Dp[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) Dp[i] = 0.0;
#pragma unroll
      for (int e = 0; e < RPL; ++e) {
        const int row = rowk[e];
#pragma unroll
        for (int j = 0; j < w1; ++j) {
          const double a1 = v1[j * RP + row];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const double v2 = srow[e] >= C + c ? xr[e][c] : 0.0;
            Dp[j * 4 + c] = fma(a1, v2, Dp[j * 4 + c]);
          }
        }
      }
#pragma unroll
      for (int mb = 16, w = 16; w > 1; mb >>= 1, w >>= 1) {
        const bool up = (lane & mb) != 0;
#pragma unroll
        for (int j = 0; j < w / 2; ++j) {
          const double send = up ? Dp[j] : Dp[j + w / 2];
          const double keep = up ? Dp[j + w / 2] : Dp[j];
          Dp[j] = keep + __shfl_xor_sync(0xffffffffu, send, mb);
        }
      }
      Dp[0] += __shfl_xor_sync(0xffffffffu, Dp[0], 1);
      double* hb = hred + hpar * (NW * kWyHS + 16);
      hpar ^= 1;
      if ((lane & 1) == 0) hb[warp * kWyHS + ((lane >> 1) & 15)] = Dp[0];
      cbar();
      if (warp == 0) {
        // C = V1^T V2 (w1 x s, entry j*s + c): lane l sums value l & 15 over half the warps, xor 16
        const int v = lane & 15, part = lane >> 4;
        double tot = 0.0;
#pragma unroll
        for (int ww = 0; ww < NW / 2; ++ww) tot += hb[(part * (NW / 2) + ww) * kWyHS + v];
        tot += __shfl_xor_sync(0xffffffffu, tot, 16);
        double* Cm = tsc + 256 + 16 * 8;  // 16 scratch words after the T columns (s <= 8 here)
        if (lane < 16) Cm[lane] = tot;
        __syncwarp();
        // T_m (8 x 8, ld 8): [T1, -T1 C T2; 0, T2]; T2 column c = col scratch of thread c
        double* Tm = L.T + b * L.tstride + mtoff;
        for (int e2 = lane; e2 < 64; e2 += 32) {
          const int i = e2 & 7, jj = e2 >> 3;
          double val = 0.0;
          if (i < w1 && jj < w1) {
            val = i <= jj ? T1[i + w1 * jj] : 0.0;
          } else if (i >= w1 && jj >= w1) {
            const int i2 = i - w1, j2 = jj - w1;
            val = i2 <= j2 ? tsc[256 + 16 * j2 + i2] : 0.0;
          } else if (i < w1 && jj >= w1) {
            const int j2 = jj - w1;
            for (int a = i; a < w1; ++a) {
              double cta = 0.0;  // (C T2)[a][j2]
              for (int bb = 0; bb <= j2; ++bb) cta += Cm[a * s + bb] * tsc[256 + 16 * j2 + bb];
              val -= T1[i + w1 * a] * cta;
            }
          }
          Tm[i + 8 * jj] = val;
        }
      }
      release(hit);
    }
    WY_TR(8);
    // ---------------- outputs: [P_b; N_b] to the parent slot, the new reflectors ----------------
    // With RPL even a lane's rows come in consecutive pairs (rowk[e + 1] = rowk[e] + 1 for even e),
    // so a warp writes each column as one contiguous 16-byte-per-lane store.
    {
      double* outb = L.out + cslot * L.cap;
      // (a chained block's outputs are its carry rows, below; its own rows hold only reflectors)
      const int rmax = chained ? 0 : (Rt < L.orows ? Rt : L.orows);
#pragma unroll
      for (int c = 0; c < S8; ++c) {
        if (c >= s) break;
        const int piv = C + c;
        const double dg = diagv[c];
        double* vcol = L.V + r0 + (int64_t)(C + c) * L.ldv;
        double* ocol = outb + (int64_t)c * L.ldo;
#pragma unroll
        for (int e = 0; e < RPL; ++e) {
          const int row = rowk[e], sr = srow[e];
          const double ov = sr < piv ? xr[e][c] : (sr == piv ? dg : 0.0);
          const double vv = sr >= piv ? xr[e][c] : 0.0;
          if constexpr (RPL % 2 == 0) {
            if (e % 2 == 0) {
              const int sr1 = srow[e + 1];
              const double ov1 = sr1 < piv ? xr[e + 1][c] : (sr1 == piv ? dg : 0.0);
              const double vv1 = sr1 >= piv ? xr[e + 1][c] : 0.0;
              if (row + 1 < Rt) {
                st2(vcol + row, vv, vv1);
              } else if (row < Rt) {
                vcol[row] = vv;
              }
              if (L.ovec && row + 1 < rmax) {
                st2(ocol + row, ov, ov1);
              } else {
                if (row < rmax) ocol[row] = ov;
                if (row + 1 < rmax) ocol[row + 1] = ov1;
              }
            }
          } else {
            if (row < rmax) ocol[row] = ov;
            if (row < Rt) vcol[row] = vv;
          }
        }
      }
      if (chained) {
        // chained block: rows [C, C+s) of its output (the N part; rows < C were written panel by
        // panel) from the carry register rows, and the carry parts of the new reflectors (rows
        // [C + c, C + s) of column C + c) into their segments [xs, xs + LS), xs = (C + c) & ~1;
        // warp 0 writes the segments' zero entries
        // (through ctl and a compact loop: the carry rows are the last warp's; an unrolled
        // per-register store loop here cost 2.7 K instructions of instruction cache)
        if (warp == NW - 1) {
#pragma unroll
          for (int e = 0; e < RPL; ++e) {
            const int sr = srow[e];
            if (sr >= C && sr < C + s) {
#pragma unroll
              for (int c = 0; c < S8; ++c) ctl[(sr - C) * S8 + c] = xr[e][c];
            }
          }
          __syncwarp();
#pragma unroll 1
          for (int e = lane; e < s * S8; e += 32) {
            const int i = e / S8, c = e % S8;
            if (c < s) {
              const double v = ctl[e];
              st_l2pol(kslot + C + i + (int64_t)c * kld, i < c ? v : (i == c ? diagv[c] : 0.0), kpol);
              if (i >= c) L.VC[(b * L.cap + C + c) * LS + C + i - ((C + c) & ~1)] = v;
            }
          }
        }
        if (warp == 0)
          for (int e = lane; e < s * LS; e += 32) {
            const int c = e / LS, rr = ((C + c) & ~1) + e % LS;
            if (!(rr >= C + c && rr < C + s)) L.VC[(b * L.cap + C + c) * LS + e % LS] = 0.0;
          }
      }
    }
    }  // stage-1 tail
  }
  WY_TR(9);
#ifdef PQR_WY_TRACE
  if (tr_on)
    for (int i = 0; i < 16; ++i) L.trace[tr_w * 16 + i] = s_tr[tr_w][i];
#endif
#undef WY_TR
}

// Level kernels: NG groups of 16 / NG consumer warps (UW in 16-warp units, as planned by the
// host).  NG = 2 when a CTA gets two or more blocks (one group's tail overlaps the other's
// panels), NG = 1 (16 warps on one block: lower latency per block) for the small tree levels.
template <int UW, int NT, int WM, bool MERGE, int NG, bool CH = false, bool NAR = false>
__global__ void __launch_bounds__(kWyLaunch, 1) k_wy_up(WyLevel L, WyPanels P, int C, int s, int merge, int mtoff) {
  wy_body<kWyWarps / NG, UW * NG, NT, WM, true, MERGE, NG, CH, NAR>(L, P, C, s, 0, 0, merge, mtoff);
}

// stage 2: Y_b = Q_b [coef; 0] (columns < t; columns t..ncol-1 zero)
template <int UW, int NT, int WM, int NG, bool CH = false>
__global__ void __launch_bounds__(kWyLaunch, 1) k_wy_down(WyLevel L, WyPanels P, int Call, int t, int ncol) {
  wy_body<kWyWarps / NG, UW * NG, NT, WM, false, false, NG, CH>(L, P, 0, t, Call, ncol, 0, 0);
}

}  // namespace pqr
