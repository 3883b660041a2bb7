// stream_kernels.cuh — TMA-pipelined CholQR2 passes (§8(a) a1 Gram, a4 update).
//
// One persistent CTA per SM (grid = #SMs), 9 warps:
//   warp 8 (producer, one elected lane) streams 8-row slabs of [Q X] into a ring of
//     NS shared-memory stages with 2-D TMA tensor copies (cp.async.bulk.tensor, SASS
//     UTMALDG): one box of 8 rows x k columns of Q and one of 8 rows x s columns of X
//     per slab; out-of-bounds rows are zero-filled by the TMA unit (so a ragged last
//     slab needs no special path);
//   warps 0..7 (consumers): warp w owns stages w, w+8, ..., w+8(R-1) and the slabs
//     that land in them; it waits on the stage's `full` mbarrier (transaction bytes),
//     computes with fp64 MMAs (mma.sync m8n8k4 .f64 = DMMA.8x8x4) and releases the
//     stage on its `empty` mbarrier.  Owning stages makes every parity wait at most
//     one phase ahead of the barrier.
// NS = 8R stages of (k+s) x 64 B (R = 2-3) keep ~100-200 KB of loads in flight per SM
// (Little's law at ~7 TB/s) without spending registers on it.
//
// A stage line is one column's 8 rows (64 B, no swizzle): the Gram A fragment (8
// columns x 4 row pairs) reads 512 contiguous bytes and the update B fragment (4
// columns x 8 rows) 256 contiguous bytes, both bank-conflict-free.
#pragma once
#include <cuda.h>

#include "cholqr_kernels.cuh"
#include "common.cuh"

namespace pqr {

constexpr int kStreamConsumers = 8;
constexpr int kStreamThreads = (kStreamConsumers + 1) * 32;
constexpr int kSlab = 8;  // rows per stage

PQR_DEV double2 lds2(const double* p) { return *reinterpret_cast<const double2*>(p); }

PQR_DEV void tma_load_2d(void* dst, const CUtensorMap* tm, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
PQR_DEV void tma_prefetch_desc(const CUtensorMap* tm) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(tm)) : "memory");
}

// Stage layout: Q box lines 0..k-1 (region padded to k8 lines), then X box lines;
// line r holds the slab's 8 rows of one column.  Returns &column j of [Q X], row `row`.
PQR_DEV const double* frag_ptr(const double* stage, int j, int k, int k8, int row) {
  const int r = j < k ? j : k8 + (j - k);
  return stage + r * kSlab + row;
}

struct StreamGeom {
  int64_t n;
  int k, sx;      // columns of Q and X
  int k8, x8;     // padded line counts (multiples of 8)
  int NS;         // stages
  int stage_dbl;  // doubles per stage = (k8 + x8) * 8
};

// shared-memory carve-up: [align 1024][NS stages][full NS][empty NS]
struct StreamSmem {
  double* stages;
  uint64_t* full;
  uint64_t* empty;
};
PQR_DEV StreamSmem carve(double* raw, const StreamGeom& g) {
  StreamSmem s;
  const uint32_t base = smem_u32(raw);
  const uint32_t aligned = (base + 1023u) & ~1023u;
  s.stages = raw + (aligned - base) / sizeof(double);
  s.full = reinterpret_cast<uint64_t*>(s.stages + (size_t)g.NS * g.stage_dbl);
  s.empty = s.full + g.NS;
  return s;
}

PQR_DEV void stream_init(const StreamSmem& s, const StreamGeom& g, const CUtensorMap* tmQ, const CUtensorMap* tmX) {
  // padding lines are never written by the TMA: zero every stage once
  for (int e = threadIdx.x; e < g.NS * g.stage_dbl; e += blockDim.x) s.stages[e] = 0.0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < g.NS; ++i) {
      mbar_init(&s.full[i], 1);
      mbar_init(&s.empty[i], 1);
    }
    fence_mbar_init();
    if (g.k > 0) tma_prefetch_desc(tmQ);
    if (g.sx > 0) tma_prefetch_desc(tmX);
  }
  fence_proxy_async_smem();
  __syncthreads();
}

// Producer loop: slab i = blockIdx.x + j*gridDim.x goes to stage j % NS.
PQR_DEV void stream_produce(const StreamSmem& s, const StreamGeom& g, const CUtensorMap* tmQ, const CUtensorMap* tmX) {
  const int64_t nsl = (g.n + kSlab - 1) / kSlab;
  const uint32_t bytes = (uint32_t)(g.k + g.sx) * kSlab * 8u;
  int j = 0;
  for (int64_t sl = blockIdx.x; sl < nsl; sl += gridDim.x, ++j) {
    const int st = j % g.NS;
    mbar_wait(&s.empty[st], ((uint32_t)(j / g.NS) & 1u) ^ 1u);
    mbar_arrive_expect_tx(&s.full[st], bytes);
    double* stage = s.stages + (size_t)st * g.stage_dbl;
    const int row0 = (int)(sl * kSlab);
    if (g.k > 0) tma_load_2d(stage, tmQ, row0, 0, &s.full[st]);
    if (g.sx > 0) tma_load_2d(stage + g.k8 * kSlab, tmX, row0, 0, &s.full[st]);
  }
}

// ----------------------------------------------------------------------------
// a1: W = [Q X]^T X
// ----------------------------------------------------------------------------
struct GramTmaArgs {
  StreamGeom g;                   // sx = s
  double* partials;               // [gridDim.x][m*s]
  double* W; int ldw;
  unsigned int* ticket;
};

// Each consumer warp accumulates all MT column tiles of W over its slabs
// (acc[MTMAX][NT][2]); the 8 warps are summed in smem in fixed order at the end.
template <int MTMAX, int NT>
__global__ void __launch_bounds__(kStreamThreads, 1)
    k_gram_tma(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmX, GramTmaArgs a) {
  extern __shared__ double sm_raw[];
  const StreamGeom& g = a.g;
  const StreamSmem S = carve(sm_raw, g);
  const int k = g.k, s = g.sx, m = k + s, MT = (m + 7) >> 3;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gq = lane >> 2, q = lane & 3;
  stream_init(S, g, &tmQ, &tmX);

  double acc[MTMAX][NT][2];
#pragma unroll
  for (int i = 0; i < MTMAX; ++i)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) acc[i][nt][0] = acc[i][nt][1] = 0.0;

  const int64_t nsl = (g.n + kSlab - 1) / kSlab;
  if (warp == kStreamConsumers) {
    if (lane == 0) stream_produce(S, g, &tmQ, &tmX);
  } else {
    int j = warp;
    for (int64_t sl = blockIdx.x + (int64_t)warp * gridDim.x; sl < nsl; sl += (int64_t)kStreamConsumers * gridDim.x,
                 j += kStreamConsumers) {
      const int st = j % g.NS;  // == warp + 8 * ((j / 8) % R): a stage this warp owns
      mbar_wait(&S.full[st], (uint32_t)(j / g.NS) & 1u);
      const double* stage = S.stages + (size_t)st * g.stage_dbl;
      double2 bv[NT];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int col = 8 * nt + gq;
        bv[nt] = col < s ? lds2(frag_ptr(stage, k + col, k, g.k8, 2 * q)) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int mt = 0; mt < MTMAX; ++mt) {
        if (mt < MT) {
          const int jj = 8 * mt + gq;
          const double2 av = jj < m ? lds2(frag_ptr(stage, jj, k, g.k8, 2 * q)) : make_double2(0.0, 0.0);
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            dmma884(acc[mt][nt][0], acc[mt][nt][1], av.x, bv[nt].x);
            dmma884(acc[mt][nt][0], acc[mt][nt][1], av.y, bv[nt].y);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.empty[st]);
    }
  }
  __syncthreads();  // pipeline drained: stage memory is free for the reduction
  // ---- CTA reduction over the 8 consumer warps (fixed order) ----
  double* red = S.stages;  // [8][MT][NT][32][2]
  const int per_warp = MT * NT * 64;
  if (warp < kStreamConsumers) {
#pragma unroll
    for (int mt = 0; mt < MTMAX; ++mt)
      if (mt < MT)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          red[warp * per_warp + ((mt * NT + nt) * 32 + lane) * 2 + 0] = acc[mt][nt][0];
          red[warp * per_warp + ((mt * NT + nt) * 32 + lane) * 2 + 1] = acc[mt][nt][1];
        }
  }
  __syncthreads();
  double* part = a.partials + (size_t)blockIdx.x * m * s;
  for (int e = tid; e < per_warp; e += blockDim.x) {
    const int v = e & 1, l = (e >> 1) & 31, rest = e >> 6;  // rest = mt*NT + nt
    const int nt = rest % NT, mt = rest / NT;
    const int jj = 8 * mt + (l >> 2), c = 8 * nt + 2 * (l & 3) + v;
    if (jj < m && c < s) {
      double sum = 0.0;
      for (int w = 0; w < kStreamConsumers; ++w) sum += red[w * per_warp + e];
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
  for (int e = tid; e < ms; e += blockDim.x) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int b = 0;
    for (; b + 4 <= nb; b += 4) {
      s0 += __ldcg(a.partials + (size_t)(b + 0) * ms + e);
      s1 += __ldcg(a.partials + (size_t)(b + 1) * ms + e);
      s2 += __ldcg(a.partials + (size_t)(b + 2) * ms + e);
      s3 += __ldcg(a.partials + (size_t)(b + 3) * ms + e);
    }
    for (; b < nb; ++b) s0 += __ldcg(a.partials + (size_t)b * ms + e);
    const int jj = e % m, c = e / m;
    a.W[jj + (int64_t)c * a.ldw] = (s0 + s1) + (s2 + s3);
  }
  if (tid == 0) *a.ticket = 0u;
}

// ----------------------------------------------------------------------------
// a4: U = [Q X] M   ("U = XN^{-1} - QPN^{-1}")
// ----------------------------------------------------------------------------
struct UpdTmaArgs {
  StreamGeom g;
  int sout;
  const double* M; int ldm;       // (k+sx) x sout
  const int* t_dev;
  double* U; int64_t ldu;
  double* U2; int64_t ldu2;
};

// U^T = M^T [Q X]^T as m8n8k4 MMAs: M-index = output column c, N-index = slab row,
// K = column j of [Q X].  Lane l reads row l>>2 of column 4kk+(l&3) (B fragment) and
// M[4kk+(l&3)][l>>2] (A fragment); the D fragment gives it rows 2(l&3), 2(l&3)+1 of
// output column l>>2.  Two accumulator chains (even / odd kk) halve the DMMA
// dependency chain.
template <int NT>
PQR_DEV void upd_store_pair(const UpdTmaArgs& a, const double (&d)[NT][2], int64_t row, int gq, int t) {
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const int c = 8 * nt + gq;
    if (c >= a.sout) continue;
    const bool valid = c < t;
    const double v0 = valid ? d[nt][0] : 0.0, v1 = valid ? d[nt][1] : 0.0;
    double* up = a.U + (int64_t)c * a.ldu + row;
    if (row + 1 < a.g.n) st2(up, v0, v1);
    else if (row < a.g.n) up[0] = v0;
    if (a.U2 && valid) {
      double* u2 = a.U2 + (int64_t)c * a.ldu2 + row;
      if (row + 1 < a.g.n) st2(u2, v0, v1);
      else if (row < a.g.n) u2[0] = v0;
    }
  }
}

template <int NT>
__global__ void __launch_bounds__(kStreamThreads, 1)
    k_update_tma(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmX, UpdTmaArgs a) {
  extern __shared__ double sm_raw[];
  const StreamGeom& g = a.g;
  const StreamSmem S = carve(sm_raw, g);
  const int k = g.k, m = k + g.sx;
  const int KS = ((m + 7) >> 3) * 2, mpad = KS * 4;  // even number of k-steps
  double* sM = reinterpret_cast<double*>(S.empty + g.NS);  // [NT][mpad][8]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gq = lane >> 2, q = lane & 3;
  for (int e = tid; e < NT * mpad * 8; e += blockDim.x) {
    const int nt = e / (mpad * 8), rem = e % (mpad * 8);
    const int j = rem >> 3, c = 8 * nt + (rem & 7);
    sM[e] = (j < m && c < a.sout) ? a.M[j + (int64_t)c * a.ldm] : 0.0;
  }
  stream_init(S, g, &tmQ, &tmX);
  const int t = a.t_dev ? *a.t_dev : a.sout;
  const int64_t nsl = (g.n + kSlab - 1) / kSlab;

  if (warp == kStreamConsumers) {
    if (lane == 0) stream_produce(S, g, &tmQ, &tmX);
    return;
  }
  int j = warp;
  for (int64_t sl = blockIdx.x + (int64_t)warp * gridDim.x; sl < nsl; sl += (int64_t)kStreamConsumers * gridDim.x,
               j += kStreamConsumers) {
    const int st = j % g.NS;
    mbar_wait(&S.full[st], (uint32_t)(j / g.NS) & 1u);
    const double* stage = S.stages + (size_t)st * g.stage_dbl;
    double d[2][NT][2];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) d[h][nt][0] = d[h][nt][1] = 0.0;
#pragma unroll 4
    for (int kk = 0; kk < KS; kk += 2) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int jj = 4 * (kk + h) + q;
        const double bv = jj < m ? *frag_ptr(stage, jj, k, g.k8, gq) : 0.0;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const double mv = sM[(nt * mpad + jj) * 8 + gq];
          dmma884(d[h][nt][0], d[h][nt][1], mv, bv);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&S.empty[st]);
    double r[NT][2];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      r[nt][0] = d[0][nt][0] + d[1][nt][0];
      r[nt][1] = d[0][nt][1] + d[1][nt][1];
    }
    upd_store_pair<NT>(a, r, sl * kSlab + 2 * q, gq, t);
  }
}

}  // namespace pqr
