// tsqr_wy.cuh — TreeTSPQR level kernels with blocked (compact-WY) reflector panels and
// fp64 MMAs (§4.1 Alg. 9 with Householder local/reduction subalgorithms).
//
// A level block holds R <= 256*UW rows; warp w (of 16) owns UW units of 16
// rows, lane (g = l>>2, q = l&3) keeping rows 16u+4q+{0..3} of columns 8nt+g in
// registers (the D-fragment layout of the update MMA below).  The block's reflectors
// are grouped in panels (the reflectors created by one call, or one LOR-build chunk):
// H_a ... H_b = I - V T V^T with T^{-1} = I/2 + striu(V^T V) (unit-norm v, Eq. (hh)).
//
//   stage 1 (Q_b^T X):  for each panel in order   Z = V^T X, Z' = T^T Z, X -= V Z'
//   stage 2 (Q_b Y):    for each panel reversed    Z = V^T Y, Z' = T Z,   Y -= V Z'
//
// Z = V^T X is an m8n8k4 DMMA Gram (K = rows: lane q supplies rows 4q..4q+3 as four
// k-steps); X -= V Z' is X^T -= Z'^T V^T (K = panel columns, N = rows, the even/odd
// row trick of the update kernel).  Panels are double-buffered in shared memory with
// cp.async; the panel stride RP = 10 (mod 16) doubles makes both fragment patterns
// bank-conflict-free (the update k-steps take columns 2q+kk so the four columns of an
// LDS.128 phase land in four distinct 32-byte bank groups).
//
// After the committed panels, stage 1 factors rows C..R-1 of the s new columns with
// Householder reflectors (Alg. 6 lines 2-9; never deflating, reading R4), stores them
// (rows < pivot zeroed) and the panel's T, and writes [P_b; N_b] to the parent slot.
#pragma once
#include "common.cuh"

namespace pqr {

constexpr int kWyWarps = 16;
constexpr int kWyThreads = 32 * kWyWarps;
constexpr int kWyRowsPerUW = 16 * kWyWarps;  // block rows covered per unit-per-warp
constexpr int kWyMaxW = 16;  // widest panel

struct WyLevel {
  int64_t q, rem2;      // block b: q + 2*(b < rem2) rows starting at b*q + 2*min(b, rem2) (even);
  int odd_last;         // ... the last block has one more row when the level's row count is odd
  int nblocks;
  const double* X; int64_t ldx;     // stage-1 input (level rows)
  double* V; int64_t ldv;           // reflectors (level rows); column j = reflector j
  double* T; int64_t tstride;       // block b's T area at T + b*tstride; panel at +16*start
  double* out; int64_t ldo;         // stage-1 output: block b -> rows b*cap ...
  const double* cin; int64_t ldci;  // stage-2 coefficients: block b -> rows b*cap ...
  double* Y; int64_t ldy;           // stage-2 output (level rows)
  int cap;
  int RP;                           // smem panel stride (>= max block rows, = 10 mod 16)
  int wmax;                         // widest panel (<= 16) -> smem panel buffer width
  int nbuf;                         // panel buffers (2 or 3)
};

struct WyPanels {
  const int2* pan;  // (start, width) per panel, device
  int np;           // panels to apply
};

PQR_DEV int64_t wy_start(const WyLevel& L, int64_t b) { return b * L.q + 2 * (b < L.rem2 ? b : L.rem2); }
PQR_DEV int wy_rows(const WyLevel& L, int64_t b) {
  return (int)(L.q + (b < L.rem2 ? 2 : 0) + (b == L.nblocks - 1 ? L.odd_last : 0));
}

// column of the update k-step kk for lane quarter q (conflict-free pattern, see header)
PQR_DEV int wy_col(int kk, int q) { return 8 * (kk >> 1) + 2 * q + (kk & 1); }

// Stage panel (start, w) of this block into buf (RP x w8 col-major); rows R..kWyRowsPerUW*UW-1
// and columns w..w8-1 are zero-filled (they meet zero rows / zero coefficients in the MMAs).
template <int UW>
PQR_DEV void wy_load_panel(double* buf, const WyLevel& L, int64_t r0, int R, int start, int w, int RP) {
  constexpr int pairs = kWyRowsPerUW * UW / 2;
  const int w8 = (w + 7) & ~7;
  for (int e = threadIdx.x; e < w8 * pairs; e += kWyThreads) {
    const int j = e / pairs, p = e - j * pairs;
    const int row = 2 * p;
    const double* src = L.V + (int64_t)(start + j) * L.ldv + r0 + row;
    const int bytes = (j < w && row < R) ? (row + 1 < R ? 16 : 8) : 0;
    cp_async16(buf + j * RP + row, bytes ? (const void*)src : (const void*)L.V, bytes);
  }
}

// Block-wide: Z (w8 x s8, smem, col-major ld 16) = sum over warps of the D fragments
// acc[mt][nt][2]; red is kWyWarps*256 doubles.  Ends with a __syncthreads.
template <int NT>
PQR_DEV void wy_reduce_Z(double (&acc)[2][NT][2], int mtn, double* red, double* Z, int wm) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, q = lane & 3;
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int i = 8 * mt + g, c = 8 * nt + 2 * q + v;
        if (i < wm && c < wm) red[warp * wm * wm + i + wm * c] = (mt < mtn) ? acc[mt][nt][v] : 0.0;
      }
  __syncthreads();
  for (int e = threadIdx.x; e < 256; e += kWyThreads) {
    const int i = e & 15, c = e >> 4;
    double a = 0.0;
    if (i < wm && c < wm) {
#pragma unroll
      for (int w = 0; w < kWyWarps; ++w) a += red[w * wm * wm + i + wm * c];
    }
    Z[e] = a;
  }
  __syncthreads();
}

// apply one panel (in smem `vb`, width w) to the register block x:
//   x <- x - V (Tp Z),  Z = V^T x,  Tp = T^T (stage 1) or T (stage 2);  Tg in smem (ld w)
template <int UW, int NT>
PQR_DEV void wy_apply_panel(double (&x)[UW][NT][4], const double* vb, const double* Tg, int w, bool transT,
                            int RP, double* red, double* Zp, int wm) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, q = lane & 3;
  const int mtn = (w + 7) >> 3;
  // ---- Z = V^T x (per-warp partials; two accumulator chains over alternate units) ----
  double acc[2][2][NT][2];
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) acc[h][mt][nt][0] = acc[h][mt][nt][1] = 0.0;
#pragma unroll
  for (int mt = 0; mt < 2; ++mt) {
    if (mt < mtn) {
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
    }
  }
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int i = 8 * mt + g, c = 8 * nt + 2 * q + v;
        if (i < wm && c < wm) red[warp * wm * wm + i + wm * c] = (mt < mtn) ? acc[0][mt][nt][v] + acc[1][mt][nt][v] : 0.0;
      }
  __syncthreads();
  // ---- Z = sum over warps of red (fixed order), then Z' = T^T Z (stage 1) or T Z (stage 2) ----
  const int E = wm * wm;
  double* Zs = red + kWyWarps * E;  // E doubles after the per-warp partials
  if (tid < E) {
    double z = 0.0;
#pragma unroll
    for (int ww = 0; ww < kWyWarps; ++ww) z += red[ww * E + tid];
    Zs[tid] = z;
  }
  __syncthreads();
  if (tid < 256) {
    const int i = tid & 15, c = tid >> 4;
    double a = 0.0;
    if (i < w && c < wm) {
      if (transT) {
        for (int l = 0; l <= i; ++l) a += Tg[l + i * w] * Zs[l + wm * c];
      } else {
        for (int l = i; l < w; ++l) a += Tg[i + l * w] * Zs[l + wm * c];
      }
    }
    Zp[tid] = a;
  }
  __syncthreads();
  // ---- x^T -= Z'^T V^T ----
  const int kks = 2 * mtn;
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    if (kk < kks) {
      const int j = wy_col(kk, q);
      double am[NT];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) am[nt] = -Zp[j + 16 * (8 * nt + g)];
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
}

// Apply the first np panels, forward (stage 1, H_0 first, T^T) or reversed (stage 2, T).
// Panels (and each panel's T, w x w) stream through L.nbuf shared-memory buffers: one
// thread issues one cp.async.bulk per panel column (R rows, contiguous in HBM: 8 KB at
// R = 1024, long enough for the bulk-copy engine) plus one for T, completing on the
// buffer's mbarrier; while panel i is applied, panels i+1 .. i+nbuf-1 are in flight.
// Rows R..(256*UW)-1 and columns w..w8-1 of every buffer are zeroed once (never copied).
template <int UW, int NT>
PQR_DEV void wy_apply_panels(double (&x)[UW][NT][4], const WyLevel& L, const WyPanels& P, int64_t b, int64_t r0,
                             int R, bool forward, double* vbuf, double* red, double* Zp, int2* pans,
                             uint64_t* full) {
  const int np = P.np;
  if (np == 0) return;
  const int RP = L.RP, nbuf = L.nbuf, wm = L.wmax;
  const int bstride = RP * wm + 256;  // panel + its T
  const int Reven = R & ~1;           // rows moved by the bulk copies
  for (int i = threadIdx.x; i < np; i += kWyThreads) pans[i] = P.pan[i];
  // zero the never-copied parts: rows >= Reven of every column (row R-1 of an odd block is
  // loaded per element below), all rows of columns >= w are zeroed per panel if w < w8
  for (int e = threadIdx.x; e < nbuf * wm * (RP - Reven); e += kWyThreads) {
    const int bb = e / (wm * (RP - Reven)), rem = e % (wm * (RP - Reven));
    const int j = rem / (RP - Reven), row = Reven + rem % (RP - Reven);
    vbuf[bb * bstride + j * RP + row] = 0.0;
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < nbuf; ++i) mbar_init(&full[i], 1);
    fence_mbar_init();
  }
  fence_proxy_async_smem();
  const double* Tb = L.T + b * L.tstride;
  __syncthreads();
  auto pidx = [&](int i) { return forward ? i : np - 1 - i; };
  auto issue = [&](int i) {  // thread 0 only
    if (i < np) {
      const int2 pn = pans[pidx(i)];
      double* buf = vbuf + (i % nbuf) * bstride;
      uint64_t* bar = &full[i % nbuf];
      const uint32_t tbytes = (uint32_t)((pn.y * pn.y + 1) & ~1) * 8u;
      mbar_arrive_expect_tx(bar, (uint32_t)pn.y * Reven * 8u + tbytes);
      for (int j = 0; j < pn.y; ++j)
        bulk_g2s(buf + j * RP, L.V + (int64_t)(pn.x + j) * L.ldv + r0, (uint32_t)Reven * 8u, bar);
      bulk_g2s(buf + RP * wm, Tb + 16 * pn.x, tbytes, bar);
    }
  };
  if (threadIdx.x == 0)
    for (int i = 0; i < nbuf - 1; ++i) issue(i);
  for (int i = 0; i < np; ++i) {
    const int2 pc = pans[pidx(i)];
    double* buf = vbuf + (i % nbuf) * bstride;
    // per-element pieces: the odd last row, and zero columns w..w8-1 (stale from a wider panel)
    if (R & 1)
      for (int j = threadIdx.x; j < pc.y; j += kWyThreads) buf[j * RP + R - 1] = L.V[(int64_t)(pc.x + j) * L.ldv + r0 + R - 1];
    const int w8 = (pc.y + 7) & ~7;
    for (int e = threadIdx.x; e < (w8 - pc.y) * Reven; e += kWyThreads) buf[(pc.y + e / Reven) * RP + e % Reven] = 0.0;
    fence_proxy_async_smem();  // order these generic writes before later bulk copies into the buffer
    mbar_wait(&full[i % nbuf], (uint32_t)(i / nbuf) & 1u);
    __syncthreads();          // panel i complete and visible; every warp is done with panel i-1
    if (threadIdx.x == 0) issue(i + nbuf - 1);  // refill the buffer panel i-1 used
    wy_apply_panel<UW, NT>(x, buf, buf + RP * wm, pc.y, forward, RP, red, Zp, wm);
  }
  __syncthreads();
}

// ----------------------------------------------------------------------------
// stage 1
// ----------------------------------------------------------------------------
template <int UW, int NT>
__global__ void __launch_bounds__(kWyThreads, 1) k_wy_up(WyLevel L, WyPanels P, int C, int s) {
  extern __shared__ __align__(16) double sm[];
  const int RP = L.RP;
  double* vbuf = sm;                                   // nbuf x (RP x wmax + 256)
  double* red = vbuf + L.nbuf * (RP * L.wmax + 256);   // (kWyWarps + 1) x wmax^2
  double* Z = red + (kWyWarps + 1) * L.wmax * L.wmax;  // 256
  double* Zp = Z + 256;                                // 256
  double* bc = Zp + 256;                               // 64 scratch
  int2* pans = reinterpret_cast<int2*>(bc + 64);       // panel list (cap + 1)
  uint64_t* full = reinterpret_cast<uint64_t*>(pans + ((L.cap + 2) & ~1));  // nbuf mbarriers
  double* Vn = vbuf;                                   // RP x s8: the new reflectors (aliases the
                                                       // panel buffers, free after the panels)
  const int64_t b = blockIdx.x;
  const int64_t r0 = wy_start(L, b);
  const int R = wy_rows(L, b);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, q = lane & 3;

  double x[UW][NT][4];
#pragma unroll
  for (int u = 0; u < UW; ++u)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int row = 16 * (warp * UW + u) + 4 * q + i, c = 8 * nt + g;
        x[u][nt][i] = (row < R && c < s) ? L.X[r0 + row + (int64_t)c * L.ldx] : 0.0;
      }
  wy_apply_panels<UW, NT>(x, L, P, b, r0, R, true, vbuf, red, Zp, pans, full);

  // ---- Householder QR of rows C..R-1 of the s new columns (Alg. 6 lines 2-9) ----
  // The block is moved from the MMA register layout to shared memory (xs, column-major),
  // where thread t owns rows t, t+512, ...: every thread takes part in each column's
  // reductions.  Two block barriers per column: red1 carries column c's norm partials
  // (written right after column c's last update), red2 the dot products of v_c with the
  // later columns; the buffers alternate, so no third barrier is needed.
  const int s8 = (s + 7) & ~7;
  double* xs = vbuf + RP * s8;   // RP x s8 (Vn = vbuf holds the new reflectors)
  __syncthreads();
  for (int e = tid; e < RP * s8; e += kWyThreads) Vn[e] = 0.0;
#pragma unroll
  for (int u = 0; u < UW; ++u)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int row = 16 * (warp * UW + u) + 4 * q + i, c = 8 * nt + g;
        if (c < s8) xs[c * RP + row] = x[u][nt][i];
      }
  constexpr int RPT = (kWyRowsPerUW * UW + kWyThreads - 1) / kWyThreads;  // rows per thread
  double* red1 = red;          // kWyWarps
  double* red2 = red + 64;     // kWyWarps x 16
  auto norm_partial = [&](int c) {
    const int r = C + c;
    double part = 0.0;
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
      const int row = tid + j * kWyThreads;
      if (row >= r && row < R) part += xs[c * RP + row] * xs[c * RP + row];
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if (lane == 0) red1[warp] = part;
  };
  __syncthreads();
  if (s > 0) norm_partial(0);
  for (int c = 0; c < s; ++c) {
    const int r = C + c;
    __syncthreads();  // S1: norm partials of column c in red1; column c final above row r
    double lam2 = 0.0;
#pragma unroll
    for (int w = 0; w < kWyWarps; ++w) lam2 += red1[w];
    const double lam = sqrt(lam2);
    const double u0 = r < R ? xs[c * RP + r] : 0.0;
    const double sigma = (u0 >= 0.0) ? -1.0 : 1.0;  // sigma = -sgn(u0), sgn(0) = +1
    const double diag = sigma * lam;
    const double nv2 = 2.0 * lam * (lam + fabs(u0));
    const double inv = nv2 > 0.0 ? rsqrt(nv2) : 0.0;  // identity reflector if lam == 0 (R4)
    double v[RPT];
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
      const int row = tid + j * kWyThreads;
      const double xv = row < R ? xs[c * RP + row] : 0.0;
      v[j] = (row > r && row < R) ? xv * inv : (row == r ? (xv - diag) * inv : 0.0);
    }
    // dot products v . x[:, c'] for c' > c (reduced over the warp, then over warps)
    for (int cc = c + 1; cc < s; ++cc) {
      double a = 0.0;
#pragma unroll
      for (int j = 0; j < RPT; ++j) {
        const int row = tid + j * kWyThreads;
        if (row < R) a += v[j] * xs[cc * RP + row];
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
      if (lane == 0) red2[warp * 16 + cc] = a;
    }
    __syncthreads();  // S2: dots in red2; every thread has read u0 and red1
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
      const int row = tid + j * kWyThreads;
      if (row < R) {
        Vn[c * RP + row] = v[j];
        if (row >= r) xs[c * RP + row] = (row == r) ? diag : 0.0;
      }
    }
    for (int cc = c + 1; cc < s; ++cc) {
      double d = 0.0;
#pragma unroll
      for (int w = 0; w < kWyWarps; ++w) d += red2[w * 16 + cc];
      const double f = 2.0 * d;
#pragma unroll
      for (int j = 0; j < RPT; ++j) {
        const int row = tid + j * kWyThreads;
        if (row < R) xs[cc * RP + row] -= f * v[j];
      }
    }
    if (c + 1 < s) norm_partial(c + 1);
  }
  __syncthreads();

  // ---- outputs: [P_b; N_b] = rows 0..C+s-1, the new reflectors, the new panel's T ----
  double* outb = L.out + b * L.cap;
  for (int e = tid; e < s * (C + s); e += kWyThreads) {
    const int c = e / (C + s), row = e - c * (C + s);
    if (row < R) outb[row + (int64_t)c * L.ldo] = xs[c * RP + row];
  }
  for (int e = tid; e < s * R; e += kWyThreads) {
    const int c = e / R, row = e - c * R;
    L.V[r0 + row + (int64_t)(C + c) * L.ldv] = Vn[c * RP + row];
  }
  // V^T V of the new panel: Gram MMA from smem Vn (same fragment pattern as Z = V^T x)
  {
    double acc[2][2][2];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
    const int mtn = (s + 7) >> 3;
#pragma unroll
    for (int u = 0; u < UW; ++u) {
      const int row = 16 * (warp * UW + u) + 4 * q;
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        if (nt < mtn) {
          const double2 b01 = *reinterpret_cast<const double2*>(Vn + (8 * nt + g) * RP + row);
          const double2 b23 = *reinterpret_cast<const double2*>(Vn + (8 * nt + g) * RP + row + 2);
#pragma unroll
          for (int mt = 0; mt < 2; ++mt) {
            if (mt < mtn) {
              const double2 a01 = *reinterpret_cast<const double2*>(Vn + (8 * mt + g) * RP + row);
              const double2 a23 = *reinterpret_cast<const double2*>(Vn + (8 * mt + g) * RP + row + 2);
              dmma884(acc[mt][nt][0], acc[mt][nt][1], a01.x, b01.x);
              dmma884(acc[mt][nt][0], acc[mt][nt][1], a01.y, b01.y);
              dmma884(acc[mt][nt][0], acc[mt][nt][1], a23.x, b23.x);
              dmma884(acc[mt][nt][0], acc[mt][nt][1], a23.y, b23.y);
            }
          }
        }
      }
    }
    wy_reduce_Z<2>(acc, mtn, red, Z, L.wmax);  // Z = V^T V (16 x 16, ld 16)
    // T^{-1} = I/2 + striu(V^T V);  T = its inverse (upper triangular), column c by lane c
    double* Tn = L.T + b * L.tstride + 16 * C;
    if (tid < s) {
      const int c = tid;
      double col[kWyMaxW];
#pragma unroll
      for (int i = 0; i < kWyMaxW; ++i) col[i] = 0.0;
      col[c] = 2.0;  // 1 / (1/2)
      for (int i = c - 1; i >= 0; --i) {
        double a = 0.0;
        for (int l = i + 1; l <= c; ++l) a += Z[i + 16 * l] * col[l];
        col[i] = -a * 2.0;
      }
      for (int i = 0; i < s; ++i) Tn[i + c * s] = i <= c ? col[i] : 0.0;
    }
  }
}

// ----------------------------------------------------------------------------
// stage 2: Y_b = Q_b [coef; 0]
// ----------------------------------------------------------------------------
template <int UW, int NT>
__global__ void __launch_bounds__(kWyThreads, 1) k_wy_down(WyLevel L, WyPanels P, int Call, int t, int ncol) {
  extern __shared__ __align__(16) double sm[];
  const int RP = L.RP;
  double* vbuf = sm;
  double* red = vbuf + L.nbuf * (RP * L.wmax + 256);
  double* Z = red + (kWyWarps + 1) * L.wmax * L.wmax;
  double* Zp = Z + 256;
  int2* pans = reinterpret_cast<int2*>(Zp + 256 + 64);
  uint64_t* full = reinterpret_cast<uint64_t*>(pans + ((L.cap + 2) & ~1));
  const int64_t b = blockIdx.x;
  const int64_t r0 = wy_start(L, b);
  const int R = wy_rows(L, b);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, q = lane & 3;
  const double* cb = L.cin + b * L.cap;
  double y[UW][NT][4];
#pragma unroll
  for (int u = 0; u < UW; ++u)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int row = 16 * (warp * UW + u) + 4 * q + i, c = 8 * nt + g;
        y[u][nt][i] = (row < Call && row < R && c < t) ? cb[row + (int64_t)c * L.ldci] : 0.0;
      }
  wy_apply_panels<UW, NT>(y, L, P, b, r0, R, false, vbuf, red, Zp, pans, full);
#pragma unroll
  for (int u = 0; u < UW; ++u)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int row = 16 * (warp * UW + u) + 4 * q + i, c = 8 * nt + g;
        if (row < R && c < ncol) L.Y[r0 + row + (int64_t)c * L.ldy] = c < t ? y[u][nt][i] : 0.0;
      }
}

}  // namespace pqr
