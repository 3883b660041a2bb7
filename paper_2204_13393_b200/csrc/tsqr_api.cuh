// tsqr_api.cuh — orchestration of the TSQR variant (TreeTSPQR, §4.1 Alg. 9),
// included by pqr_api.cu inside its anonymous namespace.
//
// Levels (kernels in tsqr_wy.cuh): leaves (level 0) partition the GPU's n_local rows
// into p0 blocks of ~n_b rows (even starts); each node level stacks `arity` children's
// top-cap coordinates (R = arity*cap rows per node); the level with one node is the GPU
// root.  With nranks > 1 the roots' (C+s) x s outputs are all-gathered and the cross-GPU
// levels — the same arity-bounded tree over the nranks roots, replicated on every GPU —
// reduce them: the "different algorithm at the cross-GPU level" slot of the paper's
// framework is this replicated stateful tree (§8(e)).  Reflectors are kept in
// panels (one per call / per LOR-build chunk) with their compact-WY T factors.
namespace {

struct TsqrLv {
  int64_t q = 0, rem2 = 0;
  int odd_last = 0, nblocks = 0;
  int64_t rows = 0;          // leading dimension of this level's V / in / dn buffers
  int UW = 0, RP = 0;
  double* V = nullptr;
  int64_t ldv = 0;
  double* T = nullptr;       // nblocks x tstride
  int64_t tstride = 0;
  double* in = nullptr;      // stage-1 input (node levels / cross level)
  double* dn = nullptr;      // stage-2 output (node levels / cross level)
  bool owns_v = true;
  bool chained = false;      // the leaf level with FlatTSPQR chains
};

struct TsqrState {
  int nb = 0, cap = 0, C = 0, nlev = 0, arity = 8, wmax = 8;
  std::vector<TsqrLv> lv;    // [0] leaves, [1..nlev] nodes
  std::vector<TsqrLv> xlv;   // cross-GPU levels ([0] stacks the nranks GPU roots), replicated
  std::vector<int4> panels;  // committed panels (start, width, T offset, merged)
  int4* d_pan = nullptr;     // device copy (+ one uncommitted slot)
  int4* d_panm = nullptr;    // down-sweep list of a merging call
  std::vector<int4> pan_mirror, panm_mirror;  // host copies of d_pan / d_panm (copy only on change:
                                              // a repeated call enqueues no host-to-device copy, so
                                              // it can be captured in a CUDA graph)
  int merge = 0, mtoff = 0;  // the last call merged its panel into the previous one
  double* in_top = nullptr;  // cap x wmax: GPU root stage-1 output (ld cap)
  double* xraw = nullptr;    // nranks * cap * wmax allgather receive (compact (C+s) x s blocks)
  double* Btop = nullptr;    // cap x wmax top coefficients of X (ld cap)
  double* Ut = nullptr;      // cap x wmax top coefficients of U (ld cap)
  double* Rt = nullptr;      // cap x cap explicit top basis (ld cap), zero-init
  double* coef = nullptr;    // cap x 16 scratch for basis_apply
  // FlatTSPQR leaf chains (§4.2 Alg. 10; WyLevel::nchain): nchain chains of leaf blocks,
  // chain c = blocks c, c + nchain, ...; 0 = every leaf block hands its block to the tree
  int nchain = 0;
  double* VC = nullptr;      // carry-area reflector segments (WyLevel::VC): nblocks x cap x (wmax + 2)
};

// reduction = PIP+ above the GPU tree (pqr.h PQR_REDUCTION_PIP2): no cross-GPU Householder levels
bool pip2(const Ctx* h) { return h->cfg.reduction == PQR_REDUCTION_PIP2; }
// local = PIP+ (pqr.h PQR_LOCAL_PIP2): an explicit, locally orthonormal basis per GPU (h->basis)
// and no on-GPU Householder tree
bool lpip(const Ctx* h) { return h->cfg.local == PQR_LOCAL_PIP2; }

// units of 16 rows per warp: even (the stage-1 tail gives every lane UW/2 whole rows)
int uw_for(int64_t rows) {
  const int uw = (int)((rows + kWyRowsPerUW - 1) / kWyRowsPerUW);
  return uw + (uw & 1);
}
int rp_for(int UW) { return kWyRowsPerUW * UW + 10; }  // >= rows + 1, = 10 (mod 16)
// level kernels may use the whole 227 KB of dynamic shared memory per CTA
constexpr size_t kWySmemBudget = 232448;
// kernels with NG groups of 16 / NG warps differ in scratch
size_t wy_smem(int RP, int wmax, int cap, int nbuf, int NG) {
  return wy_smem_bytes(RP, wmax, cap, nbuf, kWyWarps / NG, NG);
}
int nbuf_for(int RP, int wmax, int cap, int NG) {
  for (int nb = 4; nb > 2; --nb)
    if (wy_smem(RP, wmax, cap, nb, NG) <= kWySmemBudget) return nb;
  return 2;
}
// two groups when some CTA gets two or more blocks and a group's registers hold its rows
// (UW <= 4 in 16-warp units, i.e. blocks of <= 1024 rows); PQR_WY_GROUPS=1|2 forces
int groups_for(int64_t nrun, int sms, int UW) {
  static const int env = getenv("PQR_WY_GROUPS") ? atoi(getenv("PQR_WY_GROUPS")) : 0;
  if (env == 1 || env == 2) return env;
  return nrun > sms && UW <= 4 ? 2 : 1;
}

template <int UW, int NT, int WM, int NG>
cudaError_t wy_up_g(const WyLevel& L, const WyPanels& P, int C, int s, int merge, int mtoff, int grid, size_t smem,
                    cudaStream_t st) {
  if (L.nchain > 0) {  // chained leaf level: two groups (UW <= 4) by construction
    if constexpr (NG == 2 && UW <= 4) {
      if constexpr (NT == 1 && WM == 8) {
        if (merge) {
          auto f = k_wy_up<UW, NT, WM, true, NG, true>;
          ensure_smem(f, smem);
          f<<<grid, kWyLaunch, smem, st>>>(L, P, C, s, merge, mtoff);
          return cudaGetLastError();
        }
      }
      auto f = k_wy_up<UW, NT, WM, false, NG, true>;
      ensure_smem(f, smem);
      f<<<grid, kWyLaunch, smem, st>>>(L, P, C, s, 0, 0);
      return cudaGetLastError();
    }
    return cudaErrorNotSupported;
  }
  if constexpr (NT == 1 && WM == 8) {  // panel merges only pair 4-wide panels (s = 4)
    if (merge) {
      auto f = k_wy_up<UW, NT, WM, true, NG, false, true>;
      ensure_smem(f, smem);
      f<<<grid, kWyLaunch, smem, st>>>(L, P, C, s, merge, mtoff);
      return cudaGetLastError();
    }
    if (s <= 4) {  // narrow tail (4 register columns per row)
      auto f = k_wy_up<UW, NT, WM, false, NG, false, true>;
      ensure_smem(f, smem);
      f<<<grid, kWyLaunch, smem, st>>>(L, P, C, s, 0, 0);
      return cudaGetLastError();
    }
  }
  auto f = k_wy_up<UW, NT, WM, false, NG>;
  ensure_smem(f, smem);
  f<<<grid, kWyLaunch, smem, st>>>(L, P, C, s, 0, 0);
  return cudaGetLastError();
}
template <int UW, int NT, int WM>
cudaError_t wy_up_t(const WyLevel& L, const WyPanels& P, int C, int s, int merge, int mtoff, int grid, size_t smem,
                    cudaStream_t st, int NG) {
  return NG == 2 ? wy_up_g<UW, NT, WM, 2>(L, P, C, s, merge, mtoff, grid, smem, st)
                 : wy_up_g<UW, NT, WM, 1>(L, P, C, s, merge, mtoff, grid, smem, st);
}
template <int UW, int NT, int WM, int NG>
cudaError_t wy_down_g(const WyLevel& L, const WyPanels& P, int Call, int t, int ncol, int grid, size_t smem,
                      cudaStream_t st) {
  if (L.nchain > 0) {  // chained leaf level
    if constexpr (NG == 2 && UW <= 4) {
      auto f = k_wy_down<UW, NT, WM, NG, true>;
      ensure_smem(f, smem);
      f<<<grid, kWyLaunch, smem, st>>>(L, P, Call, t, ncol);
      return cudaGetLastError();
    }
    return cudaErrorNotSupported;
  }
  auto f = k_wy_down<UW, NT, WM, NG>;
  ensure_smem(f, smem);
  f<<<grid, kWyLaunch, smem, st>>>(L, P, Call, t, ncol);
  return cudaGetLastError();
}
template <int UW, int NT, int WM>
cudaError_t wy_down_t(const WyLevel& L, const WyPanels& P, int Call, int t, int ncol, int grid, size_t smem,
                      cudaStream_t st, int NG) {
  return NG == 2 ? wy_down_g<UW, NT, WM, 2>(L, P, Call, t, ncol, grid, smem, st)
                 : wy_down_g<UW, NT, WM, 1>(L, P, Call, t, ncol, grid, smem, st);
}

// (UW, NT, WM) instantiations: WM = 16 levels have UW <= 2 (alloc_level)
#define PQR_WY_SWITCH(UW_, NT_, WM_, CALL)                                                   \
  switch ((UW_) * 100 + (NT_) * 10 + ((WM_) > 8 ? 1 : 0)) {                                  \
    case 210: e = CALL(2, 1, 8); break;                                                      \
    case 410: e = CALL(4, 1, 8); break;                                                      \
    case 610: e = CALL(6, 1, 8); break;                                                      \
    case 211: e = CALL(2, 1, 16); break;                                                     \
    case 221: e = CALL(2, 2, 16); break;                                                     \
    default: return PQR_EPLAN;                                                               \
  }

// PQR_WY_TRACE=1: per-phase cycle counters of CTA 0 (warps 0 and 15) printed to stderr
// after every level kernel (tuning aid; serialises the stream).
unsigned long long* wy_trace_buf() {
  static unsigned long long* buf = nullptr;
  static const bool on = getenv("PQR_WY_TRACE") != nullptr;
  if (on && !buf) cudaMalloc(&buf, 64 * sizeof(unsigned long long));
  return on ? buf : nullptr;
}
void wy_trace_dump(const char* kind, const WyLevel& L, cudaStream_t st) {
  if (!L.trace) return;
  unsigned long long h[32];
  cudaStreamSynchronize(st);
  cudaMemcpy(h, L.trace, sizeof(h), cudaMemcpyDeviceToHost);
  fprintf(stderr, "{\"wy_trace\": \"%s\", \"nblocks\": %d, \"rows\": %lld, \"w0\": [", kind, L.nblocks, (long long)L.q);
  for (int i = 0; i < 16; ++i) fprintf(stderr, "%llu%s", h[i], i < 15 ? ", " : "], \"w15\": [");
  for (int i = 0; i < 16; ++i) fprintf(stderr, "%llu%s", h[16 + i], i < 15 ? ", " : "]}\n");
}

WyLevel to_wy(const TsqrState* ts, const TsqrLv& lv) {
  WyLevel L{};
  L.q = lv.q; L.rem2 = lv.rem2; L.odd_last = lv.odd_last; L.nblocks = lv.nblocks;
  L.b0 = 0; L.nrun = lv.nblocks;
  L.V = lv.V; L.ldv = lv.ldv; L.T = lv.T; L.tstride = lv.tstride;
  L.cap = ts->cap; L.RP = lv.RP; L.wmax = ts->wmax; L.nbuf = 2;  // set per kernel kind by the caller
  L.trace = wy_trace_buf();
  if (lv.chained) {  // the chained leaf level
    L.nchain = ts->nchain; L.LS = ts->wmax + 2; L.VC = ts->VC;
  }
  return L;
}
// grid and groups of a level launch: a chained level runs nchain / 2 CTAs of two groups (the
// chain of group g of CTA x is x + g * grid), whatever the number of blocks in the launch
void wy_shape(const Ctx* h, const TsqrLv& lv, const WyLevel& L, int* grid, int* NG) {
  if (L.nchain > 0) {
    *NG = 2;
    *grid = L.nchain / 2;
  } else {
    *NG = groups_for(L.nrun, h->sms, lv.UW);
    *grid = (int)std::min<int64_t>(L.nrun, h->sms);
  }
}

int run_wy_up(Ctx* h, const TsqrLv& lv, const double* X, int64_t ldx, double* out, int64_t ldo, int np, int C,
              int s, int merge = 0, int mtoff = 0, int64_t b0 = 0, int64_t nrun = -1) {
  TsqrState* ts = h->ts;
  WyLevel L = to_wy(ts, lv);
  if (nrun >= 0) { L.b0 = b0; L.nrun = nrun; }
  if (L.nrun == 0) return PQR_OK;
  L.X = X; L.ldx = ldx; L.out = out; L.ldo = ldo;
  L.orows = ldo < ts->cap ? (int)ldo : ts->cap;  // compact GPU-root block: C + s rows
  L.ovec = ((ts->cap & 1) == 0 && (ldo & 1) == 0 && aligned16(out)) ? 1 : 0;
  WyPanels P{ts->d_pan, np};
  const int NT = s > 8 ? 2 : 1;
  int NG, grid;
  wy_shape(h, lv, L, &grid, &NG);
  L.nbuf = nbuf_for(lv.RP, ts->wmax, ts->cap, NG);
  const size_t smem = wy_smem(lv.RP, ts->wmax, ts->cap, L.nbuf, NG);
  cudaError_t e;
#define UPC(U, N, W) wy_up_t<U, N, W>(L, P, C, s, merge, mtoff, grid, smem, h->stream, NG)
  PQR_WY_SWITCH(lv.UW, NT, ts->wmax, UPC)
#undef UPC
  wy_trace_dump("up", L, h->stream);
  ++h->st.kernel_launches;
  if (e != cudaSuccess) {
    fprintf(stderr, "[pqr] tsqr up launch: %s\n", cudaGetErrorString(e));
    return PQR_ECUDA;
  }
  return PQR_OK;
}

int run_wy_down(Ctx* h, const TsqrLv& lv, const double* cin, int64_t ldci, double* Y, int64_t ldy, int np,
                int Call, int t, int ncol, const int4* pan, int64_t b0 = 0, int64_t nrun = -1) {
  TsqrState* ts = h->ts;
  WyLevel L = to_wy(ts, lv);
  if (nrun >= 0) { L.b0 = b0; L.nrun = nrun; }
  if (L.nrun == 0) return PQR_OK;
  L.cin = cin; L.ldci = ldci; L.Y = Y; L.ldy = ldy;
  L.yvec = ((ldy & 1) == 0 && aligned16(Y)) ? 1 : 0;
  WyPanels P{pan, np};
  const int NT = ncol > 8 ? 2 : 1;
  int NG, grid;
  wy_shape(h, lv, L, &grid, &NG);
  L.nbuf = nbuf_for(lv.RP, ts->wmax, ts->cap, NG);
  const size_t smem = wy_smem(lv.RP, ts->wmax, ts->cap, L.nbuf, NG);
  cudaError_t e;
#define DNC(U, N, W) wy_down_t<U, N, W>(L, P, Call, t, ncol, grid, smem, h->stream, NG)
  PQR_WY_SWITCH(lv.UW, NT, ts->wmax, DNC)
#undef DNC
  wy_trace_dump("down", L, h->stream);
  ++h->st.kernel_launches;
  if (e != cudaSuccess) {
    fprintf(stderr, "[pqr] tsqr down launch: %s\n", cudaGetErrorString(e));
    return PQR_ECUDA;
  }
  return PQR_OK;
}

// host-pipeline chunk [u0, u1) of leaf units (chained leaves: a unit is one round of nchain blocks)
// -> blocks [b0, b0 + nrun)
void leaf_chunk(const TsqrState* ts, int64_t u0, int64_t u1, int64_t* b0, int64_t* nrun) {
  const int64_t unit = ts->nchain > 0 ? ts->nchain : 1, nb = ts->lv[0].nblocks;
  *b0 = std::min(nb, u0 * unit);
  *nrun = std::min(nb, u1 * unit) - *b0;
}

// Stage 1 over all levels: X (n_local x s) -> Btop ((C+s) x s, ld cap).  Creates s new
// reflectors (one new panel) at every level.
int tsqr_up_sweep(Ctx* h, const double* X, int64_t ldx, int s, int merge = 0, int mtoff = 0, bool pipe = false) {
  TsqrState* ts = h->ts;
  const int C = ts->C;
  const int np = (int)ts->panels.size();
  if (lpip(h)) {
    // local problem of the whole shard by BCGS-PIP+ against the explicit local basis (C columns):
    // U_loc into the basis' spare columns C.., and the coefficient block [P_loc; N_loc] ((C+s) x s)
    // into in_top (ld cap) for the reduction
    const int nch = h->hp.nch;
    h->hp.nch = 0;
    BasisView bv{h->basis, h->ld, h->cfg.n_local};
    bv.k = C;
    bv.local = true;
    int tt = 0;
    const int rc = cholqr2_solve(h, bv, X, ldx, s, 0, h->basis + (int64_t)C * h->ld, h->ld, nullptr, &tt, 0.0);
    h->hp.nch = nch;
    TRY(rc);
    if (C > 0)
      CUDA_TRY(cudaMemcpy2DAsync(ts->in_top, ts->cap * sizeof(double), h->Pf, (size_t)C * sizeof(double),
                                 (size_t)C * sizeof(double), s, cudaMemcpyDeviceToDevice, h->stream));
    CUDA_TRY(cudaMemcpy2DAsync(ts->in_top + C, ts->cap * sizeof(double), h->Nf, (size_t)kSMax * sizeof(double),
                               (size_t)s * sizeof(double), s, cudaMemcpyDeviceToDevice, h->stream));
  } else {
    PROF(h, PQR_K_TSQR_LOCAL);
    // the GPU root's block goes compact ((C+s) x s, ld C+s) when it is all-gathered
    const int64_t ldtop = h->xc && !pip2(h) ? C + s : ts->cap;
    double* out0 = ts->nlev >= 1 ? ts->lv[1].in : ts->in_top;
    const int64_t ldo0 = ts->nlev >= 1 ? ts->lv[1].rows : ldtop;
    if (pipe && h->hp.nch > 0) {
      // host X arrives chunk by chunk (leaf blocks are independent in stage 1)
      for (int c = 0; c < h->hp.nch; ++c) {
        TRY(hp_wait_in(h, c));
        int64_t b0, nrun;
        leaf_chunk(ts, h->hp.b[c], h->hp.b[c + 1], &b0, &nrun);
        TRY(run_wy_up(h, ts->lv[0], X, ldx, out0, ldo0, np, C, s, merge, mtoff, b0, nrun));
      }
    } else {
      TRY(run_wy_up(h, ts->lv[0], X, ldx, out0, ldo0, np, C, s, merge, mtoff));
    }
  }
  {
    PROF(h, PQR_K_TSQR_TREE);
    const int64_t ldtop = h->xc && !pip2(h) ? C + s : ts->cap;
    for (int l = 1; l <= ts->nlev; ++l) {
      const bool root = l == ts->nlev;
      TRY(run_wy_up(h, ts->lv[l], ts->lv[l].in, ts->lv[l].rows, root ? ts->in_top : ts->lv[l + 1].in,
                    root ? ldtop : ts->lv[l + 1].rows, np, C, s, merge, mtoff));
    }
  }
  if (h->xc && !pip2(h)) {
    const int P = h->cfg.nranks;
    const size_t cnt = (size_t)(C + s) * s;
    if (lpip(h)) {  // the allgather sends the block compact (ld C + s)
      CUDA_TRY(cudaMemcpy2DAsync(ts->Btop, (C + s) * sizeof(double), ts->in_top, ts->cap * sizeof(double),
                                 (size_t)(C + s) * sizeof(double), s, cudaMemcpyDeviceToDevice, h->stream));
      CUDA_TRY(cudaMemcpyAsync(ts->in_top, ts->Btop, cnt * sizeof(double), cudaMemcpyDeviceToDevice, h->stream));
    }
    {
      PROF(h, PQR_K_NCCL);
      TRY(h->xc->allgather(ts->in_top, ts->xraw, cnt, h->stream));
      h->st.collectives += 1;
      h->st.collective_bytes += (int64_t)cnt * 8;
    }
    PROF(h, PQR_K_TSQR_TREE);
    TsqrLv& x0 = ts->xlv[0];
    k_unpack_roots<<<std::max(1, std::min(64, (int)(((size_t)P * ts->cap * s + 255) / 256))), 256, 0, h->stream>>>(
        ts->xraw, C + s, s, P, x0.in, x0.rows, ts->cap);
    ++h->st.kernel_launches;
    CUDA_TRY(cudaGetLastError());
    const int nx = (int)ts->xlv.size();
    for (int l = 0; l < nx; ++l) {
      const bool top = l == nx - 1;
      TRY(run_wy_up(h, ts->xlv[l], ts->xlv[l].in, ts->xlv[l].rows, top ? ts->Btop : ts->xlv[l + 1].in,
                    top ? ts->cap : ts->xlv[l + 1].rows, np, C, s, merge, mtoff));
    }
  }
  return PQR_OK;
}

// Stage 2 over all levels: top coefficients cin (Call x ncol, ld cap) -> Y (n_local x ncol),
// applying the first np panels.
int tsqr_down_sweep(Ctx* h, int np, int Call, const double* cin, int t, int ncol, double* Y, int64_t ldy,
                    const int4* pan, bool pipe = false) {
  TsqrState* ts = h->ts;
  const double* root_cin = cin;
  int64_t root_ld = ts->cap;
  {
    PROF(h, PQR_K_TSQR_TREE);
    if (h->xc && !pip2(h)) {
      // the replicated cross-GPU levels, top down; this rank's root is child `rank` of the
      // first cross level
      const int nx = (int)ts->xlv.size();
      for (int l = nx - 1; l >= 0; --l) {
        const bool top = l == nx - 1;
        TRY(run_wy_down(h, ts->xlv[l], top ? cin : ts->xlv[l + 1].dn, top ? ts->cap : ts->xlv[l + 1].rows,
                        ts->xlv[l].dn, ts->xlv[l].rows, np, Call, t, ncol, pan));
      }
      root_cin = ts->xlv[0].dn + (int64_t)h->cfg.rank * ts->cap;
      root_ld = ts->xlv[0].rows;
    }
    for (int l = ts->nlev; l >= 1; --l) {
      const bool root = l == ts->nlev;
      TRY(run_wy_down(h, ts->lv[l], root ? root_cin : ts->lv[l + 1].dn, root ? root_ld : ts->lv[l + 1].rows,
                      ts->lv[l].dn, ts->lv[l].rows, np, Call, t, ncol, pan));
    }
  }
  PROF(h, PQR_K_TSQR_APPLY);
  if (lpip(h)) {
    // Y = [L_g U_loc] root_cin (Call rows: C basis columns, then Call - C columns of U_loc, which sit
    // in the basis' spare columns)
    const int C = ts->C;
    return run_update(h->cfg.n_local, C, h->basis, h->ld, Call - C, h->basis + (int64_t)C * h->ld, h->ld, root_cin,
                      (int)root_ld, ncol, nullptr, Y, ldy, nullptr, 0, h->sms, h->stream, &h->st.kernel_launches);
  }
  const double* cin0 = ts->nlev >= 1 ? ts->lv[1].dn : root_cin;
  const int64_t ldc0 = ts->nlev >= 1 ? ts->lv[1].rows : root_ld;
  if (pipe && h->hp.nch > 0) {
    // U leaves for the host chunk by chunk, each copy behind its chunk's stage-2 launch (chained
    // leaves: the chains are walked backwards, so the chunks are too)
    for (int cc = 0; cc < h->hp.nch; ++cc) {
      const int c = ts->nchain > 0 ? h->hp.nch - 1 - cc : cc;
      int64_t b0, nrun;
      leaf_chunk(ts, h->hp.b[c], h->hp.b[c + 1], &b0, &nrun);
      TRY(run_wy_down(h, ts->lv[0], cin0, ldc0, Y, ldy, np, Call, t, ncol, pan, b0, nrun));
      TRY(hp_d2h_chunk(h, c, Y, ldy, ncol));
    }
  } else {
    TRY(run_wy_down(h, ts->lv[0], cin0, ldc0, Y, ldy, np, Call, t, ncol, pan));
  }
  return PQR_OK;
}

int run_top(Ctx* h, int s, bool build, double* P, int ldp, double* N, int ldn, int* t_dev, int* defl) {
  TsqrState* ts = h->ts;
  TsqrTopArgs a{};
  a.B = ts->Btop; a.ldb = ts->cap; a.Rt = ts->Rt; a.ldr = ts->cap;
  a.C = ts->C; a.k = h->k; a.s = s;
  a.tau_rel = h->cfg.defl_tol > 0 ? h->cfg.defl_tol : 1e-12;
  a.build = build ? 1 : 0;
  a.P = P; a.ldp = ldp; a.N = N; a.ldn = ldn; a.Ut = ts->Ut; a.ldu = ts->cap;
  a.t_out = t_dev; a.deflated = defl;
  PROF(h, PQR_K_FACTOR);
  k_tsqr_top<<<1, 256, 0, h->stream>>>(a);
  ++h->st.kernel_launches;
  CUDA_TRY(cudaGetLastError());
  return PQR_OK;
}

// reduction = PIP+ (PQR_REDUCTION_PIP2): BCGS-PIP+ (Alg. 8) of the GPU root's block B_g (C+s rows)
// against this GPU's top coordinates R_g of the basis (Q = blockdiag(L_g) [R_0; ...; R_{P-1}],
// L_g the GPU's locally orthogonal basis): the CholQR2 orchestration on (C+s)-row matrices, with
// its two (k+s) x s Gram exchanges; the coordinates of U land in Ut (ld cap) for the down sweep.
int run_pip2_top(Ctx* h, int s, unsigned flags) {
  TsqrState* ts = h->ts;
  const double tau = h->cfg.defl_tol > 0 ? h->cfg.defl_tol : 1e-12;
  const int nch = h->hp.nch;  // the host-buffer pipeline concerns the leaf level only
  h->hp.nch = 0;
  int tt = 0;
  const int rc = cholqr2_solve(h, BasisView{ts->Rt, ts->cap, ts->C + s}, ts->Btop, ts->cap, s,
                               flags & (PQR_SINGLE_PASS | PQR_NO_DEFLATION), ts->Ut, ts->cap, nullptr, &tt, tau);
  h->hp.nch = nch;
  return rc;
}

// register the new panel (C, s) in the device list at slot np (uncommitted)
bool int4_eq(const int4& a, const int4& b) { return a.x == b.x && a.y == b.y && a.z == b.z && a.w == b.w; }

// d_pan[i] = v (host-to-device copy only when the device copy differs)
int set_pan(Ctx* h, int i, const int4& v) {
  TsqrState* ts = h->ts;
  if (ts->pan_mirror.size() <= (size_t)i) ts->pan_mirror.resize(i + 1, make_int4(-1, -1, -1, -1));
  if (int4_eq(ts->pan_mirror[i], v)) return PQR_OK;
  ts->pan_mirror[i] = v;
  CUDA_TRY(cudaMemcpyAsync(ts->d_pan + i, &ts->pan_mirror[i], sizeof(int4), cudaMemcpyHostToDevice, h->stream));
  return PQR_OK;
}

int tsqr_stage_panel(Ctx* h, int s) {
  TsqrState* ts = h->ts;
  const int np = (int)ts->panels.size();
  return set_pan(h, np, make_int4(ts->C, s, 16 * ts->C, 0));
}

// commit: R_top[:, k..k+t) = U~[0:C+s, 0:t);  panel (C, s) committed — or, when the call
// merged it into the previous panel, that panel widened to 8 with the merged T;  C += s
// (k += t by the caller)
int tsqr_commit(Ctx* h, int s, int t, int merge = 0, int mtoff = 0) {
  TsqrState* ts = h->ts;
  if (t > 0)
    CUDA_TRY(cudaMemcpy2DAsync(ts->Rt + (int64_t)h->k * ts->cap, ts->cap * sizeof(double), ts->Ut,
                               ts->cap * sizeof(double), (size_t)(ts->C + s) * sizeof(double), t,
                               cudaMemcpyDeviceToDevice, h->stream));
  if (merge) {
    int4& pv = ts->panels.back();
    pv = make_int4(pv.x, pv.y + s, mtoff, 1);
    const int np = (int)ts->panels.size();
    TRY(set_pan(h, np - 1, pv));
  } else {
    ts->panels.push_back(make_int4(ts->C, s, 16 * ts->C, 0));
  }
  ts->C += s;
  return PQR_OK;
}

int alloc_level(Ctx* h, TsqrLv& lv, int wmax, bool with_io) {
  TsqrState* ts = h->ts;
  int rc;
  // (a chained leaf also holds the tail's s <= wmax carried pivot rows in its last register rows)
  lv.UW = uw_for(lv.q + 2 * (lv.rem2 > 0) + lv.odd_last + (lv.chained ? wmax : 0));
  lv.RP = rp_for(lv.UW);
  if (lv.UW > 6 || (wmax > 8 && lv.UW > 2) || std::max(wy_smem(lv.RP, wmax, ts->cap, 2, 1), wy_smem(lv.RP, wmax, ts->cap, 2, 2)) > kWySmemBudget)
    return PQR_EPLAN;
  lv.tstride = (int64_t)32 * ts->cap;  // [0, 16 cap): per-panel T at 16*start; then merged-pair T
  if (lv.owns_v && (rc = dalloc(&lv.V, (size_t)lv.rows * ts->cap))) return rc;
  if (lv.owns_v && with_io) CUDA_TRY(cudaMemsetAsync(lv.V, 0, sizeof(double) * lv.rows * ts->cap, h->stream));
  if ((rc = dalloc(&lv.T, (size_t)lv.nblocks * lv.tstride))) return rc;
  if (with_io) {
    if ((rc = dalloc(&lv.in, (size_t)lv.rows * wmax)) || (rc = dalloc(&lv.dn, (size_t)lv.rows * wmax))) return rc;
    CUDA_TRY(cudaMemsetAsync(lv.in, 0, sizeof(double) * lv.rows * wmax, h->stream));
  }
  return PQR_OK;
}

int tsqr_alloc(Ctx* h) {
  TsqrState* ts = h->ts;
  const int64_t n = h->cfg.n_local;
  const int cap = h->cap;
  ts->cap = cap;
  ts->wmax = h->cfg.s_max > 8 ? 16 : 8;
  const int wmax = ts->wmax;
  // node arity: even, node rows within the register/shared-memory budget
  const int rmax = wmax > 8 ? 512 : 1024;
  // node rows arity*cap <= rmax, even (paired 16-byte rows): odd arity only with even cap
  ts->arity = std::max(2, std::min(64, rmax / cap));  // (8 before round 2: an extra level at small cap)
  if ((cap & 1) && (ts->arity & 1)) ts->arity -= 1;
  ts->arity = std::max(2, ts->arity);
  int rc;
  ts->lv.clear();
  if (lpip(h)) {
    // local = PIP+: the explicit local basis (n_local x cap) replaces the leaf and node levels
    if ((rc = dalloc(&h->basis, (size_t)h->ld * cap))) return rc;
    ts->nb = 0;
    ts->nlev = 0;
  } else {
  // leaf block rows: user's choice or ~1024 (512 when s_max > 8)
  const int RB = wmax > 8 ? 512 : 1024;  // rows a two-group level kernel holds per block
  int nb = h->cfg.block_rows > 0 ? h->cfg.block_rows : RB;
  nb = std::max(nb, 2 * cap);
  if (nb < cap || n < cap) return PQR_EPLAN;
  // FlatTSPQR chains (§4.2, Alg. 10; WyLevel): a chained block's carry rows live
  // outside the register file but the tail's s pivot rows, which take the last wmax register rows
  // (own rows <= RB - wmax); used when every chain gets several blocks (cfg.chains:
  // PQR_CHAINS_AUTO, _OFF, _ON = whenever there are more leaf blocks than chains)
  const int NC = 2 * h->sms;
  const int own = h->cfg.block_rows > 0 ? nb : RB - wmax;
  int cmode = h->cfg.chains;
  if (const char* e = getenv("PQR_CHAINS"))  // A/B aid: overrides the handle's setting
    cmode = !strcmp(e, "off") ? PQR_CHAINS_OFF : !strcmp(e, "on") ? PQR_CHAINS_ON : PQR_CHAINS_AUTO;
  // (AUTO = the pure tree: on B200 the chained leaf kernels are measured slower than the tree
  // levels they replace)
  const bool chains = cmode == PQR_CHAINS_ON && own >= cap && own <= RB - wmax && n / own >= (int64_t)NC + 1;
  if (chains) nb = own;
  int64_t p0 = std::max<int64_t>(1, (n + nb - 1) / nb);
  // the largest block (q, + 2 for the first rem2 blocks, + 1 odd row) must not exceed nb
  auto max_rows = [&](int64_t p) {
    const int64_t q = (n / p) & ~int64_t(1), rest = n - p * q;
    return q + (rest / 2 > 0 ? 2 : 0) + (rest & 1);
  };
  while (max_rows(p0) > nb && (n / (p0 + 1)) >= cap) ++p0;
  while (p0 > 1 && ((n / p0) & ~int64_t(1)) < cap) --p0;
  TsqrLv leaf;
  leaf.nblocks = (int)p0;
  leaf.q = (n / p0) & ~int64_t(1);
  const int64_t rest = n - p0 * leaf.q;
  leaf.rem2 = rest / 2;
  leaf.odd_last = (int)(rest & 1);
  leaf.rows = h->ld;
  leaf.ldv = h->ld;
  leaf.chained = chains;
  ts->nb = nb;
  ts->nchain = chains ? NC : 0;
  TRY(alloc_level(h, leaf, wmax, false));
  if (chains) {
    if ((rc = dalloc(&ts->VC, (size_t)p0 * cap * (wmax + 2)))) return rc;
  }
  if (n & 1)  // zero pad row n of every reflector column (bulk copies of the odd last block read it)
    CUDA_TRY(cudaMemset2DAsync(leaf.V + n, leaf.ldv * sizeof(double), 0, sizeof(double), cap, h->stream));
  ts->lv.clear();
  ts->lv.push_back(leaf);
  int pl = chains ? NC : (int)p0;  // children of the first node level: chains or leaf blocks
  while (pl > 1) {
    pl = (pl + ts->arity - 1) / ts->arity;
    TsqrLv nd;
    nd.nblocks = pl;
    nd.q = (int64_t)ts->arity * cap;
    nd.rows = (int64_t)pl * nd.q;
    nd.ldv = nd.rows;
    TRY(alloc_level(h, nd, wmax, true));
    ts->lv.push_back(nd);
  }
  ts->nlev = (int)ts->lv.size() - 1;
  }

  if ((rc = dalloc(&ts->in_top, (size_t)cap * wmax))) return rc;
  CUDA_TRY(cudaMemsetAsync(ts->in_top, 0, sizeof(double) * cap * wmax, h->stream));
  if ((rc = dalloc(&ts->Ut, (size_t)cap * 16))) return rc;
  if ((rc = dalloc(&ts->Rt, (size_t)cap * cap))) return rc;
  CUDA_TRY(cudaMemsetAsync(ts->Rt, 0, sizeof(double) * cap * cap, h->stream));
  if ((rc = dalloc(&ts->coef, (size_t)cap * 16))) return rc;
  if ((rc = dalloc(&ts->d_pan, (size_t)cap + 1)) || (rc = dalloc(&ts->d_panm, (size_t)cap + 1))) return rc;
  if (h->xc && !pip2(h)) {
    // cross-GPU levels over the nranks GPU roots, arity-bounded like the on-GPU node levels
    // (a level with more children than the arity is split into nodes of arity children; the
    // last level is one node of its children, an odd row count kept as the odd last row)
    int cnt = h->cfg.nranks;
    ts->xlv.clear();
    for (;;) {
      TsqrLv x;
      if (cnt <= ts->arity) {
        const int64_t r = (int64_t)cnt * cap;
        x.nblocks = 1;
        x.q = r & ~int64_t(1);
        x.odd_last = (int)(r & 1);
        x.rows = r + (r & 1);
      } else {
        x.nblocks = (cnt + ts->arity - 1) / ts->arity;
        x.q = (int64_t)ts->arity * cap;
        x.rows = (int64_t)x.nblocks * x.q;
      }
      x.ldv = x.rows;
      TRY(alloc_level(h, x, wmax, true));
      ts->xlv.push_back(x);
      if (x.nblocks == 1) break;
      cnt = x.nblocks;
    }
    if ((rc = dalloc(&ts->xraw, (size_t)h->cfg.nranks * cap * wmax))) return rc;
    if ((rc = dalloc(&ts->Btop, (size_t)cap * wmax))) return rc;
  } else {
    ts->Btop = ts->in_top;
  }
  h->st.block_rows = lpip(h) ? 0 : (int)ts->lv[0].q;
  h->st.tree_levels = ts->nlev;
  h->st.leaf_chains = ts->nchain;
  return PQR_OK;
}

// LOR build (§8(a) a9): one up-sweep per chunk of wmax columns of Q; the top
// coefficients of each chunk become R_top's columns (Q = L [R_top; 0]).
int tsqr_create(Ctx* h, const double* Q, int64_t ldq, int k) {
  h->ts = new TsqrState();
  TRY(tsqr_alloc(h));
  TsqrState* ts = h->ts;
  h->k = 0;
  ts->C = 0;
  // (local = PIP+: the local CholQR2's small buffers hold s_max columns)
  const int chunk = lpip(h) ? std::min(ts->wmax, h->cfg.s_max) : ts->wmax;
  // 16-byte aligned copy of Q with even ld for the bulk copies (freed on every exit path)
  struct AlignedQ {
    double* p = nullptr;
    cudaStream_t st = nullptr;
    ~AlignedQ() {
      if (p) {
        cudaStreamSynchronize(st);
        cudaFree(p);
      }
    }
  } qa;
  qa.st = h->stream;
  if (k > 0 && ((ldq & 1) || !aligned16(Q))) {
    TRY(dalloc(&qa.p, (size_t)h->ld * k));
    CUDA_TRY(cudaMemcpy2DAsync(qa.p, h->ld * sizeof(double), Q, ldq * sizeof(double),
                               h->cfg.n_local * sizeof(double), k, cudaMemcpyDeviceToDevice, h->stream));
    Q = qa.p;
    ldq = h->ld;
  }
  for (int c0 = 0; c0 < k; c0 += chunk) {
    const int cs = std::min(chunk, k - c0);
    TRY(tsqr_up_sweep(h, Q + (int64_t)c0 * ldq, ldq, cs));
    if (pip2(h)) {
      // the chunk's coordinates are the new columns of R_g (Q = L [R; 0]: no PQR to solve)
      CUDA_TRY(cudaMemcpy2DAsync(ts->Ut, ts->cap * sizeof(double), ts->in_top, ts->cap * sizeof(double),
                                 (size_t)(ts->C + cs) * sizeof(double), cs, cudaMemcpyDeviceToDevice, h->stream));
    } else {
      TRY(run_top(h, cs, true, h->Pf, std::max(1, h->k), h->Nf, kSMax, h->ints + 2, h->ints + 3));
    }
    TRY(tsqr_stage_panel(h, cs));
    TRY(tsqr_commit(h, cs, cs));
    h->k += cs;
  }
  return PQR_OK;
}

// start rows of the leaf blocks (nblocks + 1 entries, the last = n_local): host-pipeline chunking
// (chained leaves: one entry per round of nchain blocks; leaf_chunk maps units back to blocks)
void tsqr_leaf_bounds(Ctx* h, std::vector<int64_t>* out) {
  const TsqrLv& lv = h->ts->lv[0];
  const int64_t unit = h->ts->nchain > 0 ? h->ts->nchain : 1;
  const int64_t nu = (lv.nblocks + unit - 1) / unit;
  out->resize((size_t)nu + 1);
  for (int64_t u = 0; u < nu; ++u) {
    const int64_t b = u * unit;
    (*out)[u] = b * lv.q + 2 * std::min<int64_t>(b, lv.rem2);
  }
  (*out)[nu] = h->cfg.n_local;
}

int tsqr_solve(Ctx* h, const double* X, int64_t ldx, int s, unsigned flags, double* Ud, int64_t ldud, bool append,
               int* t_host) {
  TsqrState* ts = h->ts;
  if (ts->C + s > ts->cap) return PQR_ECAPACITY;
  const int np = (int)ts->panels.size();
  if ((ldx & 1) || !aligned16(X)) {  // the leaf kernel streams X with 16-byte bulk copies
    if (!h->stageX && dalloc(&h->stageX, (size_t)h->ld * h->cfg.s_max)) return PQR_ENOMEM;
    CUDA_TRY(cudaMemcpy2DAsync(h->stageX, h->ld * sizeof(double), X, ldx * sizeof(double),
                               h->cfg.n_local * sizeof(double), s, cudaMemcpyDeviceToDevice, h->stream));
    X = h->stageX;
    ldx = h->ld;
  }
  // Narrow blocks (Arnoldi's s = 4): a 4-wide panel is merged with the previous 4-wide one
  // into a full 8-wide panel (the up kernels build the merged T).
  static const bool no_merge = getenv("PQR_NO_MERGE") != nullptr;
  ts->merge = 0;
  ts->mtoff = 0;
  if (!no_merge && !lpip(h) && ts->wmax == 8 && np >= 1) {
    const int4 pv = ts->panels.back();
    if (pv.w == 0 && pv.y == 4 && s == 4 && pv.x + pv.y == ts->C) {
      ts->merge = 1;
      ts->mtoff = 16 * ts->cap + 16 * pv.x;
    }
  }
  TRY(tsqr_up_sweep(h, X, ldx, s, ts->merge, ts->mtoff, true));
  if (pip2(h)) {
    TRY(run_pip2_top(h, s, flags));
  } else {
    TRY(run_top(h, s, false, h->Pf, std::max(1, h->k), h->Nf, kSMax, h->ints + 2, h->ints + 3));
  }
  // U~ columns >= t are zero, so the down sweep writes zeros there.
  if (ts->merge) {
    std::vector<int4> lst(ts->panels);
    lst.back() = make_int4(lst.back().x, 8, ts->mtoff, 1);
    bool same = ts->panm_mirror.size() == lst.size();
    for (size_t i = 0; same && i < lst.size(); ++i) same = int4_eq(ts->panm_mirror[i], lst[i]);
    if (!same) {
      ts->panm_mirror = lst;
      CUDA_TRY(cudaMemcpyAsync(ts->d_panm, ts->panm_mirror.data(), sizeof(int4) * np, cudaMemcpyHostToDevice,
                               h->stream));
    }
    TRY(tsqr_down_sweep(h, np, ts->C + s, ts->Ut, s, s, Ud, ldud, ts->d_panm, true));
  } else {
    TRY(tsqr_stage_panel(h, s));
    TRY(tsqr_down_sweep(h, np + 1, ts->C + s, ts->Ut, s, s, Ud, ldud, ts->d_pan, true));
  }
  // t reaches the host with the caller's single synchronisation; the caller commits the
  // panel (tsqr_commit) once t is known and the call has not failed
  CUDA_TRY(cudaMemcpyAsync(h->h_ints, h->ints, sizeof(int) * 8, cudaMemcpyDeviceToHost, h->stream));
  (void)t_host;
  (void)flags;
  (void)append;
  return PQR_OK;
}

// Y = Q C = L [R_top C; 0]: coef = R_top C (small update-kernel product), then stage 2.
int tsqr_apply(Ctx* h, const double* C, int ldc, int m, double* Y, int64_t ldy) {
  TsqrState* ts = h->ts;
  const int k = h->k;
  const bool stage = is_host_ptr(Y) || (ldy & 1) || !aligned16(Y);
  if (stage && !h->stageU && dalloc(&h->stageU, (size_t)h->ld * h->cfg.s_max)) return PQR_ENOMEM;
  if (!h->stageC && dalloc(&h->stageC, (size_t)h->cap * 16)) return PQR_ENOMEM;
  const int nt_max = lpip(h) || (ts->lv[0].UW <= 2 && (ts->nlev == 0 || ts->lv[1].UW <= 2)) ? 2 : 1;
  int chunk = std::min(8 * nt_max, stage ? h->cfg.s_max : 16);
  const int np = (int)ts->panels.size();
  for (int c0 = 0; c0 < m; c0 += chunk) {
    const int mc = std::min(chunk, m - c0);
    double* dst = stage ? h->stageU : Y + (int64_t)c0 * ldy;
    const int64_t ldd = stage ? h->ld : ldy;
    if (k == 0) {
      CUDA_TRY(cudaMemset2DAsync(dst, ldd * sizeof(double), 0, h->cfg.n_local * sizeof(double), mc, h->stream));
    } else {
      CUDA_TRY(cudaMemcpy2DAsync(h->stageC, (size_t)k * sizeof(double), C + (int64_t)c0 * ldc,
                                 (size_t)ldc * sizeof(double), (size_t)k * sizeof(double), mc, cudaMemcpyDefault,
                                 h->stream));
      {
        PROF(h, PQR_K_UPDATE);
        // coef (C x mc, ld cap) = R_top (C x k) * Cchunk (k x mc)
        TRY(run_update(ts->C, k, ts->Rt, ts->cap, 0, nullptr, 0, h->stageC, k, mc, nullptr, ts->coef, ts->cap,
                       nullptr, 0, h->sms, h->stream, &h->st.kernel_launches));
      }
      TRY(tsqr_down_sweep(h, np, ts->C, ts->coef, mc, mc, dst, ldd, ts->d_pan));
    }
    if (stage)
      CUDA_TRY(cudaMemcpy2DAsync(Y + (int64_t)c0 * ldy, ldy * sizeof(double), h->stageU, h->ld * sizeof(double),
                                 h->cfg.n_local * sizeof(double), mc, cudaMemcpyDefault, h->stream));
  }
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  prof_collect(h);
  return PQR_OK;
}

void free_level(TsqrLv& lv) {
  if (lv.owns_v) cudaFree(lv.V);
  cudaFree(lv.T);
  cudaFree(lv.in);
  cudaFree(lv.dn);
  lv.V = lv.T = lv.in = lv.dn = nullptr;
}

void tsqr_free(Ctx* h) {
  TsqrState* ts = h->ts;
  if (!ts) return;
  for (auto& lv : ts->lv) free_level(lv);
  for (auto& lv : ts->xlv) free_level(lv);
  cudaFree(ts->in_top);
  cudaFree(ts->xraw);
  if (ts->Btop != ts->in_top) cudaFree(ts->Btop);
  cudaFree(ts->Ut);
  cudaFree(ts->Rt);
  cudaFree(ts->coef);
  cudaFree(ts->VC);
  cudaFree(ts->d_pan);
  cudaFree(ts->d_panm);
  delete ts;
  h->ts = nullptr;
}

}  // namespace
