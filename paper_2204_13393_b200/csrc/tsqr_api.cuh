// tsqr_api.cuh — orchestration of the TSQR variant (TreeTSPQR, §4.1 Alg. 9),
// included by pqr_api.cu inside its anonymous namespace.
//
// Levels (see tsqr_kernels.cuh): leaves (level 0) partition the GPU's n_local rows
// into p0 blocks of ~n_b rows; each node level stacks `arity` children's top-cap
// coordinates (R = arity*cap rows per node); the level with one node is the GPU
// root.  With nranks > 1 the roots' outputs are all-gathered and one more node (the
// cross-GPU level, arity = nranks, replicated on every GPU) reduces them — the
// "different algorithm at the cross-GPU level" slot of the paper's framework is
// this replicated stateful node (§8(e)).
namespace {

constexpr int kArity = 8;

struct TsqrState {
  int nb = 0, cap = 0, C = 0, nlev = 0;
  int p0 = 0;
  int64_t q0 = 0, rem0 = 0;
  int rpt_leaf = 0, rpt_node = 0, rpt_x = 0;
  std::vector<int> p;            // nodes per level, index 1..nlev
  std::vector<int64_t> ldl;      // rows of a level's buffers (p_L * R)
  double* Vleaf = nullptr;       // n_local x cap, ld = h->ld
  std::vector<double*> Vn, in, dn;
  double* in_top = nullptr;      // cap x s_max: GPU root stage-1 output (ld cap)
  double* xraw = nullptr;        // nranks * cap * s_max allgather receive
  double* xin = nullptr;         // (nranks*cap) x s_max cross node input
  double* Vx = nullptr;          // (nranks*cap) x cap cross node reflectors
  double* xdn = nullptr;         // (nranks*cap) x s_max cross node stage-2 output
  double* Btop = nullptr;        // cap x s_max top coefficients of X (ld cap)
  double* Ut = nullptr;          // cap x s_max top coefficients of U (ld cap)
  double* Rt = nullptr;          // cap x cap explicit top basis (ld cap), zero-init
  double* coef = nullptr;        // cap x 16 scratch for basis_apply
};

int pick_S(int s) { return s <= 4 ? 4 : (s <= 8 ? 8 : 16); }
int pick_rpt(int64_t rows) {
  const int r = (int)((rows + kTsqrThreads - 1) / kTsqrThreads);
  if (r <= 1) return 1;
  if (r <= 2) return 2;
  if (r <= 4) return 4;
  if (r <= 5) return 5;
  if (r <= 6) return 6;
  if (r <= 8) return 8;
  return -1;
}

template <int RPT, int S>
cudaError_t launch_up_t(const TsqrLevel& L, int C, int s, cudaStream_t st) {
  k_tsqr_up<RPT, S><<<L.nblocks, kTsqrThreads, 0, st>>>(L, C, s);
  return cudaGetLastError();
}
template <int RPT, int S>
cudaError_t launch_down_t(const TsqrLevel& L, int C, int t, int ncol, cudaStream_t st) {
  k_tsqr_down<RPT, S><<<L.nblocks, kTsqrThreads, 0, st>>>(L, C, t, ncol);
  return cudaGetLastError();
}

int run_up(Ctx* h, const TsqrLevel& L, int rpt, int C, int s) {
  cudaError_t e = cudaSuccess;
  const int S = pick_S(s);
#define UPCALL(R, SS) launch_up_t<R, SS>(L, C, s, h->stream)
  switch (rpt * 100 + S) {
    case 104: e = UPCALL(1, 4); break;  case 108: e = UPCALL(1, 8); break;
    case 116: e = UPCALL(1, 16); break; case 204: e = UPCALL(2, 4); break;
    case 208: e = UPCALL(2, 8); break;  case 216: e = UPCALL(2, 16); break;
    case 404: e = UPCALL(4, 4); break;  case 408: e = UPCALL(4, 8); break;
    case 416: e = UPCALL(4, 16); break; case 504: e = UPCALL(5, 4); break;
    case 508: e = UPCALL(5, 8); break;  case 604: e = UPCALL(6, 4); break;
    case 608: e = UPCALL(6, 8); break;  case 804: e = UPCALL(8, 4); break;
    case 808: e = UPCALL(8, 8); break;
    default: return PQR_EPLAN;
  }
#undef UPCALL
  ++h->st.kernel_launches;
  if (e != cudaSuccess) {
    fprintf(stderr, "[pqr] tsqr up launch: %s\n", cudaGetErrorString(e));
    return PQR_ECUDA;
  }
  return PQR_OK;
}

int run_down(Ctx* h, const TsqrLevel& L, int rpt, int C, int t, int ncol, int Sw) {
  cudaError_t e = cudaSuccess;
  const int S = pick_S(Sw);
#define DNCALL(R, SS) launch_down_t<R, SS>(L, C, t, ncol, h->stream)
  switch (rpt * 100 + S) {
    case 104: e = DNCALL(1, 4); break;  case 108: e = DNCALL(1, 8); break;
    case 116: e = DNCALL(1, 16); break; case 204: e = DNCALL(2, 4); break;
    case 208: e = DNCALL(2, 8); break;  case 216: e = DNCALL(2, 16); break;
    case 404: e = DNCALL(4, 4); break;  case 408: e = DNCALL(4, 8); break;
    case 416: e = DNCALL(4, 16); break; case 504: e = DNCALL(5, 4); break;
    case 508: e = DNCALL(5, 8); break;  case 604: e = DNCALL(6, 4); break;
    case 608: e = DNCALL(6, 8); break;  case 804: e = DNCALL(8, 4); break;
    case 808: e = DNCALL(8, 8); break;
    default: return PQR_EPLAN;
  }
#undef DNCALL
  ++h->st.kernel_launches;
  if (e != cudaSuccess) {
    fprintf(stderr, "[pqr] tsqr down launch: %s\n", cudaGetErrorString(e));
    return PQR_ECUDA;
  }
  return PQR_OK;
}

bool rpt_ok(int rpt, int S) { return rpt > 0 && rpt * S <= 64 && !(rpt >= 5 && S == 16); }

// largest column chunk (S) usable with every level's rows-per-thread
int max_chunk(const TsqrState* ts) {
  const int r = std::max(ts->rpt_leaf, std::max(ts->rpt_node, ts->rpt_x));
  if (rpt_ok(r, 16)) return 16;
  if (rpt_ok(r, 8)) return 8;
  return 4;
}

TsqrLevel leaf_level(Ctx* h) {
  TsqrState* ts = h->ts;
  TsqrLevel L{};
  L.q = ts->q0; L.rem = ts->rem0; L.nblocks = ts->p0; L.cap = ts->cap;
  L.V = ts->Vleaf; L.ldv = h->ld;
  return L;
}
TsqrLevel node_level(Ctx* h, int lev) {
  TsqrState* ts = h->ts;
  TsqrLevel L{};
  L.q = (int64_t)kArity * ts->cap; L.rem = 0; L.nblocks = ts->p[lev]; L.cap = ts->cap;
  L.V = ts->Vn[lev]; L.ldv = ts->ldl[lev];
  L.X = ts->in[lev]; L.ldx = ts->ldl[lev];
  L.Y = ts->dn[lev]; L.ldy = ts->ldl[lev];
  return L;
}
TsqrLevel cross_level(Ctx* h) {
  TsqrState* ts = h->ts;
  TsqrLevel L{};
  const int64_t R = (int64_t)h->cfg.nranks * ts->cap;
  L.q = R; L.rem = 0; L.nblocks = 1; L.cap = ts->cap;
  L.V = ts->Vx; L.ldv = R;
  L.X = ts->xin; L.ldx = R;
  L.Y = ts->xdn; L.ldy = R;
  return L;
}

// Stage 1 over all levels: X (n_local x s) -> Btop ((C+s) x s, ld cap).  Creates s new
// reflectors at every level (columns C..C+s-1).
int tsqr_up_sweep(Ctx* h, const double* X, int64_t ldx, int s) {
  TsqrState* ts = h->ts;
  const int C = ts->C;
  {
    PROF(h, PQR_K_TSQR_LOCAL);
    TsqrLevel L = leaf_level(h);
    L.X = X; L.ldx = ldx;
    L.out = ts->nlev >= 1 ? ts->in[1] : ts->in_top;
    L.ldo = ts->nlev >= 1 ? ts->ldl[1] : ts->cap;
    TRY(run_up(h, L, ts->rpt_leaf, C, s));
  }
  {
    PROF(h, PQR_K_TSQR_TREE);
    for (int lev = 1; lev <= ts->nlev; ++lev) {
      TsqrLevel L = node_level(h, lev);
      L.out = lev < ts->nlev ? ts->in[lev + 1] : ts->in_top;
      L.ldo = lev < ts->nlev ? ts->ldl[lev + 1] : ts->cap;
      TRY(run_up(h, L, ts->rpt_node, C, s));
    }
  }
  if (h->cfg.nranks > 1) {
    const int P = h->cfg.nranks;
    {
      PROF(h, PQR_K_NCCL);
      NCCL_TRY(ncclAllGather(ts->in_top, ts->xraw, (size_t)ts->cap * s, ncclDouble, h->comm, h->stream));
      h->st.collectives += 1;
      h->st.collective_bytes += (int64_t)ts->cap * s * 8;
    }
    PROF(h, PQR_K_TSQR_TREE);
    for (int g = 0; g < P; ++g)
      CUDA_TRY(cudaMemcpy2DAsync(ts->xin + (int64_t)g * ts->cap, (size_t)P * ts->cap * sizeof(double),
                                 ts->xraw + (int64_t)g * ts->cap * s, (size_t)ts->cap * sizeof(double),
                                 (size_t)ts->cap * sizeof(double), s, cudaMemcpyDeviceToDevice, h->stream));
    TsqrLevel L = cross_level(h);
    L.out = ts->Btop; L.ldo = ts->cap;
    TRY(run_up(h, L, ts->rpt_x, C, s));
  }
  return PQR_OK;
}

// Stage 2 over all levels: top coefficients cin ((Call) x ncol, ld cap) -> Y (n_local x ncol).
int tsqr_down_sweep(Ctx* h, int Call, const double* cin, int t, int ncol, double* Y, int64_t ldy) {
  TsqrState* ts = h->ts;
  const double* root_cin = cin;
  int64_t root_ld = ts->cap;
  {
    PROF(h, PQR_K_TSQR_TREE);
    if (h->cfg.nranks > 1) {
      TsqrLevel L = cross_level(h);
      L.cin = cin; L.ldci = ts->cap;
      TRY(run_down(h, L, ts->rpt_x, Call, t, ncol, ncol));
      root_cin = ts->xdn + (int64_t)h->cfg.rank * ts->cap;
      root_ld = (int64_t)h->cfg.nranks * ts->cap;
    }
    for (int lev = ts->nlev; lev >= 1; --lev) {
      TsqrLevel L = node_level(h, lev);
      L.cin = lev == ts->nlev ? root_cin : ts->dn[lev + 1];
      L.ldci = lev == ts->nlev ? root_ld : ts->ldl[lev + 1];
      TRY(run_down(h, L, ts->rpt_node, Call, t, ncol, ncol));
    }
  }
  PROF(h, PQR_K_TSQR_APPLY);
  TsqrLevel L = leaf_level(h);
  L.cin = ts->nlev >= 1 ? ts->dn[1] : root_cin;
  L.ldci = ts->nlev >= 1 ? ts->ldl[1] : root_ld;
  L.Y = Y; L.ldy = ldy;
  TRY(run_down(h, L, ts->rpt_leaf, Call, t, ncol, ncol));
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

// commit: R_top[:, k..k+t) = U~[0:C+s, 0:t);  C += s;  (k += t by the caller)
int tsqr_commit(Ctx* h, int s, int t) {
  TsqrState* ts = h->ts;
  if (t > 0)
    CUDA_TRY(cudaMemcpy2DAsync(ts->Rt + (int64_t)h->k * ts->cap, ts->cap * sizeof(double), ts->Ut,
                               ts->cap * sizeof(double), (size_t)(ts->C + s) * sizeof(double), t,
                               cudaMemcpyDeviceToDevice, h->stream));
  ts->C += s;
  return PQR_OK;
}

int tsqr_alloc(Ctx* h) {
  TsqrState* ts = h->ts;
  const int64_t n = h->cfg.n_local;
  const int cap = h->cap;
  const int sm = h->cfg.s_max;
  ts->cap = cap;
  const int Smax = pick_S(sm);
  // leaf block rows: user's choice or the largest that keeps RPT*S <= 64 (rows in registers)
  int nb = h->cfg.block_rows;
  if (nb <= 0) {
    nb = kTsqrThreads * (64 / Smax) / 2;
    if (Smax == 4) nb = 2048;
    nb = std::max(nb, 2 * cap);
  }
  if (nb < cap) return PQR_EPLAN;
  if (n < cap) return PQR_EPLAN;
  int64_t p0 = (n + nb - 1) / nb;
  if (n / p0 < cap) p0 = std::max<int64_t>(1, n / cap);
  ts->nb = nb;
  ts->p0 = (int)p0;
  ts->q0 = n / p0;
  ts->rem0 = n % p0;
  ts->rpt_leaf = pick_rpt(ts->q0 + (ts->rem0 ? 1 : 0));
  ts->rpt_node = pick_rpt((int64_t)kArity * cap);
  ts->rpt_x = pick_rpt((int64_t)h->cfg.nranks * cap);
  if (!rpt_ok(ts->rpt_leaf, Smax) || !rpt_ok(ts->rpt_node, Smax) || !rpt_ok(ts->rpt_x, Smax)) return PQR_EPLAN;
  int rc;
  if ((rc = dalloc(&ts->Vleaf, (size_t)h->ld * cap))) return rc;
  ts->p.assign(1, 0);
  ts->ldl.assign(1, 0);
  ts->Vn.assign(1, nullptr);
  ts->in.assign(1, nullptr);
  ts->dn.assign(1, nullptr);
  int pl = ts->p0;
  while (pl > 1) {
    pl = (pl + kArity - 1) / kArity;
    const int64_t rows = (int64_t)pl * kArity * cap;
    double *V = nullptr, *in = nullptr, *dn = nullptr;
    if ((rc = dalloc(&V, (size_t)rows * cap)) || (rc = dalloc(&in, (size_t)rows * sm)) ||
        (rc = dalloc(&dn, (size_t)rows * sm))) {
      cudaFree(V); cudaFree(in); cudaFree(dn);
      return rc;
    }
    CUDA_TRY(cudaMemsetAsync(in, 0, sizeof(double) * rows * sm, h->stream));
    ts->p.push_back(pl);
    ts->ldl.push_back(rows);
    ts->Vn.push_back(V);
    ts->in.push_back(in);
    ts->dn.push_back(dn);
  }
  ts->nlev = (int)ts->p.size() - 1;
  if ((rc = dalloc(&ts->in_top, (size_t)cap * sm))) return rc;
  CUDA_TRY(cudaMemsetAsync(ts->in_top, 0, sizeof(double) * cap * sm, h->stream));
  if ((rc = dalloc(&ts->Ut, (size_t)cap * std::max(sm, 16)))) return rc;
  if ((rc = dalloc(&ts->Rt, (size_t)cap * cap))) return rc;
  CUDA_TRY(cudaMemsetAsync(ts->Rt, 0, sizeof(double) * cap * cap, h->stream));
  if ((rc = dalloc(&ts->coef, (size_t)cap * 16))) return rc;
  if (h->cfg.nranks > 1) {
    const int64_t R = (int64_t)h->cfg.nranks * cap;
    if ((rc = dalloc(&ts->xraw, (size_t)R * std::max(sm, 16)))) return rc;
    if ((rc = dalloc(&ts->xin, (size_t)R * std::max(sm, 16)))) return rc;
    if ((rc = dalloc(&ts->Vx, (size_t)R * cap))) return rc;
    if ((rc = dalloc(&ts->xdn, (size_t)R * std::max(sm, 16)))) return rc;
    if ((rc = dalloc(&ts->Btop, (size_t)cap * std::max(sm, 16)))) return rc;
    CUDA_TRY(cudaMemsetAsync(ts->xin, 0, sizeof(double) * R * std::max(sm, 16), h->stream));
  } else {
    ts->Btop = ts->in_top;
  }
  h->st.block_rows = (int)ts->q0;
  h->st.tree_levels = ts->nlev;
  return PQR_OK;
}

// LOR build (§8(a) a9): one up-sweep per chunk of <= 16 columns of Q; the top
// coefficients of each chunk become R_top's columns (Q = L [R_top; 0]).
int tsqr_create(Ctx* h, const double* Q, int64_t ldq, int k) {
  h->ts = new TsqrState();
  TRY(tsqr_alloc(h));
  TsqrState* ts = h->ts;
  h->k = 0;
  ts->C = 0;
  // build chunks must also fit the in/dn buffers (s_max columns) -> chunk <= s_max when > 16? no:
  // buffers for node inputs are sized s_max; chunk must not exceed it.
  const int chunk = std::min(max_chunk(ts), h->cfg.s_max);
  for (int c0 = 0; c0 < k; c0 += chunk) {
    const int cs = std::min(chunk, k - c0);
    TRY(tsqr_up_sweep(h, Q + (int64_t)c0 * ldq, ldq, cs));
    TRY(run_top(h, cs, true, h->Pf, std::max(1, h->k), h->Nf, kSMax, h->ints + 2, h->ints + 3));
    TRY(tsqr_commit(h, cs, cs));
    h->k += cs;
  }
  return PQR_OK;
}

int tsqr_solve(Ctx* h, const double* X, int64_t ldx, int s, unsigned flags, double* Ud, int64_t ldud, bool append,
               int* t_host) {
  TsqrState* ts = h->ts;
  if (ts->C + s > ts->cap) return PQR_ECAPACITY;
  if (!rpt_ok(ts->rpt_leaf, pick_S(s))) return PQR_EPLAN;
  TRY(tsqr_up_sweep(h, X, ldx, s));
  TRY(run_top(h, s, false, h->Pf, std::max(1, h->k), h->Nf, kSMax, h->ints + 2, h->ints + 3));
  TRY(tsqr_down_sweep(h, ts->C + s, ts->Ut, s, s, Ud, ldud));
  // U~ columns >= t are zero, so the down sweep writes zeros there.
  CUDA_TRY(cudaMemcpyAsync(h->h_ints, h->ints, sizeof(int) * 8, cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  const int t = h->h_ints[2];
  *t_host = t;
  if ((flags & PQR_NO_DEFLATION) && h->h_ints[3] > 0) return PQR_EBREAKDOWN;
  if (append) TRY(tsqr_commit(h, s, t));
  return PQR_OK;
}

// Y = Q C = L [R_top C; 0]: coef = R_top C (small update-kernel product), then stage 2.
int tsqr_apply(Ctx* h, const double* C, int ldc, int m, double* Y, int64_t ldy) {
  TsqrState* ts = h->ts;
  const int k = h->k;
  const bool stage = is_host_ptr(Y) || (ldy & 1) || !aligned16(Y);
  if (stage && !h->stageU && dalloc(&h->stageU, (size_t)h->ld * h->cfg.s_max)) return PQR_ENOMEM;
  if (!h->stageC && dalloc(&h->stageC, (size_t)h->cap * 16)) return PQR_ENOMEM;
  int chunk = std::min(max_chunk(ts), h->cfg.s_max);
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
      TRY(tsqr_down_sweep(h, ts->C, ts->coef, mc, mc, dst, ldd));
    }
    if (stage)
      CUDA_TRY(cudaMemcpy2DAsync(Y + (int64_t)c0 * ldy, ldy * sizeof(double), h->stageU, h->ld * sizeof(double),
                                 h->cfg.n_local * sizeof(double), mc, cudaMemcpyDefault, h->stream));
  }
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  prof_collect(h);
  return PQR_OK;
}

void tsqr_free(Ctx* h) {
  TsqrState* ts = h->ts;
  if (!ts) return;
  cudaFree(ts->Vleaf);
  for (size_t i = 1; i < ts->Vn.size(); ++i) {
    cudaFree(ts->Vn[i]);
    cudaFree(ts->in[i]);
    cudaFree(ts->dn[i]);
  }
  cudaFree(ts->in_top);
  cudaFree(ts->xraw);
  cudaFree(ts->xin);
  cudaFree(ts->Vx);
  cudaFree(ts->xdn);
  if (ts->Btop != ts->in_top) cudaFree(ts->Btop);
  cudaFree(ts->Ut);
  cudaFree(ts->Rt);
  cudaFree(ts->coef);
  delete ts;
  h->ts = nullptr;
}

}  // namespace
