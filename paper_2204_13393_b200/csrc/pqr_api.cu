// pqr_api.cu — the C-ABI of libpqr.so (include/pqr.h): handle, plans, the
// CholQR2 (BCGS-PIP+) orchestration, the TSQR orchestration (tsqr_api.cuh),
// NCCL plumbing and step-level entry points (include/pqr_steps.h).
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <vector>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "../../include/pqr.h"
#include "../../include/pqr_steps.h"
#include "../../include/pqr_support.h"
#include "cholqr_kernels.cuh"
#include "tsqr_kernels.cuh"
#include "tsqr_wy.cuh"
#include "stream_kernels.cuh"
#include "stream2_kernels.cuh"
#include "small_kernels.cuh"
#include "support_kernels.cuh"
#include "exchange.cuh"
#include "lsa_exchange.cuh"

using namespace pqr;

namespace {

constexpr int kThreads = 256;

struct Ctx;
int tsqr_create(Ctx* h, const double* Q, int64_t ldq, int k);
int tsqr_solve(Ctx* h, const double* X, int64_t ldx, int s, unsigned flags, double* Ud, int64_t ldud,
               bool append, int* t_host);
int tsqr_apply(Ctx* h, const double* C, int ldc, int m, double* Y, int64_t ldy);
void tsqr_free(Ctx* h);

#define CUDA_TRY(x)                                   \
  do {                                                \
    cudaError_t e_ = (x);                             \
    if (e_ != cudaSuccess) {                          \
      fprintf(stderr, "[pqr] CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      return PQR_ECUDA;                               \
    }                                                 \
  } while (0)
#define NCCL_TRY(x)                                   \
  do {                                                \
    ncclResult_t r_ = (x);                            \
    if (r_ != ncclSuccess) {                          \
      fprintf(stderr, "[pqr] NCCL error %s at %s:%d\n", ncclGetErrorString(r_), __FILE__, __LINE__); \
      return PQR_ENCCL;                               \
    }                                                 \
  } while (0)
#define TRY(x)                   \
  do {                           \
    int rc_ = (x);               \
    if (rc_ != PQR_OK) return rc_; \
  } while (0)

struct TsqrState;  // defined in tsqr_api.cuh

// Host-buffer pipeline (pqr_project_normalize with host X and U, one rank): X goes up and U
// comes back in row chunks on a second stream, each chunk's copy overlapped with the kernels
// of the other chunks (the first and the last pass are launched per chunk).
constexpr int kHostChunksMax = 16;
struct HostPipe {
  int nch = 0;                          // chunks of this call (0: not pipelined)
  int64_t r[kHostChunksMax + 1] = {};   // row boundaries
  int64_t b[kHostChunksMax + 1] = {};   // TSQR leaf-block boundaries (rows r[c] = start of block b[c])
  const double* Xh = nullptr; int64_t ldxh = 0;
  double* Uh = nullptr; int64_t lduh = 0;
};

// A call's arguments: repeated calls with the same key (device buffers, PQR_NO_APPEND, one rank)
// replay a CUDA graph captured from the second such call (no per-kernel host launch cost).
struct GraphKey {
  const void* X = nullptr; int64_t ldx = 0; int s = 0; unsigned flags = 0;
  const void* U = nullptr; int64_t ldu = 0; const void* P = nullptr; int ldp = 0;
  const void* N = nullptr; int ldn = 0; int k = -1;
  bool operator==(const GraphKey& o) const {
    return X == o.X && ldx == o.ldx && s == o.s && flags == o.flags && U == o.U && ldu == o.ldu && P == o.P &&
           ldp == o.ldp && N == o.N && ldn == o.ldn && k == o.k;
  }
};

struct Ctx {
  pqr_config cfg{};
  cudaStream_t stream = nullptr;
  int sms = 148;
  int k = 0;
  int cap = 0;           // k_max + s_max
  int64_t ld = 0;        // leading dimension of the explicit basis / staging buffers
  double* basis = nullptr;  // CHOLQR2: explicit basis, n_local x cap
  // CholQR2 workspaces
  double* partials = nullptr;
  int64_t partials_elems = 0;
  unsigned int* ticket = nullptr;
  double* Wloc = nullptr;   // m x s, compact (ld m) - this rank's Gram
  double* Wall = nullptr;   // nranks x (m*s)
  double *P1 = nullptr, *N1 = nullptr, *M1 = nullptr, *P2 = nullptr, *N2 = nullptr, *M2 = nullptr;
  double *Pf = nullptr, *Nf = nullptr;
  int* ints = nullptr;      // [0] t1 [1] t2 [2] tf [3] defl1 [4] defl2 [16..] piv1 [32..] piv2
  int* h_ints = nullptr;    // pinned host mirror
  int* d_hints = nullptr;   // device view of h_ints (mapped pinned memory: kernels write t directly)
  // the caller's device P / N of the current call (nullptr: host or absent); a kernel that writes
  // them itself sets outs_written so the call enqueues no output copies
  double* outP = nullptr; int outldp = 0; double* outN = nullptr; int outldn = 0;
  bool outs_written = false;
  double* stageX = nullptr;  // n x s_max staging for host X
  double* stageU = nullptr;  // n x s_max staging for host U / internal U1
  double* stageC = nullptr;  // cap x 16 staging for host C
  HostPipe hp;
  cudaStream_t cstream = nullptr;  // copy stream of the host-buffer pipeline (created on first use)
  cudaEvent_t hp_in[kHostChunksMax] = {}, hp_out[kHostChunksMax] = {}, hp_done = nullptr;
  double* Wchunks = nullptr;       // kHostChunksMax x (cap x s_max): per-chunk Grams of the first pass
  Exchange* xc = nullptr;          // cross-rank exchange (nranks > 1, PQR_FORCE_NCCL or a virtual group)
  int device = 0;                  // the handle's CUDA device (made current at every entry point)
  pqr_stats st{};
  TsqrState* ts = nullptr;
  // CUDA-graph replay of repeated calls (GraphKey)
  GraphKey gcand{}, gkey{};
  cudaGraphExec_t gexec = nullptr;
  cudaStream_t gstream = nullptr;  // capture/replay stream when the handle's stream is the legacy
                                   // default stream (which cannot be captured)
  cudaEvent_t gev = nullptr;
  int64_t g_launches = 0;  // kernels per replay
  // profiling (pqr_profile_enable)
  bool prof = false;
  pqr_profile prof_tot{};
  std::vector<cudaEvent_t> ev_pool;
  struct Pending { int kind; cudaEvent_t a, b; };
  std::vector<Pending> pending;
};

struct ProfScope {
  Ctx* h;
  int kind;
  cudaEvent_t a = nullptr;
  ProfScope(Ctx* h_, int kind_) : h(h_), kind(kind_) {
    if (!h->prof) return;
    a = get_event();
    cudaEventRecord(a, h->stream);
  }
  ~ProfScope() {
    if (!h->prof || !a) return;
    cudaEvent_t b = get_event();
    cudaEventRecord(b, h->stream);
    h->pending.push_back({kind, a, b});
  }
  cudaEvent_t get_event() {
    if (!h->ev_pool.empty()) {
      cudaEvent_t e = h->ev_pool.back();
      h->ev_pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
};
#define PQR_CAT2(a, b) a##b
#define PQR_CAT(a, b) PQR_CAT2(a, b)
#define PROF(h, kind) ProfScope PQR_CAT(prof_scope_, __LINE__)((h), (kind))

void prof_collect(Ctx* h) {
  for (auto& p : h->pending) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) {
      h->prof_tot.ms[p.kind] += ms;
      h->prof_tot.launches[p.kind] += 1;
    } else {
      cudaGetLastError();
    }
    h->ev_pool.push_back(p.a);
    h->ev_pool.push_back(p.b);
  }
  h->pending.clear();
}

bool is_host_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes at;
  cudaError_t e = cudaPointerGetAttributes(&at, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return at.type == cudaMemoryTypeHost || at.type == cudaMemoryTypeUnregistered;
}

// makes the handle's device current for the duration of a C-ABI call (a handle may be driven
// from any host thread; a new thread starts on device 0) and restores the caller's device
struct DevGuard {
  int prev = -1;
  explicit DevGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) {
      cudaGetLastError();
      prev = -1;
    }
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DevGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

template <typename T>
int dalloc(T** p, size_t count) {
  if (count == 0) count = 1;
  if (cudaMalloc(reinterpret_cast<void**>(p), count * sizeof(T)) != cudaSuccess) {
    cudaGetLastError();
    return PQR_ENOMEM;
  }
  return PQR_OK;
}

// ---- host-buffer pipeline helpers (HostPipe) ----
int hp_wait_in(Ctx* h, int c) {
  CUDA_TRY(cudaStreamWaitEvent(h->stream, h->hp_in[c], 0));
  return PQR_OK;
}
// U rows of chunk c (device Ud, ld ldud; ncol columns) to the caller's host U once the stream
// has produced them
int hp_d2h_chunk(Ctx* h, int c, const double* Ud, int64_t ldud, int ncol) {
  HostPipe& p = h->hp;
  CUDA_TRY(cudaEventRecord(h->hp_out[c], h->stream));
  CUDA_TRY(cudaStreamWaitEvent(h->cstream, h->hp_out[c], 0));
  const int64_t r0 = p.r[c], rows = p.r[c + 1] - p.r[c];
  if (rows > 0)
    CUDA_TRY(cudaMemcpy2DAsync(p.Uh + r0, p.lduh * sizeof(double), Ud + r0, ldud * sizeof(double),
                               rows * sizeof(double), ncol, cudaMemcpyDeviceToHost, h->cstream));
  return PQR_OK;
}
// the call's stream waits for the copy stream (the caller's one synchronisation covers both)
int hp_finish(Ctx* h) {
  if (h->hp.nch == 0) return PQR_OK;
  CUDA_TRY(cudaEventRecord(h->hp_done, h->cstream));
  CUDA_TRY(cudaStreamWaitEvent(h->stream, h->hp_done, 0));
  return PQR_OK;
}
// Decide the chunking and enqueue the chunked X upload into stageX.  Chunk count: PQR_HOST_CHUNKS
// (default 8 from 2^18 rows; 0 or 1 disables), rows per chunk a multiple of 64 (CholQR2) or whole leaf
// blocks (TSQR, `bounds` = leaf-block start rows, nb + 1 entries).
int hp_plan_upload(Ctx* h, const double* X, int64_t ldx, int s, double* U, int64_t ldu,
                   const std::vector<int64_t>* bounds) {
  HostPipe& p = h->hp;
  p.nch = 0;
  const char* env = getenv("PQR_HOST_CHUNKS");  // read per call (tests switch it)
  const int want = std::min(env ? atoi(env) : 8, kHostChunksMax);
  const int64_t n = h->cfg.n_local;
  // by default only problems large enough for the copies to dominate (>= 2^18 rows)
  if (want < 2 || n < (env ? (int64_t)64 * want : (int64_t)1 << 18)) return PQR_OK;
  if (!h->cstream) {
    CUDA_TRY(cudaStreamCreateWithFlags(&h->cstream, cudaStreamNonBlocking));
    for (int c = 0; c < kHostChunksMax; ++c) {
      CUDA_TRY(cudaEventCreateWithFlags(&h->hp_in[c], cudaEventDisableTiming));
      CUDA_TRY(cudaEventCreateWithFlags(&h->hp_out[c], cudaEventDisableTiming));
    }
    CUDA_TRY(cudaEventCreateWithFlags(&h->hp_done, cudaEventDisableTiming));
  }
  int nch = want;
  if (bounds) {
    const int64_t nb = (int64_t)bounds->size() - 1;
    nch = (int)std::min<int64_t>(nch, nb);
    for (int c = 0; c <= nch; ++c) {
      p.b[c] = nb * c / nch;
      p.r[c] = (*bounds)[p.b[c]];
    }
  } else {
    const int64_t step = ((n + nch - 1) / nch + 63) / 64 * 64;
    for (int c = 0; c <= nch; ++c) p.r[c] = std::min<int64_t>(n, (int64_t)c * step);
  }
  p.nch = nch;
  p.Xh = X; p.ldxh = ldx; p.Uh = U; p.lduh = ldu;
  // the copy stream may only overwrite stageX once earlier work on the call's stream is done
  CUDA_TRY(cudaEventRecord(h->hp_done, h->stream));
  CUDA_TRY(cudaStreamWaitEvent(h->cstream, h->hp_done, 0));
  for (int c = 0; c < nch; ++c) {
    const int64_t r0 = p.r[c], rows = p.r[c + 1] - p.r[c];
    if (rows > 0)
      CUDA_TRY(cudaMemcpy2DAsync(h->stageX + r0, h->ld * sizeof(double), X + r0, ldx * sizeof(double),
                                 rows * sizeof(double), s, cudaMemcpyHostToDevice, h->cstream));
    CUDA_TRY(cudaEventRecord(h->hp_in[c], h->cstream));
  }
  return PQR_OK;
}

// ---------------------------------------------------------------------------
// kernel launchers (shared by the handle path and the step entry points)
// ---------------------------------------------------------------------------
int grid_cap(int sms) { return sms * 4; }

struct GramPlan {
  int G, MTW, NT, grid;
  int64_t rows_per_cta;
  size_t smem;
};

GramPlan plan_gram(int64_t n, int k, int s, int sms) {
  GramPlan p{};
  const int m = k + s;
  const int MT = (m + 7) / 8;
  p.NT = s > 8 ? 2 : 1;
  p.G = 1;
  while ((MT + p.G - 1) / p.G > 6) p.G *= 2;
  p.MTW = (MT + p.G - 1) / p.G;
  const int RW = 8 / p.G;
  const int64_t min_rows = 8 * RW * 4;
  int64_t target = (n + grid_cap(sms) - 1) / grid_cap(sms);
  target = ((target + 7) / 8) * 8;
  p.rows_per_cta = std::max<int64_t>(min_rows, target);
  p.grid = (int)std::max<int64_t>(1, (n + p.rows_per_cta - 1) / p.rows_per_cta);
  p.smem = (size_t)8 * p.MTW * p.NT * 64 * sizeof(double);
  return p;
}

template <int MTW, int NT>
cudaError_t launch_gram_t(const GramPlan& p, const GramArgs& a, bool vec, cudaStream_t st) {
  // (always raise the limit: 48 KB of dynamic plus the kernel's static shared memory is
  // already over the default)
  if (vec) {
    auto f = k_gram<MTW, NT, true>;
    ensure_smem(f, p.smem);
    f<<<p.grid, kThreads, p.smem, st>>>(a);
  } else {
    auto f = k_gram<MTW, NT, false>;
    ensure_smem(f, p.smem);
    f<<<p.grid, kThreads, p.smem, st>>>(a);
  }
  return cudaGetLastError();
}

template <int NT>
cudaError_t launch_gram_mtw(const GramPlan& p, const GramArgs& a, bool vec, cudaStream_t st) {
  switch (p.MTW) {
    case 1: return launch_gram_t<1, NT>(p, a, vec, st);
    case 2: return launch_gram_t<2, NT>(p, a, vec, st);
    case 3: return launch_gram_t<3, NT>(p, a, vec, st);
    case 4: return launch_gram_t<4, NT>(p, a, vec, st);
    case 5: return launch_gram_t<5, NT>(p, a, vec, st);
    default: return launch_gram_t<6, NT>(p, a, vec, st);
  }
}

constexpr int kSmemBudget = 225 * 1024;
int run_s2(int mode, const S2Args& a0, int sms, cudaStream_t st, int64_t* launches);

template <int MTH, int NT, int RB>
cudaError_t launch_gram_cpa_t(int grid, size_t smem, const GramCpaArgs& a, cudaStream_t st) {
  auto f = k_gram_cpa<MTH, NT, RB>;
  ensure_smem(f, smem);
  f<<<grid, kCpaThreads, smem, st>>>(a);
  return cudaGetLastError();
}

// W (ld ldw) = [Q X]^T X over n rows.  partials must hold max(grid)*m*s doubles.
int run_gram(int64_t n, int k, int s, const double* Q, int64_t ldq, const double* X, int64_t ldx,
             double* W, int ldw, double* partials, unsigned int* ticket, int sms, cudaStream_t st,
             int64_t* launches) {
  static const bool s2g = getenv("PQR_S2_GRAM") && atoi(getenv("PQR_S2_GRAM")) != 0;
  if (s2g) {
    S2Args b{};
    b.Q = Q; b.ldq = ldq; b.X = X; b.ldx = ldx; b.n = n; b.k = k; b.sx = s; b.sout = 0;
    b.partials = partials; b.W = W; b.ldw = ldw; b.ticket = ticket;
    const int rc = run_s2(kS2Gram, b, sms, st, launches);
    if (rc != PQR_EPLAN) return rc;
  }
  const bool vec = (k == 0 || ((ldq & 1) == 0 && aligned16(Q))) && (ldx & 1) == 0 && aligned16(X);
  static const int env_rb = getenv("PQR_GRAM_RB") ? atoi(getenv("PQR_GRAM_RB")) : 32;
  // two CTAs per SM (two stages each) beat one CTA with five stages for wide [Q X] (weak
  // config -1.5 %, config D -5 %), one CTA is faster at m = 72 (config S); PQR_GRAM_CTAS forces
  static const int env_ctas = getenv("PQR_GRAM_CTAS") ? atoi(getenv("PQR_GRAM_CTAS")) : 0;
  const int RB = env_rb == 32 ? 32 : 16;
  const int groups = kCpaWarps / (RB / 8);
  const int m = k + s, MT = (m + 7) / 8, MTH = (MT + groups - 1) / groups, NT = s > 8 ? 2 : 1;
  const int ctas = env_ctas == 1 ? 1 : env_ctas == 2 ? 2 : (m >= 100 ? 2 : 1);
  const size_t stage_bytes = (size_t)MT * 8 * (RB + 8) * sizeof(double);
  const size_t red_bytes = (size_t)kCpaWarps * MTH * NT * 64 * sizeof(double);
  const size_t budget = ctas == 2 ? kSmemBudget / 2 - 2048 : kSmemBudget;
  int NS = (int)std::min<size_t>(8, budget / (stage_bytes + 16));
  while (NS >= 2 && (size_t)NS * stage_bytes < red_bytes) ++NS;
  const size_t smem = std::max((size_t)NS * stage_bytes, red_bytes) + 2 * NS * sizeof(uint64_t);
  cudaError_t e;
  if (vec && MTH <= 10 && NS >= (ctas == 2 ? 2 : 3) && smem <= budget) {
    GramCpaArgs a{};
    a.Q = Q; a.ldq = ldq; a.X = X; a.ldx = ldx; a.n = n; a.k = k; a.s = s; a.NS = NS;
    a.partials = partials; a.W = W; a.ldw = ldw; a.ticket = ticket;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)sms * ctas, (n + RB - 1) / RB));
#define PQR_GRAM_CASE(H)                                                                                    \
  case H * 100 + 10 + 1: e = launch_gram_cpa_t<H, 1, 16>(grid, smem, a, st); break;                       \
  case H * 100 + 10 + 2: e = launch_gram_cpa_t<H, 2, 16>(grid, smem, a, st); break;                       \
  case H * 100 + 20 + 1: e = launch_gram_cpa_t<H, 1, 32>(grid, smem, a, st); break;                       \
  case H * 100 + 20 + 2: e = launch_gram_cpa_t<H, 2, 32>(grid, smem, a, st); break;
    switch (MTH * 100 + (RB / 16) * 10 + NT) {
      PQR_GRAM_CASE(1) PQR_GRAM_CASE(2) PQR_GRAM_CASE(3) PQR_GRAM_CASE(4) PQR_GRAM_CASE(5)
      PQR_GRAM_CASE(6) PQR_GRAM_CASE(7) PQR_GRAM_CASE(8) PQR_GRAM_CASE(9) PQR_GRAM_CASE(10)
      default: e = cudaErrorInvalidValue; break;
    }
#undef PQR_GRAM_CASE
  } else {
    const GramPlan p = plan_gram(n, k, s, sms);
    GramArgs a{};
    a.Q = Q; a.ldq = ldq; a.X = X; a.ldx = ldx; a.n = n; a.k = k; a.s = s;
    a.G = p.G; a.rows_per_cta = p.rows_per_cta; a.partials = partials; a.W = W; a.ldw = ldw; a.ticket = ticket;
    e = p.NT == 1 ? launch_gram_mtw<1>(p, a, vec, st) : launch_gram_mtw<2>(p, a, vec, st);
  }
  if (launches) ++*launches;
  if (e != cudaSuccess) {
    fprintf(stderr, "[pqr] gram launch: %s\n", cudaGetErrorString(e));
    return PQR_ECUDA;
  }
  return PQR_OK;
}

int64_t gram_partials_needed(int64_t n, int k, int s, int sms) {
  const GramPlan p = plan_gram(n, k, s, sms);
  return (int64_t)std::max(p.grid, 2 * sms) * (k + s) * s;
}

// U (cols < sout) = [Q X] M, optionally also into U2 (cols < t).
int run_update(int64_t n, int k, const double* Q, int64_t ldq, int sx, const double* X, int64_t ldx,
               const double* M, int ldm, int sout, const int* t_dev, double* U, int64_t ldu,
               double* U2, int64_t ldu2, int sms, cudaStream_t st, int64_t* launches) {
  if (n <= 0 || sout <= 0) return PQR_OK;
  static const bool s2u = getenv("PQR_S2_UPD") && atoi(getenv("PQR_S2_UPD")) != 0;
  if (s2u) {
    S2Args b{};
    b.Q = Q; b.ldq = ldq; b.X = X; b.ldx = ldx; b.n = n; b.k = k; b.sx = sx; b.sout = sout;
    b.M = M; b.ldm = ldm; b.t_dev = t_dev; b.U = U; b.ldu = ldu; b.U2 = U2; b.ldu2 = ldu2;
    const int rc = run_s2(kS2Update, b, sms, st, launches);
    if (rc != PQR_EPLAN) return rc;
  }
  UpdateArgs a{};
  a.Q = Q; a.ldq = ldq; a.X = X; a.ldx = ldx; a.n = n; a.k = k; a.sx = sx; a.sout = sout;
  a.M = M; a.ldm = ldm; a.t_dev = t_dev; a.U = U; a.ldu = ldu; a.U2 = U2; a.ldu2 = ldu2;
  const int m = k + sx;
  const int NT = sout > 8 ? 2 : 1;
  const int mpad = ((m + 3) / 4) * 4;
  const size_t smem = (size_t)NT * mpad * 8 * sizeof(double);
  const bool vec = (k == 0 || ((ldq & 1) == 0 && aligned16(Q))) && (sx == 0 || ((ldx & 1) == 0 && aligned16(X))) &&
                   (ldu & 1) == 0 && aligned16(U);
  const int64_t nslab = (n + 15) / 16;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)sms * 6, (nslab + 7) / 8));
  // column chunk of the stages: 32 from m = 128 (weak config: 6.28 -> 6.14 ms), else 16
  // (k = 64: 16 is faster); PQR_UPD_CW forces
  static const int env_cw = getenv("PQR_UPD_CW") ? atoi(getenv("PQR_UPD_CW")) : 0;
  static const int env_ctas = getenv("PQR_UPD_CTAS") ? atoi(getenv("PQR_UPD_CTAS")) : 2;
  const int CW = env_cw == 16 ? 16 : env_cw == 32 ? 32 : (m >= 128 ? 32 : 16);
  const int ctas = env_ctas == 2 ? 2 : 1;
  const int nch = (m + CW - 1) / CW;
  const size_t smM = (size_t)NT * nch * CW * 8 * sizeof(double);
  const size_t stg = (size_t)CW * kUpdRBP * sizeof(double);
  const size_t budget = ctas == 2 ? kSmemBudget / 2 - 2048 : kSmemBudget;
  const int NS = smM + 3 * stg < budget ? (int)std::min<size_t>(12, (budget - smM) / (stg + 16)) : 0;
  const bool cpa_ok = vec && NS >= 3 && (sx == 0 || ((ldx & 1) == 0 && aligned16(X)));
  if (cpa_ok) {
    UpdCpaArgs b{};
    b.Q = Q; b.ldq = ldq; b.X = X; b.ldx = ldx; b.n = n; b.k = k; b.sx = sx; b.sout = sout;
    b.M = M; b.ldm = ldm; b.t_dev = t_dev; b.U = U; b.ldu = ldu; b.U2 = U2; b.ldu2 = ldu2; b.NS = NS;
    const size_t sm2 = smM + NS * stg + 2 * NS * sizeof(uint64_t);
    const int g2 = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)sms * ctas, (n + kUpdRB - 1) / kUpdRB));
    auto go = [&](auto kern) {
      ensure_smem(kern, sm2);
      kern<<<g2, kCpaThreads, sm2, st>>>(b);
    };
    if (NT == 1) {
      if (CW == 16) go(k_update_cpa<1, 16>); else go(k_update_cpa<1, 32>);
    } else {
      if (CW == 16) go(k_update_cpa<2, 16>); else go(k_update_cpa<2, 32>);
    }
  } else if (NT == 1) {
    if (vec) k_update<1, true><<<grid, kThreads, smem, st>>>(a);
    else k_update<1, false><<<grid, kThreads, smem, st>>>(a);
  } else {
    if (vec) k_update<2, true><<<grid, kThreads, smem, st>>>(a);
    else k_update<2, false><<<grid, kThreads, smem, st>>>(a);
  }
  cudaError_t e = cudaGetLastError();
  if (launches) ++*launches;
  if (e != cudaSuccess) {
    fprintf(stderr, "[pqr] update launch: %s\n", cudaGetErrorString(e));
    return PQR_ECUDA;
  }
  return PQR_OK;
}

// nparts < 0: the Grams cross the ranks inside the factor kernel (NCCL device API, lsa)
int run_factor(const FactorArgs& a, cudaStream_t st, int64_t* launches, const LsaArgs* lsa = nullptr) {
  if (a.nparts < 0) {
    if (!lsa) return PQR_EARG;
    k_factor_lsa<<<1, kThreads, 0, st>>>(a, *lsa);
  } else {
    k_factor<<<1, kThreads, 0, st>>>(a);
  }
  if (launches) ++*launches;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    fprintf(stderr, "[pqr] factor launch: %s\n", cudaGetErrorString(e));
    return PQR_ECUDA;
  }
  return PQR_OK;
}

// Producer-free warp-unit streaming kernels (stream2_kernels.cuh).  mode: kS2Fused (default for
// the fused pass; PQR_S2=0 disables), kS2Gram / kS2Update (PQR_S2_GRAM=1 / PQR_S2_UPD=1).
// Returns PQR_EPLAN when no instantiation fits (the caller uses the stream_kernels.cuh kernels).
int run_s2(int mode, const S2Args& a0, int sms, cudaStream_t st, int64_t* launches) {
  const int MT = (a0.k + a0.sx + 7) / 8;
  const int NT = (mode == kS2Gram ? a0.sx : a0.sout) > 8 ? 2 : 1;
  if (MT > 20) return PQR_EPLAN;
  const bool vec = (a0.k == 0 || ((a0.ldq & 1) == 0 && aligned16(a0.Q))) &&
                   (a0.sx == 0 || ((a0.ldx & 1) == 0 && aligned16(a0.X))) &&
                   (mode == kS2Gram || ((a0.ldu & 1) == 0 && aligned16(a0.U))) &&
                   (!a0.U2 || ((a0.ldu2 & 1) == 0 && aligned16(a0.U2)));
  if (!vec) return PQR_EPLAN;
  S2Args a = a0;
  // warp-specialised fused pass (a producer warpgroup issues the slot copies): faster with two
  // output tiles (config D, s = 16: 1.10 -> 1.00 ms), slower with one (weak config: 8.3-8.4 ->
  // 8.8-8.9 ms; configs[1]: 1.99 -> 2.21 ms; tools/ws_ab.sh); PQR_S2_WS=0|1 forces
  static const int env_ws = getenv("PQR_S2_WS") ? atoi(getenv("PQR_S2_WS")) : -1;
  a.ws = mode == kS2Fused && (env_ws >= 0 ? env_ws > 0 : NT == 2) ? 1 : 0;
  a.nslot = s2_nslot(MT, NT, mode, kSmemBudget, a.ws != 0);
  // slot cap: with 17 one-tile columns groups (weak config) 12 slots beat the 13 that fit
  // (fused pass 8.30-8.42 -> 7.82-7.99 ms, 3 interleaved pairs; 10 and 11: 7.85 / 7.97), while
  // configs[1] (MT = 9) wants all 24 (12: 1.97 -> 2.04 ms; tools/nsl_ab.sh).  PQR_S2_NSL caps (A/B)
  static const int env_nsl = getenv("PQR_S2_NSL") ? atoi(getenv("PQR_S2_NSL")) : -1;
  const int cap = env_nsl >= 0 ? env_nsl : (mode == kS2Fused && NT == 1 && MT >= 16 && !a.ws ? 12 : 0);
  if (cap > 0) a.nslot = std::min(a.nslot, cap);
  // refill copies interleaved with the G phase: faster up to 12 tiles (config S: 2.14 -> 1.95 ms),
  // slower at 17 (weak config: 7.7 -> 9.3 ms), so the kernel compiles it out past
  // kS2InterleaveMaxMT tiles; PQR_S2_IL=0 disables it below
  static const int env_il = getenv("PQR_S2_IL") ? atoi(getenv("PQR_S2_IL")) : -1;
  static const int env_pf = getenv("PQR_S2_PF") ? atoi(getenv("PQR_S2_PF")) : 0;
  a.interleave = MT <= kS2InterleaveMaxMT && (env_il >= 0 ? env_il != 0 : true) ? 1 : 0;
  a.pf_rounds = env_pf;
  if (a.nslot < kS2Consumers + 1) return PQR_EPLAN;
  const int64_t nunits = (a.n + kS2Rows - 1) / kS2Rows;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(sms, nunits));
  cudaError_t e = mode == kS2Fused ? pqr_launch_s2_fused(a, grid, st)
                  : mode == kS2Gram ? pqr_launch_s2_gram(a, grid, st)
                                    : pqr_launch_s2_update(a, grid, st);
  if (e == cudaErrorNotSupported) return PQR_EPLAN;
  if (launches) ++*launches;
  if (e != cudaSuccess) {
    fprintf(stderr, "[pqr] stream2 launch (mode %d): %s\n", mode, cudaGetErrorString(e));
    return PQR_ECUDA;
  }
  return PQR_OK;
}

// Fused second CholQR pass: U1 = [Q X] M1 (into U1) and W2 = [Q U1]^T U1 (into W).
// Returns PQR_EPLAN when the fused kernel cannot be used (caller falls back).
template <int MTH, int NT>
cudaError_t launch_update_gram_t(int grid, size_t smem, const UpdGramArgs& a, cudaStream_t st) {
  auto f = k_update_gram_cpa<MTH, NT>;
  ensure_smem(f, smem);
  f<<<grid, kCpaThreads, smem, st>>>(a);
  return cudaGetLastError();
}

int run_update_gram(int64_t n, int k, int s, const double* Q, int64_t ldq, const double* X, int64_t ldx,
                    const double* M, int ldm, const int* t_dev, double* U1, int64_t ldu, double* W, int ldw,
                    double* partials, unsigned int* ticket, int sms, cudaStream_t st, int64_t* launches) {
  static const bool disabled = getenv("PQR_NO_FUSE") != nullptr;
  static const bool s2 = !(getenv("PQR_S2") && atoi(getenv("PQR_S2")) == 0);
  if (!disabled && s2) {
    S2Args b{};
    b.Q = Q; b.ldq = ldq; b.X = X; b.ldx = ldx; b.n = n; b.k = k; b.sx = s; b.sout = s;
    b.M = M; b.ldm = ldm; b.t_dev = t_dev; b.U = U1; b.ldu = ldu;
    b.partials = partials; b.W = W; b.ldw = ldw; b.ticket = ticket;
    const int rc = run_s2(kS2Fused, b, sms, st, launches);
    if (rc != PQR_EPLAN) return rc;
  }
  const bool vec = (k == 0 || ((ldq & 1) == 0 && aligned16(Q))) && (ldx & 1) == 0 && aligned16(X) &&
                   (ldu & 1) == 0 && aligned16(U1);
  const int m = k + s, MT = (m + 7) / 8, MTH = (MT + 1) / 2, NT = s > 8 ? 2 : 1;
  const int KS = (m + 3) / 4, mpad = KS * 4;
  const size_t stage_bytes = (size_t)MT * 8 * kFuseRBP * sizeof(double);
  const size_t extra = ((size_t)NT * mpad * 8 + 8 * NT * kFuseRBP + kCpaWarps * NT * 128) * sizeof(double);
  const size_t red_bytes = (size_t)kCpaWarps * MTH * NT * 64 * sizeof(double);
  static const int env_ctas = getenv("PQR_FUSE_CTAS") ? atoi(getenv("PQR_FUSE_CTAS")) : 2;
  const int ctas = (env_ctas == 1 || NT > 1) ? 1 : 2;
  const size_t budget = ctas == 2 ? kSmemBudget / 2 - 2048 : kSmemBudget;
  int NS = budget > extra ? (int)std::min<size_t>(8, (budget - extra) / (stage_bytes + 16)) : 0;
  while (NS >= 2 && (size_t)NS * stage_bytes < red_bytes) ++NS;
  const size_t smem = std::max((size_t)NS * stage_bytes, red_bytes) + extra + 2 * NS * sizeof(uint64_t);
  if (disabled || !vec || MTH > 10 || NS < 2 || smem > budget) return PQR_EPLAN;
  UpdGramArgs a{};
  a.Q = Q; a.ldq = ldq; a.X = X; a.ldx = ldx; a.n = n; a.k = k; a.s = s; a.NS = NS;
  a.M = M; a.ldm = ldm; a.t_dev = t_dev; a.U1 = U1; a.ldu = ldu;
  a.partials = partials; a.W = W; a.ldw = ldw; a.ticket = ticket;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)sms * ctas, (n + kFuseRB - 1) / kFuseRB));
  cudaError_t e;
#define PQR_FUSE_CASE(H)                                                                    \
  case H * 10 + 1: e = launch_update_gram_t<H, 1>(grid, smem, a, st); break;               \
  case H * 10 + 2: e = launch_update_gram_t<H, 2>(grid, smem, a, st); break;
  switch (MTH * 10 + NT) {
    PQR_FUSE_CASE(1) PQR_FUSE_CASE(2) PQR_FUSE_CASE(3) PQR_FUSE_CASE(4) PQR_FUSE_CASE(5)
    PQR_FUSE_CASE(6) PQR_FUSE_CASE(7) PQR_FUSE_CASE(8) PQR_FUSE_CASE(9) PQR_FUSE_CASE(10)
    default: return PQR_EPLAN;
  }
#undef PQR_FUSE_CASE
  if (launches) ++*launches;
  if (e != cudaSuccess) {
    fprintf(stderr, "[pqr] update+gram launch: %s\n", cudaGetErrorString(e));
    return PQR_ECUDA;
  }
  return PQR_OK;
}

// Gram of this rank, then (nranks > 1) allgather so every rank sums all ranks'
// partial Grams in rank order inside k_factor (bitwise identical replicas).
int exchange(Ctx* h, int m, int s, const double** Wsum, int* nparts);
// The basis a CholQR2 solve works on: the handle's explicit basis (CholQR2 variant), or a TSQR
// handle's top coordinates R_g with the GPU root's block (TSQR with reduction = PIP+).
struct BasisView {
  const double* Q; int64_t ldq; int64_t n;
  int k = -1;          // basis columns (-1: the handle's k)
  bool local = false;  // this rank alone: no cross-rank exchange, deflation only of non-positive
                       // pivots (a TSQR local problem never drops columns, reading R4)
  bool user_out = false;  // the call's own solve: kernels may write the caller's P / N directly
};

int gram_and_exchange(Ctx* h, const BasisView& bv, int k, int s, const double* X, int64_t ldx, const double** Wsum,
                      int* nparts) {
  const int m = k + s;
  {
    PROF(h, PQR_K_GRAM);
    TRY(run_gram(bv.n, k, s, bv.Q, bv.ldq, X, ldx, h->Wloc, m, h->partials, h->ticket, h->sms, h->stream,
                 &h->st.kernel_launches));
  }
  if (bv.local) {
    *Wsum = h->Wloc;
    *nparts = 1;
    return PQR_OK;
  }
  return exchange(h, m, s, Wsum, nparts);
}

// (nranks > 1) allgather this rank's Gram so every rank sums all ranks' in rank order
int exchange(Ctx* h, int m, int s, const double** Wsum, int* nparts) {
  if (h->xc && h->xc->lsa()) {
    // device-API exchange: k_factor_lsa stores this Gram into every peer's window itself
    h->st.collectives += 1;
    h->st.collective_bytes += (int64_t)m * s * 8;
    *Wsum = h->Wloc;
    *nparts = -1;
  } else if (h->xc) {
    PROF(h, PQR_K_NCCL);
    TRY(h->xc->allgather(h->Wloc, h->Wall, (size_t)m * s, h->stream));
    h->st.collectives += 1;
    h->st.collective_bytes += (int64_t)m * s * 8;
    *Wsum = h->Wall;
    *nparts = h->cfg.nranks;
  } else {
    *Wsum = h->Wloc;
    *nparts = 1;
  }
  return PQR_OK;
}

// One-launch CholQR2 for small n (k_cholqr2_small).  PQR_EPLAN when the call does not qualify:
// n above PQR_SMALL_MAX (default 32768) or its rows do not fit the CTAs' shared memory.
int run_small(Ctx* h, const BasisView& bv, const double* X, int64_t ldx, int s, bool single, double tol2, double eta,
              double* Ud, int64_t ldud, double* Uappend) {
  static const int64_t nmax = getenv("PQR_SMALL_MAX") ? atoll(getenv("PQR_SMALL_MAX")) : 32768;
  const int64_t n = bv.n;
  const int k = bv.k >= 0 ? bv.k : h->k;
  if (n > nmax) return PQR_EPLAN;
  // rows per CTA (even): at least 256 (fewer partials to sum), at most what the shared memory holds
  int R = (int)std::max<int64_t>(256, (n + h->sms - 1) / h->sms);
  R += R & 1;
  const size_t budget = 232448 - 28 * 1024;  // minus factor_body's static shared memory
  while (R > 16 && small_smem(R, k, s) > budget) R -= 16;
  const int G = (int)((n + R - 1) / R);
  if (small_smem(R, k, s) > budget || G > h->sms || (int64_t)G * R < n) return PQR_EPLAN;
  const size_t smem = small_smem(R, k, s);
  if (ensure_smem(k_cholqr2_small, smem) != cudaSuccess) {
    cudaGetLastError();
    return PQR_EPLAN;
  }
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_cholqr2_small, kSmallThreads, smem) != cudaSuccess ||
      per_sm * h->sms < G) {
    cudaGetLastError();
    return PQR_EPLAN;
  }
  const int m = k + s;
  SmallArgs a{};
  a.Q = bv.Q; a.ldq = bv.ldq; a.X = X; a.ldx = ldx; a.n = n; a.k = k; a.s = s; a.R = R;
  a.vec = ((k == 0 || (aligned16(bv.Q) && (bv.ldq & 1) == 0)) && aligned16(X) && (ldx & 1) == 0) ? 1 : 0;
  a.single = single ? 1 : 0; a.tol2 = tol2; a.eta = eta;
  a.U = Ud; a.ldu = ldud; a.U2 = Uappend; a.ldu2 = h->ld;
  a.part1 = h->partials; a.part2 = h->partials + (size_t)h->sms * m * s;
  a.bar = h->ticket + 1;  // zeroed at pqr_create, reset by every launch
  a.Pf = h->Pf; a.ldp = std::max(1, k); a.Nf = h->Nf; a.ints = h->ints;
  a.hints = h->d_hints;
  if (bv.user_out) {
    a.Pout = k > 0 ? h->outP : nullptr; a.ldpo = h->outldp;
    a.Nout = h->outN; a.ldno = h->outldn;
  }
  {
    PROF(h, PQR_K_UPDATE_GRAM);
    void* args[] = {&a};
    CUDA_TRY(cudaLaunchCooperativeKernel((const void*)k_cholqr2_small, G, kSmallThreads, args, smem, h->stream));
  }
  ++h->st.kernel_launches;
  if (!h->d_hints) CUDA_TRY(cudaMemcpyAsync(h->h_ints, h->ints, sizeof(int) * 8, cudaMemcpyDeviceToHost, h->stream));
  if (bv.user_out) h->outs_written = true;
  return PQR_OK;
}

// ---------------------------------------------------------------------------
// CholQR2 (BCGS-PIP+) solve, Alg. 8 with the recombination of DESIGN.md R1.
// ---------------------------------------------------------------------------
int cholqr2_solve(Ctx* h, const BasisView& bv, const double* X, int64_t ldx, int s, unsigned flags, double* Ud,
                  int64_t ldud, double* Uappend, int* t_host, double tau) {
  const int k = bv.k >= 0 ? bv.k : h->k;
  const int m = k + s;
  const int64_t n = bv.n;
  int* d_t1 = h->ints + 0;
  int* d_t2 = h->ints + 1;
  int* d_def = h->ints + 3;
  const double tol2 = bv.local ? 0.0 : tau * tau;
  const double eta = bv.local ? 0.0 : (h->cfg.gram_eta > 0 ? h->cfg.gram_eta : 1e-13);
  const bool single = (flags & PQR_SINGLE_PASS) != 0;

  // small n, one rank: the whole call as one cooperative kernel (small_kernels.cuh)
  if (h->hp.nch == 0 && (!h->xc || bv.local)) {
    const int rc = run_small(h, bv, X, ldx, s, single, tol2, eta, Ud, ldud, Uappend);
    if (rc != PQR_EPLAN) return rc;
  }
  // pass 1: W1 = [Q X]^T X -> P1, N1, M1, t1 -> U1 = [Q X] M1
  const double* Wsum = nullptr;
  int nparts = 1;
  if (h->hp.nch > 0) {
    // host X: one Gram per uploaded chunk; k_factor sums the chunk Grams in chunk order
    PROF(h, PQR_K_GRAM);
    for (int c = 0; c < h->hp.nch; ++c) {
      const int64_t r0 = h->hp.r[c];
      TRY(hp_wait_in(h, c));
      TRY(run_gram(h->hp.r[c + 1] - r0, k, s, bv.Q + r0, bv.ldq, X + r0, ldx, h->Wchunks + (size_t)c * m * s, m,
                   h->partials, h->ticket, h->sms, h->stream, &h->st.kernel_launches));
    }
    Wsum = h->Wchunks;
    nparts = h->hp.nch;
  } else {
    TRY(gram_and_exchange(h, bv, k, s, X, ldx, &Wsum, &nparts));
  }
  FactorArgs f{};
  f.W = Wsum; f.w_stride = (int64_t)m * s; f.nparts = nparts; f.ldw = m; f.k = k; f.s = s; f.s_dev = nullptr;
  f.tol2 = tol2; f.eta = eta;
  f.P = h->P1; f.ldp = std::max(1, k); f.N = h->N1; f.ldn = kSMax; f.M = h->M1; f.ldm = m;
  f.t_out = d_t1; f.piv_out = h->ints + 16; f.deflated = d_def;
  {
    PROF(h, PQR_K_FACTOR);
    TRY(run_factor(f, h->stream, &h->st.kernel_launches, h->xc ? h->xc->lsa() : nullptr));
  }
  bool fused = false;
  if (!single) {
    // second pass fused with the first update: U1 = [Q X] M1 and W2 = [Q U1]^T U1 in one read
    int rc;
    {
      PROF(h, PQR_K_UPDATE_GRAM);
      rc = run_update_gram(n, k, s, bv.Q, bv.ldq, X, ldx, h->M1, m, d_t1, Ud, ldud, h->Wloc, m, h->partials,
                           h->ticket, h->sms, h->stream, &h->st.kernel_launches);
    }
    if (rc == PQR_OK) {
      fused = true;
      if (bv.local) {
        Wsum = h->Wloc;
        nparts = 1;
      } else {
        TRY(exchange(h, m, s, &Wsum, &nparts));
      }
    } else if (rc != PQR_EPLAN) {
      return rc;
    }
  }
  if (!fused) {
    PROF(h, PQR_K_UPDATE);
    TRY(run_update(n, k, bv.Q, bv.ldq, s, X, ldx, h->M1, m, s, d_t1, Ud, ldud, single ? Uappend : nullptr,
                   h->ld, h->sms, h->stream, &h->st.kernel_launches));
  }
  if (!single) {
    // pass 2 on [Q U1]: W2 -> P2, N2, M2 (+ recombination) -> U = [Q U1] M2 (in place)
    if (!fused) TRY(gram_and_exchange(h, bv, k, s, Ud, ldud, &Wsum, &nparts));
    FactorArgs f2{};
    f2.W = Wsum; f2.w_stride = (int64_t)m * s; f2.nparts = nparts; f2.ldw = m; f2.k = k; f2.s = s; f2.s_dev = d_t1;
    f2.tol2 = 0.0; f2.eta = 0.0;
    f2.P = h->P2; f2.ldp = std::max(1, k); f2.N = h->N2; f2.ldn = kSMax; f2.M = h->M2; f2.ldm = m;
    f2.t_out = d_t2; f2.piv_out = h->ints + 32; f2.deflated = h->ints + 4;
    f2.P1 = h->P1; f2.ldp1 = std::max(1, k); f2.N1 = h->N1; f2.ldn1 = kSMax; f2.t1_dev = d_t1; f2.s0 = s;
    f2.Pf = h->Pf; f2.ldpf = std::max(1, k); f2.Nf = h->Nf; f2.ldnf = kSMax; f2.tf = h->ints + 2;
    {
      PROF(h, PQR_K_FACTOR);
      TRY(run_factor(f2, h->stream, &h->st.kernel_launches, h->xc ? h->xc->lsa() : nullptr));
    }
    if (h->hp.nch > 0) {
      // host U: the final pass per chunk, each chunk's rows copied out behind it
      PROF(h, PQR_K_UPDATE);
      for (int c = 0; c < h->hp.nch; ++c) {
        const int64_t r0 = h->hp.r[c];
        TRY(run_update(h->hp.r[c + 1] - r0, k, bv.Q + r0, bv.ldq, s, Ud + r0, ldud, h->M2, m, s, d_t2, Ud + r0,
                       ldud, Uappend ? Uappend + r0 : nullptr, h->ld, h->sms, h->stream, &h->st.kernel_launches));
        TRY(hp_d2h_chunk(h, c, Ud, ldud, s));
      }
    } else {
      PROF(h, PQR_K_UPDATE);
      TRY(run_update(n, k, bv.Q, bv.ldq, s, Ud, ldud, h->M2, m, s, d_t2, Ud, ldud, Uappend, h->ld, h->sms,
                     h->stream, &h->st.kernel_launches));
    }
  } else {
    CUDA_TRY(cudaMemcpyAsync(h->Pf, h->P1, sizeof(double) * std::max(1, k) * s, cudaMemcpyDeviceToDevice, h->stream));
    CUDA_TRY(cudaMemcpyAsync(h->Nf, h->N1, sizeof(double) * kSMax * kSMax, cudaMemcpyDeviceToDevice, h->stream));
    CUDA_TRY(cudaMemcpyAsync(h->ints + 2, d_t1, sizeof(int), cudaMemcpyDeviceToDevice, h->stream));
  }
  // t (ints[2]) and the deflation count (ints[3]) reach the host with the caller's single
  // synchronisation in pqr_project_normalize
  CUDA_TRY(cudaMemcpyAsync(h->h_ints, h->ints, sizeof(int) * 8, cudaMemcpyDeviceToHost, h->stream));
  (void)t_host;
  (void)flags;
  return PQR_OK;
}

}  // namespace

// ===========================================================================
// TSQR variant (kept in its own translation-unit-style header)
// ===========================================================================
#include "tsqr_api.cuh"

// ===========================================================================
// C-ABI
// ===========================================================================
extern "C" {

const char* pqr_strerror(int code) {
  switch (code) {
    case PQR_OK: return "ok";
    case PQR_EARG: return "invalid argument (dimension, leading dimension or null pointer)";
    case PQR_ECAPACITY: return "capacity exceeded (k + s > k_max + s_max or s > s_max)";
    case PQR_EBREAKDOWN: return "Cholesky breakdown / deflation needed with PQR_NO_DEFLATION";
    case PQR_EPLAN: return "invalid TSQR block plan";
    case PQR_ECUDA: return "CUDA error";
    case PQR_ENCCL: return "NCCL error";
    case PQR_ENOMEM: return "device allocation failed";
    default: return "unknown error";
  }
}

int pqr_create(pqr_handle* out, const pqr_config* cfg, const double* Q, int64_t ldq, int k) {
  if (!out || !cfg) return PQR_EARG;
  *out = nullptr;
  if (cfg->n_local <= 0 || cfg->k_max < 0 || cfg->s_max < 1 || cfg->s_max > kSMax || k < 0 || k > cfg->k_max)
    return PQR_EARG;
  if (cfg->k_max + cfg->s_max > kMMax) return PQR_ECAPACITY;
  if (cfg->variant != PQR_CHOLQR2 && cfg->variant != PQR_TSQR) return PQR_EARG;
  if (cfg->reduction != PQR_REDUCTION_HH && cfg->reduction != PQR_REDUCTION_PIP2) return PQR_EARG;
  if (cfg->local != PQR_LOCAL_HH && cfg->local != PQR_LOCAL_PIP2) return PQR_EARG;
  if (cfg->chains < PQR_CHAINS_AUTO || cfg->chains > PQR_CHAINS_ON) return PQR_EARG;
  if (cfg->nranks < 1 || cfg->rank < 0 || cfg->rank >= cfg->nranks) return PQR_EARG;
  if (cfg->nranks > 1 && !cfg->nccl_id && !cfg->vgroup) return PQR_EARG;
  if (k > 0 && (!Q || ldq < cfg->n_local)) return PQR_EARG;
  if (k > cfg->n_local) return PQR_EARG;

  Ctx* h = new Ctx();
  h->cfg = *cfg;
  h->stream = (cudaStream_t)cfg->stream;
  int dev = 0;
  cudaGetDevice(&dev);  // the caller's current device becomes the handle's device
  h->device = dev;
  cudaDeviceGetAttribute(&h->sms, cudaDevAttrMultiProcessorCount, dev);
  if (const char* e = getenv("PQR_SMS")) {  // testing aid: size grids for fewer SMs (several blocks per CTA)
    const int v = atoi(e);
    if (v >= 1 && v < h->sms) h->sms = v;
  }
  h->cap = cfg->k_max + cfg->s_max;
  h->ld = (cfg->n_local + 1) & ~int64_t(1);  // even leading dimension: 16-byte row pairs
  const int64_t n = cfg->n_local;
  const int sm = cfg->s_max;
  int rc = PQR_OK;
  auto fail = [&](int code) {
    pqr_destroy(reinterpret_cast<pqr_handle>(h));
    return code;
  };
  // small workspaces (both variants)
  int64_t pe = 0;
  for (int kk = 0; kk <= cfg->k_max; ++kk) pe = std::max(pe, gram_partials_needed(n, kk, sm, h->sms));
  h->partials_elems = pe;
  if ((rc = dalloc(&h->partials, pe))) return fail(rc);
  if ((rc = dalloc(&h->ticket, 4))) return fail(rc);
  if ((rc = dalloc(&h->Wloc, (size_t)h->cap * sm))) return fail(rc);
  if ((rc = dalloc(&h->Wall, (size_t)h->cap * sm * cfg->nranks))) return fail(rc);
  const size_t pk = (size_t)std::max(1, cfg->k_max) * sm;
  if ((rc = dalloc(&h->P1, pk)) || (rc = dalloc(&h->P2, pk)) || (rc = dalloc(&h->Pf, pk))) return fail(rc);
  const size_t nn = (size_t)kSMax * kSMax;
  if ((rc = dalloc(&h->N1, nn)) || (rc = dalloc(&h->N2, nn)) || (rc = dalloc(&h->Nf, nn))) return fail(rc);
  if ((rc = dalloc(&h->M1, (size_t)h->cap * sm)) || (rc = dalloc(&h->M2, (size_t)h->cap * sm))) return fail(rc);
  if ((rc = dalloc(&h->ints, 64))) return fail(rc);
  if (cudaMallocHost(&h->h_ints, 64 * sizeof(int)) != cudaSuccess) return fail(PQR_ENOMEM);
  if (cudaHostGetDevicePointer((void**)&h->d_hints, h->h_ints, 0) != cudaSuccess) {
    cudaGetLastError();  // not mapped: t comes back with a copy
    h->d_hints = nullptr;
  }
  if (cudaMemsetAsync(h->ticket, 0, 4 * sizeof(unsigned int), h->stream) != cudaSuccess) return fail(PQR_ECUDA);
  if (cudaMemsetAsync(h->ints, 0, 64 * sizeof(int), h->stream) != cudaSuccess) return fail(PQR_ECUDA);

  // cross-rank exchange: a virtual group (P handles in this process), or NCCL (nranks > 1;
  // PQR_FORCE_NCCL=1, a test aid, builds a single-rank communicator and runs every cross-GPU
  // step with one rank)
  static const bool force_nccl = getenv("PQR_FORCE_NCCL") && atoi(getenv("PQR_FORCE_NCCL")) != 0;
  if (cfg->vgroup) {
    VirtualGroup* g = reinterpret_cast<VirtualGroup*>(cfg->vgroup);
    if (g->P != cfg->nranks) return fail(PQR_EARG);
    auto* vx = new VirtualExchange();
    h->xc = vx;
    if (const int e = vx->init(g, cfg->rank)) return fail(e == -1 ? PQR_EARG : PQR_ECUDA);
  } else if (cfg->nranks > 1 || force_nccl) {
    ncclUniqueId id;
    if (cfg->nccl_id) {
      memcpy(&id, cfg->nccl_id, sizeof(id));
    } else if (ncclGetUniqueId(&id) != ncclSuccess) {
      return fail(PQR_ENCCL);
    }
    if (cfg->exchange != PQR_EXCHANGE_AUTO && cfg->exchange != PQR_EXCHANGE_COLLECTIVE &&
        cfg->exchange != PQR_EXCHANGE_LSA)
      return fail(PQR_EARG);
    static const bool env_lsa = getenv("PQR_EXCHANGE") && strcmp(getenv("PQR_EXCHANGE"), "lsa") == 0;
    const bool use_lsa = cfg->exchange == PQR_EXCHANGE_LSA || (cfg->exchange == PQR_EXCHANGE_AUTO && env_lsa);
    NcclExchange* nx = use_lsa ? new LsaExchange() : new NcclExchange();
    nx->rank = cfg->rank;
    nx->nranks = cfg->nranks;
    h->xc = nx;
    ncclResult_t r = ncclCommInitRank(&nx->comm, cfg->nranks, id, cfg->rank);
    if (r != ncclSuccess) {
      fprintf(stderr, "[pqr] ncclCommInitRank: %s\n", ncclGetErrorString(r));
      nx->comm = nullptr;
      return fail(PQR_ENCCL);
    }
    // window slots hold the largest block either variant sends: (k_max + s_max) x s_max
    if (use_lsa)
      if (const int e = static_cast<LsaExchange*>(nx)->setup((int64_t)h->cap * cfg->s_max))
        return fail(e == -7 ? PQR_ENOMEM : (e == -5 ? PQR_ECUDA : PQR_ENCCL));
  }

  // host Q is staged through a temporary device copy
  const double* Qd = Q;
  double* Qtmp = nullptr;
  int64_t ldqd = ldq;
  if (k > 0 && is_host_ptr(Q)) {
    if ((rc = dalloc(&Qtmp, (size_t)h->ld * k))) return fail(rc);
    if (cudaMemcpy2DAsync(Qtmp, h->ld * sizeof(double), Q, ldq * sizeof(double), n * sizeof(double), k,
                          cudaMemcpyHostToDevice, h->stream) != cudaSuccess) {
      cudaFree(Qtmp);
      return fail(PQR_ECUDA);
    }
    Qd = Qtmp;
    ldqd = h->ld;
  }
  if (cfg->variant == PQR_CHOLQR2) {
    if ((rc = dalloc(&h->basis, (size_t)h->ld * h->cap))) {
      cudaFree(Qtmp);
      return fail(rc);
    }
    if (k > 0 && cudaMemcpy2DAsync(h->basis, h->ld * sizeof(double), Qd, ldqd * sizeof(double), n * sizeof(double),
                                   k, cudaMemcpyDeviceToDevice, h->stream) != cudaSuccess) {
      cudaFree(Qtmp);
      return fail(PQR_ECUDA);
    }
    h->k = k;
  } else {
    rc = tsqr_create(h, Qd, ldqd, k);
    if (rc) {
      cudaFree(Qtmp);
      return fail(rc);
    }
  }
  if (cudaStreamSynchronize(h->stream) != cudaSuccess) {
    cudaFree(Qtmp);
    return fail(PQR_ECUDA);
  }
  cudaFree(Qtmp);
  h->st.k = h->k;
  *out = reinterpret_cast<pqr_handle>(h);
  return PQR_OK;
}

int pqr_project_normalize(pqr_handle hh, const double* X, int64_t ldx, int s, unsigned flags, double* U,
                          int64_t ldu, double* P, int ldp, double* N, int ldn, int* t) {
  Ctx* h = reinterpret_cast<Ctx*>(hh);
  if (!h || !X || !t || s < 1) return PQR_EARG;
  DevGuard dg(h->device);
  const int64_t n = h->cfg.n_local;
  const int k = h->k;
  if (s > h->cfg.s_max || k + s > h->cap) return PQR_ECAPACITY;
  if (ldx < n) return PQR_EARG;
  if (U && ldu < n) return PQR_EARG;
  if (P && k > 0 && ldp < k) return PQR_EARG;
  if (N && ldn < s) return PQR_EARG;
  const bool append = !(flags & PQR_NO_APPEND);
  if (!append && !U) return PQR_EARG;

  static const bool no_graph = getenv("PQR_NO_GRAPH") != nullptr;
  GraphKey key;
  key.X = X; key.ldx = ldx; key.s = s; key.flags = flags; key.U = U; key.ldu = ldu; key.P = P; key.ldp = ldp;
  key.N = N; key.ldn = ldn; key.k = k;
  if (h->gexec && !h->prof && key == h->gkey) {
    if (h->gstream) {  // legacy default stream: replay on the handle's own stream behind it
      CUDA_TRY(cudaEventRecord(h->gev, h->stream));
      CUDA_TRY(cudaStreamWaitEvent(h->gstream, h->gev, 0));
    }
    CUDA_TRY(cudaGraphLaunch(h->gexec, h->gstream ? h->gstream : h->stream));
    CUDA_TRY(cudaStreamSynchronize(h->gstream ? h->gstream : h->stream));
    const int tg = h->h_ints[2];
    h->st.kernel_launches += h->g_launches;
    if ((flags & PQR_NO_DEFLATION) && h->h_ints[3] > 0) return PQR_EBREAKDOWN;
    *t = tg;
    h->st.calls += 1;
    h->st.last_t = tg;
    return PQR_OK;
  }

  // stage host inputs (host X and U on one rank: pipelined in row chunks, HostPipe)
  const double* Xd = X;
  int64_t ldxd = ldx;
  const bool x_host = is_host_ptr(X);
  const bool u_host = U && is_host_ptr(U);
  h->hp.nch = 0;
  if (x_host) {
    if (!h->stageX && dalloc(&h->stageX, (size_t)h->ld * h->cfg.s_max)) return PQR_ENOMEM;
    if (u_host && !h->xc && !(flags & PQR_SINGLE_PASS) &&
        !(h->cfg.variant == PQR_TSQR && h->cfg.local == PQR_LOCAL_PIP2)) {
      if (h->cfg.variant == PQR_CHOLQR2) {
        if (!h->Wchunks && dalloc(&h->Wchunks, (size_t)kHostChunksMax * h->cap * h->cfg.s_max)) return PQR_ENOMEM;
        TRY(hp_plan_upload(h, X, ldx, s, U, ldu, nullptr));
      } else {
        std::vector<int64_t> bounds;
        tsqr_leaf_bounds(h, &bounds);
        TRY(hp_plan_upload(h, X, ldx, s, U, ldu, &bounds));
      }
    }
    if (h->hp.nch == 0)
      CUDA_TRY(cudaMemcpy2DAsync(h->stageX, h->ld * sizeof(double), X, ldx * sizeof(double), n * sizeof(double), s,
                                 cudaMemcpyHostToDevice, h->stream));
    Xd = h->stageX;
    ldxd = h->ld;
  }
  double* Ud = nullptr;
  int64_t ldud = 0;
  if (U && !u_host && (ldu & 1) == 0 && aligned16(U)) {
    Ud = U;
    ldud = ldu;
  } else if (!U && append && h->cfg.variant == PQR_CHOLQR2) {
    Ud = h->basis + (int64_t)k * h->ld;  // compute in place in the basis' spare columns
    ldud = h->ld;
  } else {
    if (!h->stageU && dalloc(&h->stageU, (size_t)h->ld * h->cfg.s_max)) return PQR_ENOMEM;
    Ud = h->stageU;
    ldud = h->ld;
  }
  const double tau = h->cfg.defl_tol > 0 ? h->cfg.defl_tol : 1e-12;
  int tt = 0;
  // graph capture: the second consecutive call with the same key, device buffers only, one rank
  const bool graphable = !no_graph && !append && !x_host && !u_host && Ud == U && !h->xc && !h->prof &&
                         h->hp.nch == 0 && !(P && k > 0 && is_host_ptr(P)) && !(N && is_host_ptr(N));
  bool capturing = false;
  if (graphable && key == h->gcand) {
    if (h->gexec) {
      cudaGraphExecDestroy(h->gexec);
      h->gexec = nullptr;
    }
    if (!h->stream && !h->gstream) {
      if (cudaStreamCreateWithFlags(&h->gstream, cudaStreamNonBlocking) != cudaSuccess ||
          cudaEventCreateWithFlags(&h->gev, cudaEventDisableTiming) != cudaSuccess) {
        cudaGetLastError();
        if (h->gstream) cudaStreamDestroy(h->gstream);
        h->gstream = nullptr;
      }
    }
    if (!h->stream && h->gstream) {
      // capture on the handle's own stream (the legacy stream cannot be captured)
      CUDA_TRY(cudaEventRecord(h->gev, h->stream));
      CUDA_TRY(cudaStreamWaitEvent(h->gstream, h->gev, 0));
      h->stream = h->gstream;
    }
    capturing = h->stream && !wy_trace_buf() && cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
    if (!capturing) cudaGetLastError();
  }
  h->gcand = graphable ? key : GraphKey{};
  const int64_t launches0 = h->st.kernel_launches;
  auto enqueue = [&]() -> int {
    int rc;
    h->outP = (P && k > 0 && !is_host_ptr(P)) ? P : nullptr;
    h->outldp = ldp;
    h->outN = (N && !is_host_ptr(N)) ? N : nullptr;
    h->outldn = ldn;
    h->outs_written = false;
    if (h->cfg.variant == PQR_CHOLQR2) {
      double* Uapp = (append && Ud != h->basis + (int64_t)k * h->ld) ? h->basis + (int64_t)k * h->ld : nullptr;
      BasisView bv{h->basis, h->ld, n};
      bv.user_out = true;
      rc = cholqr2_solve(h, bv, Xd, ldxd, s, flags, Ud, ldud, Uapp, &tt, tau);
    } else {
      rc = tsqr_solve(h, Xd, ldxd, s, flags, Ud, ldud, append, &tt);
    }
    if (rc != PQR_OK) return rc;
    // outputs (enqueued before the one synchronisation of the call)
    TRY(hp_finish(h));
    if (U && Ud != U && h->hp.nch == 0) {
      CUDA_TRY(cudaMemcpy2DAsync(U, ldu * sizeof(double), Ud, ldud * sizeof(double), n * sizeof(double), s,
                                 cudaMemcpyDefault, h->stream));
    }
    if (P && k > 0 && !(h->outs_written && h->outP == P))
      CUDA_TRY(cudaMemcpy2DAsync(P, (size_t)ldp * sizeof(double), h->Pf, (size_t)std::max(1, k) * sizeof(double),
                                 (size_t)k * sizeof(double), s, cudaMemcpyDefault, h->stream));
    if (N && !(h->outs_written && h->outN == N))
      CUDA_TRY(cudaMemcpy2DAsync(N, (size_t)ldn * sizeof(double), h->Nf, (size_t)kSMax * sizeof(double),
                                 (size_t)s * sizeof(double), s, cudaMemcpyDefault, h->stream));
    return PQR_OK;
  };
  int rc = enqueue();
  if (capturing) {
    cudaGraph_t graph = nullptr;
    const cudaError_t ec = cudaStreamEndCapture(h->stream, &graph);
    if (rc == PQR_OK && ec == cudaSuccess && graph &&
        cudaGraphInstantiate(&h->gexec, graph, 0) == cudaSuccess) {
      h->gkey = key;
      h->g_launches = h->st.kernel_launches - launches0;
      rc = cudaGraphLaunch(h->gexec, h->stream) == cudaSuccess ? PQR_OK : PQR_ECUDA;
    } else {
      // capture failed: run the call uncaptured
      cudaGetLastError();
      h->gexec = nullptr;
      h->gcand = GraphKey{};
      if (rc == PQR_OK) rc = enqueue();
    }
    if (graph) cudaGraphDestroy(graph);
    if (h->gstream && h->stream == h->gstream) {
      h->stream = (cudaStream_t)h->cfg.stream;  // back to the legacy stream after this call
      CUDA_TRY(cudaStreamSynchronize(h->gstream));
    }
  }
  if (rc != PQR_OK) {
    if (h->hp.nch > 0) cudaStreamSynchronize(h->cstream);
    h->hp.nch = 0;
    return rc;
  }
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  h->hp.nch = 0;
  prof_collect(h);
  tt = h->h_ints[2];
  if ((flags & PQR_NO_DEFLATION) && h->h_ints[3] > 0) return PQR_EBREAKDOWN;  // basis unchanged
  if (append && h->cfg.variant == PQR_TSQR) TRY(tsqr_commit(h, s, tt, h->ts->merge, h->ts->mtoff));
  *t = tt;
  if (append) h->k += tt;
  h->st.calls += 1;
  h->st.k = h->k;
  h->st.last_t = tt;
  return PQR_OK;
}

int pqr_basis_apply(pqr_handle hh, const double* C, int ldc, int m, double* Y, int64_t ldy) {
  Ctx* h = reinterpret_cast<Ctx*>(hh);
  if (!h || m < 0 || !Y) return PQR_EARG;
  DevGuard dg(h->device);
  const int64_t n = h->cfg.n_local;
  const int k = h->k;
  if (ldy < n || (k > 0 && (!C || ldc < k))) return PQR_EARG;
  if (m == 0) return PQR_OK;
  if (h->cfg.variant == PQR_TSQR) return tsqr_apply(h, C, ldc, m, Y, ldy);
  // Y = Q C in chunks of <= 16 output columns (host / unaligned Y staged through stageU)
  const bool stage = is_host_ptr(Y) || (ldy & 1) || !aligned16(Y);
  if (stage && !h->stageU && dalloc(&h->stageU, (size_t)h->ld * h->cfg.s_max)) return PQR_ENOMEM;
  if (!h->stageC && dalloc(&h->stageC, (size_t)h->cap * 16)) return PQR_ENOMEM;
  const int chunk = stage ? std::min(16, h->cfg.s_max) : 16;
  for (int c0 = 0; c0 < m; c0 += chunk) {
    const int mc = std::min(chunk, m - c0);
    double* dst = stage ? h->stageU : Y + (int64_t)c0 * ldy;
    const int64_t ldd = stage ? h->ld : ldy;
    if (k == 0) {
      CUDA_TRY(cudaMemset2DAsync(dst, ldd * sizeof(double), 0, n * sizeof(double), mc, h->stream));
    } else {
      CUDA_TRY(cudaMemcpy2DAsync(h->stageC, (size_t)k * sizeof(double), C + (int64_t)c0 * ldc,
                                 (size_t)ldc * sizeof(double), (size_t)k * sizeof(double), mc, cudaMemcpyDefault,
                                 h->stream));
      PROF(h, PQR_K_UPDATE);
      TRY(run_update(n, k, h->basis, h->ld, 0, nullptr, 0, h->stageC, k, mc, nullptr, dst, ldd, nullptr, 0, h->sms,
                     h->stream, &h->st.kernel_launches));
    }
    if (stage)
      CUDA_TRY(cudaMemcpy2DAsync(Y + (int64_t)c0 * ldy, ldy * sizeof(double), h->stageU, h->ld * sizeof(double),
                                 n * sizeof(double), mc, cudaMemcpyDefault, h->stream));
  }
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  prof_collect(h);
  return PQR_OK;
}

int pqr_destroy(pqr_handle hh) {
  Ctx* h = reinterpret_cast<Ctx*>(hh);
  if (!h) return PQR_OK;
  DevGuard dg(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  else cudaDeviceSynchronize();
  tsqr_free(h);
  cudaFree(h->basis);
  cudaFree(h->partials);
  cudaFree(h->ticket);
  cudaFree(h->Wloc);
  cudaFree(h->Wall);
  cudaFree(h->P1); cudaFree(h->N1); cudaFree(h->M1);
  cudaFree(h->P2); cudaFree(h->N2); cudaFree(h->M2);
  cudaFree(h->Pf); cudaFree(h->Nf);
  cudaFree(h->ints);
  if (h->h_ints) cudaFreeHost(h->h_ints);
  cudaFree(h->stageX); cudaFree(h->stageU); cudaFree(h->stageC); cudaFree(h->Wchunks);
  if (h->cstream) {
    cudaStreamSynchronize(h->cstream);
    for (int c = 0; c < kHostChunksMax; ++c) {
      cudaEventDestroy(h->hp_in[c]);
      cudaEventDestroy(h->hp_out[c]);
    }
    cudaEventDestroy(h->hp_done);
    cudaStreamDestroy(h->cstream);
  }
  delete h->xc;
  if (h->gexec) cudaGraphExecDestroy(h->gexec);
  if (h->gstream) cudaStreamDestroy(h->gstream);
  if (h->gev) cudaEventDestroy(h->gev);
  for (auto& p : h->pending) { h->ev_pool.push_back(p.a); h->ev_pool.push_back(p.b); }
  for (auto e : h->ev_pool) cudaEventDestroy(e);
  delete h;
  return PQR_OK;
}

int pqr_get_stats(pqr_handle hh, pqr_stats* st) {
  Ctx* h = reinterpret_cast<Ctx*>(hh);
  if (!h || !st) return PQR_EARG;
  *st = h->st;
  st->exchange = h->xc ? h->xc->kind : 0;
  return PQR_OK;
}

int pqr_profile_enable(pqr_handle hh, int enable) {
  Ctx* h = reinterpret_cast<Ctx*>(hh);
  if (!h) return PQR_EARG;
  DevGuard dg(h->device);
  cudaStreamSynchronize(h->stream);
  prof_collect(h);
  h->prof = enable != 0;
  h->prof_tot = pqr_profile{};
  return PQR_OK;
}

int pqr_get_profile(pqr_handle hh, pqr_profile* out) {
  Ctx* h = reinterpret_cast<Ctx*>(hh);
  if (!h || !out) return PQR_EARG;
  DevGuard dg(h->device);
  cudaStreamSynchronize(h->stream);
  prof_collect(h);
  *out = h->prof_tot;
  return PQR_OK;
}

#ifdef PQR_SMALL_TRACE
int pqr_small_trace(unsigned long long* out16) {
  if (cudaMemcpyFromSymbol(out16, g_small_trace, 9 * sizeof(unsigned long long)) != cudaSuccess) return PQR_ECUDA;
  return cudaMemcpyFromSymbol(out16 + 9, g_factor_trace, 5 * sizeof(unsigned long long)) == cudaSuccess ? PQR_OK
                                                                                                       : PQR_ECUDA;
}
#endif

int pqr_vgroup_create(int nranks, void** out) {
  if (!out || nranks < 1 || nranks > 1024) return PQR_EARG;
  *out = new VirtualGroup(nranks);
  return PQR_OK;
}

int pqr_vgroup_destroy(void* group) {
  delete reinterpret_cast<VirtualGroup*>(group);
  return PQR_OK;
}

int pqr_nccl_unique_id(void* id128) {
  if (!id128) return PQR_EARG;
  ncclUniqueId id;
  NCCL_TRY(ncclGetUniqueId(&id));
  static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
  memcpy(id128, &id, sizeof(id));
  return PQR_OK;
}

// ---------------------------------------------------------------------------
// step-level entry points (include/pqr_steps.h)
// ---------------------------------------------------------------------------
int pqr_laplacian7_apply(int nx, int ny, int nz, int s, const double* V, int64_t ldv, double* Y, int64_t ldy,
                         void* stream) {
  const int64_t npts = (int64_t)nx * ny * nz;
  if (nx < 1 || ny < 1 || nz < 1 || s < 1 || s > 16 || !V || !Y || ldv < npts || ldy < npts) return PQR_EARG;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // z-chunks so that the grid covers the SMs several times over (each chunk re-reads 2 halo planes)
  const int64_t tiles = (int64_t)((nx + kLapTX - 1) / kLapTX) * ((ny + kLapTY - 1) / kLapTY);
  if (tiles > INT32_MAX) return PQR_EARG;
  int zchunk = nz;
  while (zchunk > 8 && tiles * s * ((nz + zchunk - 1) / zchunk) < (int64_t)sms * 8) zchunk = (zchunk + 1) / 2;
  const dim3 grid((unsigned)tiles, (unsigned)((nz + zchunk - 1) / zchunk), (unsigned)s);
  k_laplacian7<<<grid, dim3(kLapTX, kLapTY), 0, (cudaStream_t)stream>>>(nx, ny, nz, zchunk, V, ldv, Y, ldy);
  return cudaGetLastError() == cudaSuccess ? PQR_OK : PQR_ECUDA;
}

int pqr_step_gram(int64_t n, int k, int s, const double* Q, int64_t ldq, const double* X, int64_t ldx, double* W,
                  int ldw, void* stream) {
  if (n <= 0 || k < 0 || s < 1 || s > kSMax || k + s > kMMax || !X || ldx < n || (k > 0 && (!Q || ldq < n)) ||
      !W || ldw < k + s)
    return PQR_EARG;
  cudaStream_t st = (cudaStream_t)stream;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* part = nullptr;
  unsigned int* ticket = nullptr;
  if (dalloc(&part, gram_partials_needed(n, k, s, sms)) || dalloc(&ticket, 1)) {
    cudaFree(part);
    return PQR_ENOMEM;
  }
  cudaMemsetAsync(ticket, 0, sizeof(unsigned int), st);
  int rc = run_gram(n, k, s, Q, ldq, X, ldx, W, ldw, part, ticket, sms, st, nullptr);
  cudaStreamSynchronize(st);
  cudaFree(part);
  cudaFree(ticket);
  return rc ? rc : (cudaGetLastError() == cudaSuccess ? PQR_OK : PQR_ECUDA);
}

int pqr_step_factor(int k, int s, const double* W, int ldw, double tol2_rel, double eta, double* N, int ldn,
                    double* M, int ldm, int* t_host, int* piv_host, void* stream) {
  if (k < 0 || s < 1 || s > kSMax || k + s > kMMax || !W || ldw < k + s || !N || ldn < s || !M || ldm < k + s ||
      !t_host)
    return PQR_EARG;
  cudaStream_t st = (cudaStream_t)stream;
  double *P = nullptr, *Nt = nullptr;
  int* ints = nullptr;
  if (dalloc(&P, (size_t)std::max(1, k) * s) || dalloc(&Nt, kSMax * kSMax) || dalloc(&ints, 64)) {
    cudaFree(P);
    cudaFree(Nt);
    return PQR_ENOMEM;
  }
  FactorArgs f{};
  f.W = W; f.w_stride = 0; f.nparts = 1; f.ldw = ldw; f.k = k; f.s = s; f.tol2 = tol2_rel; f.eta = eta;
  f.P = P; f.ldp = std::max(1, k); f.N = Nt; f.ldn = kSMax; f.M = M; f.ldm = ldm;
  f.t_out = ints; f.piv_out = ints + 16; f.deflated = ints + 1;
  int rc = run_factor(f, st, nullptr);
  int hbuf[32];
  if (!rc) {
    cudaMemcpy2DAsync(N, ldn * sizeof(double), Nt, kSMax * sizeof(double), s * sizeof(double), s, cudaMemcpyDefault,
                      st);
    cudaMemcpyAsync(hbuf, ints, 32 * sizeof(int), cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) rc = PQR_ECUDA;
  }
  if (!rc) {
    *t_host = hbuf[0];
    if (piv_host)
      for (int i = 0; i < s; ++i) piv_host[i] = hbuf[16 + i];
  }
  cudaFree(P);
  cudaFree(Nt);
  cudaFree(ints);
  return rc;
}

int pqr_step_update(int64_t n, int k, int s, const double* Q, int64_t ldq, const double* X, int64_t ldx,
                    const double* M, int ldm, int t, double* U, int64_t ldu, void* stream) {
  if (n <= 0 || k < 0 || s < 1 || s > kSMax || t < 0 || t > s || k + s > kMMax || !X || ldx < n ||
      (k > 0 && (!Q || ldq < n)) || !M || ldm < k + s || !U || ldu < n)
    return PQR_EARG;
  cudaStream_t st = (cudaStream_t)stream;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int* td = nullptr;
  if (dalloc(&td, 1)) return PQR_ENOMEM;
  cudaMemcpyAsync(td, &t, sizeof(int), cudaMemcpyHostToDevice, st);
  int rc = run_update(n, k, Q, ldq, s, X, ldx, M, ldm, s, td, U, ldu, nullptr, 0, sms, st, nullptr);
  if (cudaStreamSynchronize(st) != cudaSuccess) rc = PQR_ECUDA;
  cudaFree(td);
  return rc;
}

}  // extern "C"
