/*
 * pqr.h — C-ABI of libpqr.so, a B200-native (sm_100a) fp64 project-and-normalize
 * (PQR) library after arXiv 2204.13393 ("TSPQR", PAPER.md).
 *
 * The PQR problem (§1 Eq. (1)):  given Q (n x k, orthonormal
 * columns) and a new block X (n x s), compute U (n x t, orthonormal, Q^T U = 0),
 * P (k x s) and N (t x s, upper triangular / row echelon when t < s) with
 *
 *        [Q X] = [Q U] [ I  P ]
 *                      [ 0  N ] .
 *
 * Two variants (BASELINE.json north_star):
 *   PQR_CHOLQR2 — BCGS-PIP applied twice (BCGS-PIP+, Alg. 8):
 *                 fused Gram pass, small Cholesky, fused update pass, x2.
 *   PQR_TSQR    — TreeTSPQR (Alg. 9) with Householder local and
 *                 Householder reduction subalgorithms; the basis is kept in its
 *                 locally orthogonal representation (LOR):
 *                 per-block reflectors plus a stateful reflector tree.
 *
 * Conventions (all calls):
 *  - Matrices are fp64, column-major (LAPACK) with an explicit leading dimension
 *    ld >= rows.
 *  - Matrix pointers may be DEVICE pointers (cudaMalloc'd, the fast path) or HOST
 *    pointers (pageable or pinned); the library detects host memory with
 *    cudaPointerGetAttributes and stages it through handle-owned device buffers on
 *    the handle's stream.  With both X and U on the host (one rank, from 2^18 rows) the
 *    staging is pipelined: row chunks move on a second, handle-owned copy stream while
 *    the first and last passes run chunk by chunk.  The caller owns every pointer it
 *    passes.
 *  - Every call is ordered on the handle's stream (pqr_config.stream).  Calls that
 *    return a host scalar (t) synchronise that stream (and the copy stream) before
 *    returning.
 *  - Handles share no mutable state: distinct handles (each with its own stream) may
 *    be called concurrently from different host threads; one handle must not be.
 *  - Multi-GPU: one process per GPU; every rank calls every function collectively
 *    with its own contiguous row shard (n_local rows).  P, N and t are replicated
 *    (bitwise identical) on all ranks.
 *  - Errors: 0 = PQR_OK, negative codes below.  On any error the basis is left
 *    unchanged (it is only extended after a successful solve).
 */
#ifndef PQR_H
#define PQR_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PQR_OK          0
#define PQR_EARG       -1  /* bad dimension, leading dimension or null pointer   */
#define PQR_ECAPACITY  -2  /* k + s exceeds k_max + s_max, or s > s_max           */
#define PQR_EBREAKDOWN -3  /* Cholesky pivot <= threshold with PQR_NO_DEFLATION    */
#define PQR_EPLAN      -4  /* TSQR block plan invalid (block_rows < k_max + s_max) */
#define PQR_ECUDA      -5  /* CUDA runtime error                                   */
#define PQR_ENCCL      -6  /* NCCL error                                           */
#define PQR_ENOMEM     -7  /* device allocation failed                             */

typedef struct pqr_ctx* pqr_handle;

typedef enum { PQR_CHOLQR2 = 0, PQR_TSQR = 1 } pqr_variant;

/* PQR_TSQR: the reduction subalgorithm above the GPU's local Householder tree (§4,
 * "local" and "reduction" subalgorithms; fig:architecture, L1186-1204, maps a reduction by
 * BCGS-PIP+ onto the message-passing level):
 *   PQR_REDUCTION_HH   — Householder: an arity-bounded tree over the GPU roots' (C+s) x s blocks,
 *                        replicated on every GPU, then the top Householder solve with deflation
 *                        (stable at any condition number);
 *   PQR_REDUCTION_PIP2 — BCGS-PIP+ (Alg. 8) on the stacked GPU-root coordinates: two Gram
 *                        exchanges of (k+s) x s per call; each GPU keeps its own top coordinates
 *                        of the basis.  Stable only while eps*kappa^2 <= 1/2;
 *                        beyond, orthogonality is lost (the call does not fail). */
#define PQR_REDUCTION_HH   0
#define PQR_REDUCTION_PIP2 1
/* PQR_TSQR: the local subalgorithm on each GPU (§4: "local" subalgorithm):
 *   PQR_LOCAL_HH   — Householder on row blocks with the on-GPU reduction tree; the basis in its
 *                    locally orthogonal representation (default);
 *   PQR_LOCAL_PIP2 — BCGS-PIP+ of the GPU's whole shard against an explicit, locally orthonormal
 *                    basis of that shard (one local problem per GPU, no on-GPU tree); the GPU's
 *                    (C+s) x s coefficient block goes to the reduction as with PQR_LOCAL_HH, and U
 *                    is formed from the local basis and the reduction's coefficients.  Stable only
 *                    while eps*kappa^2 <= 1/2 (the local problem inherits BCGS-PIP+'s bound).
 *                    Exists for the stability experiment of PAPER.md:L1274-1291 (fig:heatmap). */
#define PQR_LOCAL_HH   0
#define PQR_LOCAL_PIP2 1
/* How the small blocks cross GPUs (nranks > 1 with nccl_id, or PQR_FORCE_NCCL=1):
 *   PQR_EXCHANGE_COLLECTIVE — ncclAllGather on the handle's stream between the library's kernels
 *                             (kernel -> NCCL kernel -> kernel);
 *   PQR_EXCHANGE_LSA        — the NCCL device API: a kernel stores the rank's block straight into
 *                             every peer's slot of a symmetric NCCL window over NVLink and meets
 *                             the peers at an LSA barrier; for CholQR2 this is done by the factor
 *                             kernel itself (no separate exchange launch).  Needs every rank in one
 *                             NVLink (LSA) domain and symmetric-memory support; pqr_create returns
 *                             PQR_ENCCL when either is missing.  (PAPER.md:L1160-1166, L1546-1552:
 *                             the reduction as a stateful in-network step.)
 *   PQR_EXCHANGE_AUTO (0)   — COLLECTIVE, unless PQR_EXCHANGE=lsa is set in the environment. */
/* PQR_TSQR with PQR_LOCAL_HH: FlatTSPQR chains of leaf blocks (§4.2, Alg. 10, Eqs.
 * flat_tsqr / flattspqr_q, L815-983; the paper's own on-node choice, fig:architecture L1195-1200):
 * the GPU's leaf blocks form 2 x (SM count) chains (chain c = blocks c, c + nchain, ...); block i of
 * a chain solves the stacked problem [Q_i | P_{i-1}; N_{i-1}; X_i] against its reflectors (which
 * span the chain's carried coordinates and its own rows), so only the chains' last [P; N] blocks
 * reach the reduction tree (TreeTSPQR over the chains).  Stage 2 walks every chain backwards
 * (Eq. flattspqr_q).  The result is another locally orthogonal representation of the same basis:
 * P, N, t and U agree with the pure tree to rounding.
 *   PQR_CHAINS_AUTO (0) - the library's choice: currently the pure tree (the chained leaf
 *                         kernels measure slower than the tree levels they remove);
 *   PQR_CHAINS_OFF      - pure TreeTSPQR (every leaf block's [P; N] goes to the tree);
 *   PQR_CHAINS_ON       - chains whenever there are more leaf blocks than chains.
 * The plan is fixed at pqr_create (pqr_stats.leaf_chains reports the chain count, 0 = none). */
#define PQR_CHAINS_AUTO 0
#define PQR_CHAINS_OFF  1
#define PQR_CHAINS_ON   2
#define PQR_EXCHANGE_AUTO       0
#define PQR_EXCHANGE_COLLECTIVE 1
#define PQR_EXCHANGE_LSA        2

/* flags of pqr_project_normalize */
#define PQR_NO_APPEND     1u  /* do not append U to the basis (k unchanged)          */
#define PQR_NO_DEFLATION  2u  /* return PQR_EBREAKDOWN instead of deflating (t < s)  */
#define PQR_SINGLE_PASS   4u  /* CHOLQR2 only: one BCGS-PIP pass (Alg. 7), no reiteration */

typedef struct {
  int64_t n_local;      /* rows held by this rank (> 0)                                    */
  int k_max;            /* largest basis width ever appended to (capacity, >= 0)           */
  int s_max;            /* largest block width s (1..16)                                   */
  int variant;          /* pqr_variant                                                     */
  double defl_tol;      /* deflation tolerance relative to ||X||_F; <= 0 selects 1e-12     */
  double gram_eta;      /* CHOLQR2: per-column relative pivot floor eta (R3b);
                           <= 0 selects 1e-13                                              */
  int block_rows;       /* TSQR leaf block rows n_b; 0 = automatic; must be >= k_max+s_max */
  void* stream;         /* cudaStream_t to order all work on; NULL = legacy default stream */
  int rank, nranks;     /* this process's rank and the number of ranks (nranks >= 1)       */
  const void* nccl_id;  /* 128-byte ncclUniqueId (same bytes on all ranks); NULL if nranks==1 */
  void* vgroup;         /* virtual-rank group (pqr_vgroup_create) or NULL.  When set, the
                           nranks handles of this group live in ONE process on one device
                           and exchange through device copies instead of NCCL (see
                           pqr_vgroup_create); nccl_id is then ignored.                     */
  int reduction;        /* PQR_TSQR: PQR_REDUCTION_HH (default) or PQR_REDUCTION_PIP2          */
  int local;            /* PQR_TSQR: PQR_LOCAL_HH (default) or PQR_LOCAL_PIP2                  */
  int exchange;         /* PQR_EXCHANGE_AUTO / _COLLECTIVE / _LSA (NCCL ranks only; ignored for
                           one rank without PQR_FORCE_NCCL and for virtual groups)            */
  int chains;           /* PQR_TSQR: PQR_CHAINS_AUTO (default) / _OFF / _ON (FlatTSPQR leaves)  */
} pqr_config;

/* Create a handle owning the basis (capacity k_max + s_max columns), its workspaces
 * and (nranks > 1) an NCCL communicator built from nccl_id.  The basis is initialised
 * from Q (n_local x k, ldq >= n_local; k = 0 allowed, Q may then be NULL).  Q must
 * have orthonormal columns globally (sum over ranks of Q_r^T Q_r = I).  For PQR_TSQR
 * the explicit Q is converted to the locally orthogonal representation (one TSQR of Q
 * per block, §8(a) a9).  Errors: PQR_EARG, PQR_ECAPACITY, PQR_EPLAN, PQR_ENOMEM,
 * PQR_ECUDA, PQR_ENCCL. */
int pqr_create(pqr_handle* out, const pqr_config* cfg, const double* Q, int64_t ldq, int k);

/* Solve Eq. (1) for the current basis Q (k columns) and X (n_local x s, ldx >= n_local):
 *   U (n_local x s buffer, ldu >= n_local): columns 0..t-1 receive U; may be NULL
 *     unless PQR_NO_APPEND is set (without NO_APPEND, U is always appended to the
 *     basis and can be read back with pqr_basis_apply);
 *   P (k x s, ldp >= max(1,k)) receives P = Q^T X;  may be NULL;
 *   N (s x s, ldn >= s) receives N: t x s row echelon with positive pivots, rows
 *     t..s-1 zero-filled; may be NULL;
 *   *t (HOST int) receives the numerical rank t <= s of the new block.
 * Deflation (t < s) is decided in order, column by column
 * (R3).  flags: PQR_NO_APPEND | PQR_NO_DEFLATION | PQR_SINGLE_PASS.
 * Errors: PQR_EARG, PQR_ECAPACITY, PQR_EBREAKDOWN, PQR_ECUDA, PQR_ENCCL, PQR_ENOMEM. */
int pqr_project_normalize(pqr_handle h, const double* X, int64_t ldx, int s, unsigned flags,
                          double* U, int64_t ldu, double* P, int ldp, double* N, int ldn, int* t);

/* Stage-2 product Y = Q C (§5.1): Q the current basis (n_local x k),
 * C (k x m, ldc >= max(1,k), replicated on every rank), Y (n_local x m, ldy >= n_local).
 * For PQR_TSQR this applies the locally orthogonal representation (§8(a) a8).
 * Errors: PQR_EARG, PQR_ECUDA, PQR_ENOMEM. */
int pqr_basis_apply(pqr_handle h, const double* C, int ldc, int m, double* Y, int64_t ldy);

/* Release the handle, its device memory and its NCCL communicator.  NULL is a no-op. */
int pqr_destroy(pqr_handle h);

/* Static string for an error code. */
const char* pqr_strerror(int code);

/* ---- introspection (counters for tests and the benchmark) ------------------- */
typedef struct {
  int k;                     /* current basis width                                   */
  int last_t;                /* rank of the last solve                                */
  int64_t calls;             /* successful pqr_project_normalize calls                */
  int64_t collectives;       /* NCCL collectives issued (all calls)                   */
  int64_t collective_bytes;  /* bytes sent by this rank in those collectives          */
  int64_t kernel_launches;   /* kernels launched by the library (all calls)           */
  int block_rows;            /* TSQR leaf block rows in use (0 for CHOLQR2)           */
  int tree_levels;           /* TSQR on-GPU tree levels (0 for CHOLQR2)               */
  int exchange;              /* 0 none (one rank), 1 NCCL collective, 2 NCCL device API
                                (LSA), 3 virtual-rank group                              */
  int leaf_chains;           /* TSQR FlatTSPQR leaf chains (0: pure tree)                 */
} pqr_stats;
int pqr_get_stats(pqr_handle h, pqr_stats* st);

/* Per-kernel-kind device timing (CUDA events recorded on the handle's stream around every
 * launch while enabled; read after a call has returned).  Kinds index pqr_profile.ms[]: */
#define PQR_K_GRAM        0   /* a1 fused Gram pass                         */
#define PQR_K_FACTOR      1   /* a3/a5 small factorisation                  */
#define PQR_K_UPDATE      2   /* a4 update pass                             */
#define PQR_K_NCCL        3   /* a2 / C2 cross-GPU exchange                 */
#define PQR_K_TSQR_LOCAL  4   /* a6 TSQR stage-1 local Householder          */
#define PQR_K_TSQR_TREE   5   /* a7 TSQR reduction tree (up + down sweeps)  */
#define PQR_K_TSQR_APPLY  6   /* a8 TSQR stage-2 LOR apply                  */
#define PQR_K_OTHER       7   /* copies / staging                           */
#define PQR_K_UPDATE_GRAM 8   /* a4+a1 fused second CholQR pass              */
#define PQR_NUM_KINDS     9
typedef struct {
  double ms[PQR_NUM_KINDS];       /* summed device milliseconds per kind */
  int64_t launches[PQR_NUM_KINDS];
} pqr_profile;
int pqr_profile_enable(pqr_handle h, int enable);   /* also resets the totals */
int pqr_get_profile(pqr_handle h, pqr_profile* out);

/* ncclGetUniqueId into a 128-byte buffer (rank 0 creates it; the caller broadcasts it). */
int pqr_nccl_unique_id(void* id128);

/* Virtual ranks: a group of nranks handles in ONE process on one device that exchange their
 * small matrices (the (k+s) x s Grams of CholQR2, the (C+s) x s GPU-root blocks of TSQR;
 * PAPER.md:L1130-1166, §5.2) through device-to-device copies ordered by CUDA events, in
 * place of ncclAllGather.  Every handle of the group (pqr_config.vgroup = group, rank =
 * 0..nranks-1) must be created and then driven collectively, each from its own host thread
 * and with its own stream, exactly as the ranks of a multi-GPU job; results are those of an
 * nranks-GPU run on the same row shards (bitwise: P, N, t are identical on every rank).  A
 * rank that stops calling makes its peers' next exchange fail with PQR_ENCCL after 300 s.
 * The caller owns the group: destroy it after every handle of the group.
 * Errors: PQR_EARG (nranks < 1 or out NULL). */
int pqr_vgroup_create(int nranks, void** group);
int pqr_vgroup_destroy(void* group);

#ifdef __cplusplus
}
#endif
#endif /* PQR_H */
