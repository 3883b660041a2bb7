// lsa_exchange.cuh — the cross-GPU exchange through the NCCL device API (
// PAPER.md:L1160-1166, §5.2, and L1546-1552, §7: the reduction as a stateful, in-network step
// rather than a separate message-passing call).
//
// Every rank's small block (a (k+s) x s Gram of CholQR2, or a GPU root's (C+s) x s block of
// TSQR) is stored by a kernel straight into every peer's slot of a symmetric NCCL window over
// NVLink (load/store accessible "LSA" team = the ranks of this NVSwitch domain), followed by an
// LSA barrier; each rank then reads all slots from its own copy of the window in rank order.
// For CholQR2 this happens inside the factor kernel itself (k_factor_lsa): Gram kernel ->
// factor kernel, with no NCCL launch, proxy or host involvement between them.
//
// Window layout (doubles): [2 halves][nranks slots][slot], slot >= the largest block.  Exchange
// number q (a device-resident counter, so CUDA-graph replays stay consistent) uses half q & 1.
// Reuse is safe with two halves: a rank writes half h again only at exchange q + 2, after it
// passed barrier q + 1, which every peer enters only after it finished reading exchange q.
#pragma once
#include <nccl.h>
#include <nccl_device.h>

#include "cholqr_kernels.cuh"

namespace pqr {

struct LsaArgs {
  ncclDevComm dc;
  ncclWindow_t win;
  int rank, nranks;  // LSA rank / size (the LSA team is the whole communicator, checked at setup)
  int64_t slot;      // doubles per rank slot
  int* seq;          // exchange counter (device)
};

// One CTA: put `count` doubles of `send` (device memory of this rank) into slot [half][rank] of
// every rank's window, then the LSA barrier.  Returns this rank's local pointer to half `half`.
__device__ __forceinline__ const double* lsa_put_barrier(const LsaArgs& l, const double* send, int64_t count,
                                                         int half) {
  const size_t off = ((size_t)half * l.nranks + l.rank) * (size_t)l.slot * sizeof(double);
  for (int64_t e = threadIdx.x; e < (int64_t)l.nranks * count; e += blockDim.x) {
    const int peer = (int)(e / count);
    const int64_t i = e - (int64_t)peer * count;
    double* dst = reinterpret_cast<double*>(ncclGetLsaPointer(l.win, off, peer));
    dst[i] = __ldcg(send + i);
  }
  {
    // arrive: CTA barrier, then a system-scope release store into every peer's inbox; wait:
    // acquire loads of this rank's inboxes (nccl_device/impl/lsa_barrier__funcs.h)
    ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), l.dc, ncclTeamTagLsa(), 0);
    bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
  }
  return reinterpret_cast<const double*>(ncclGetLocalPointer(l.win, (size_t)half * l.nranks * l.slot * sizeof(double)));
}

__device__ __forceinline__ void lsa_advance(const LsaArgs& l) {
  __syncthreads();
  if (threadIdx.x == 0) *l.seq += 1;
}

// a2 + a3 fused (CholQR2): this rank's Gram a.W (m x s, ld a.ldw = m) goes to every rank; the
// factor then sums the nranks Grams in rank order from the local window (R7).
__global__ void __launch_bounds__(256) k_factor_lsa(FactorArgs a, LsaArgs l) {
  const int half = *(volatile int*)l.seq & 1;
  const double* base = lsa_put_barrier(l, a.W, (int64_t)a.ldw * a.s, half);
  FactorArgs f = a;
  f.W = base;
  f.w_stride = l.slot;
  f.nparts = l.nranks;
  factor_body(f);
  lsa_advance(l);
}

// a7 (TSQR, Householder reduction): the all-gather of the GPU roots' blocks as one kernel.
__global__ void __launch_bounds__(256) k_lsa_allgather(LsaArgs l, const double* send, double* recv, int64_t count) {
  const int half = *(volatile int*)l.seq & 1;
  const double* base = lsa_put_barrier(l, send, count, half);
  for (int64_t e = threadIdx.x; e < (int64_t)l.nranks * count; e += blockDim.x) {
    const int r = (int)(e / count);
    const int64_t i = e - (int64_t)r * count;
    recv[e] = __ldcg(base + (size_t)r * l.slot + i);
  }
  lsa_advance(l);
}

}  // namespace pqr

namespace pqr {

// Host side: the communicator of NcclExchange plus a symmetric window of 2 x nranks slots, a
// device communicator with one LSA barrier, and the exchange counter.  allgather() (TSQR) is one
// k_lsa_allgather launch; CholQR2 passes lsa() to k_factor_lsa instead of calling allgather().
struct LsaExchange : NcclExchange {
  void* buf = nullptr;
  ncclWindow_t win = nullptr;
  ncclDevComm dc{};
  bool dc_ok = false;
  LsaArgs args{};
  LsaExchange() { kind = kXLsa; }
  ~LsaExchange() override {
    if (dc_ok) ncclDevCommDestroy(comm, &dc);
    if (win) ncclCommWindowDeregister(comm, win);
    if (buf) ncclMemFree(buf);
    if (args.seq) cudaFree(args.seq);
  }
  const LsaArgs* lsa() const override { return &args; }
  // collective over the communicator (every rank, same slot); 0 or PQR_ENCCL / PQR_ENOMEM
  int setup(int64_t slot_doubles) {
    const ncclTeam_t lsa_team = ncclTeamLsa(comm);
    if (lsa_team.nRanks != nranks) {
      fprintf(stderr, "[pqr] LSA exchange needs all %d ranks in one NVLink domain (LSA team: %d)\n", nranks,
              lsa_team.nRanks);
      return -6;
    }
    const size_t bytes = (size_t)2 * nranks * slot_doubles * sizeof(double);
    ncclResult_t r = ncclMemAlloc(&buf, bytes);
    if (r != ncclSuccess) {
      fprintf(stderr, "[pqr] ncclMemAlloc: %s\n", ncclGetErrorString(r));
      buf = nullptr;
      return -7;
    }
    if (cudaMemset(buf, 0, bytes) != cudaSuccess) return -5;
    r = ncclCommWindowRegister(comm, buf, bytes, &win, NCCL_WIN_COLL_SYMMETRIC);
    if (r != ncclSuccess) {
      fprintf(stderr, "[pqr] ncclCommWindowRegister: %s\n", ncclGetErrorString(r));
      win = nullptr;
      return -6;
    }
    ncclDevCommRequirements reqs;
    memset(&reqs, 0, sizeof(reqs));
    reqs.lsaBarrierCount = 1;
    r = ncclDevCommCreate(comm, &reqs, &dc);
    if (r != ncclSuccess) {
      fprintf(stderr, "[pqr] ncclDevCommCreate: %s\n", ncclGetErrorString(r));
      return -6;
    }
    dc_ok = true;
    if (cudaMalloc(&args.seq, sizeof(int)) != cudaSuccess) {
      args.seq = nullptr;
      return -7;
    }
    if (cudaMemset(args.seq, 0, sizeof(int)) != cudaSuccess) return -5;
    args.dc = dc;
    args.win = win;
    args.rank = lsa_team.rank;
    args.nranks = nranks;
    args.slot = slot_doubles;
    return 0;
  }
  int allgather(const double* send, double* recv, size_t count, cudaStream_t st) override {
    if ((int64_t)count > args.slot) return -1;
    k_lsa_allgather<<<1, 256, 0, st>>>(args, send, recv, (int64_t)count);
    if (cudaGetLastError() != cudaSuccess) return -5;
    ++calls;
    bytes += (int64_t)count * 8;
    return 0;
  }
};

}  // namespace pqr
