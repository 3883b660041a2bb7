// exchange.cuh — the cross-rank exchange of the small matrices (SURVEY §8(a) a2 and a7,
// §8(e); §5.2): the only data that leaves a rank is a (k+s) x s Gram
// (CholQR2, one per pass) or a GPU root's (C+s) x s top block (TSQR, one per call).  Both
// are all-gathers; every rank then reduces the gathered blocks in rank order itself, so the
// replicas stay bitwise identical (R7).
//
// Two implementations of one interface, chosen at pqr_create:
//   NcclExchange    — one process per GPU, ncclAllGather on the handle's communicator.
//   VirtualExchange — P handles in ONE process on one device ("virtual ranks", each driven
//                     from its own host thread with its own stream).  Rank r publishes its
//                     send buffer and a CUDA event; after a host barrier every rank's
//                     stream waits on the other ranks' events and copies their blocks.  No
//                     kernel ever waits on another rank's kernel (the ordering is carried
//                     by stream-event dependencies), so nothing can deadlock on the device.
//                     It executes every rank >= 1 branch of the library (row offsets of the
//                     cross-GPU tree, nparts = nranks in the factor) with one GPU.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <vector>

namespace pqr {

struct LsaArgs;  // lsa_exchange.cuh

enum { kXNccl = 1, kXLsa = 2, kXVirtual = 3 };  // pqr_stats.exchange

struct Exchange {
  int rank = 0, nranks = 1;
  int kind = 0;
  int64_t calls = 0, bytes = 0;
  virtual ~Exchange() {}
  // NCCL device-API exchange: the arguments a kernel needs to exchange by itself (else nullptr)
  virtual const LsaArgs* lsa() const { return nullptr; }
  // recv[j*count, (j+1)*count) = rank j's send[0, count) for every rank j, ordered on st
  // (send must not be overwritten by later work of this rank before every rank has read
  // it: both implementations guarantee that on the stream).  Returns 0 or a PQR_E* code.
  virtual int allgather(const double* send, double* recv, size_t count, cudaStream_t st) = 0;
};

struct NcclExchange : Exchange {
  ncclComm_t comm = nullptr;
  NcclExchange() { kind = kXNccl; }
  ~NcclExchange() override {
    if (comm) ncclCommDestroy(comm);
  }
  int allgather(const double* send, double* recv, size_t count, cudaStream_t st) override {
    ncclResult_t r = ncclAllGather(send, recv, count, ncclDouble, comm, st);
    if (r != ncclSuccess) {
      fprintf(stderr, "[pqr] ncclAllGather: %s\n", ncclGetErrorString(r));
      return -6;  // PQR_ENCCL
    }
    ++calls;
    bytes += (int64_t)count * 8;
    return 0;
  }
};

// In-process group of P virtual ranks (pqr_vgroup_create).  The host barrier is a
// generation-counting barrier with a timeout (300 s, PQR_VGROUP_TIMEOUT), so a rank that failed before an exchange
// turns its peers' exchange into an error instead of a hang.
struct VirtualGroup {
  int P = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  bool broken = false;
  std::vector<const double*> send;
  std::vector<cudaEvent_t> ready, done;
  explicit VirtualGroup(int p) : P(p), send(p, nullptr), ready(p, nullptr), done(p, nullptr) {}
  // the group owns the ranks' events: a rank whose handle is destroyed (e.g. after a failed
  // call) leaves its events valid for peers that already enqueued waits on them
  ~VirtualGroup() {
    for (auto e : ready)
      if (e) cudaEventDestroy(e);
    for (auto e : done)
      if (e) cudaEventDestroy(e);
  }
  void leave() {  // a member handle is gone: later barriers fail instead of waiting
    std::lock_guard<std::mutex> lk(mu);
    broken = true;
    cv.notify_all();
  }
  bool barrier() {
    std::unique_lock<std::mutex> lk(mu);
    if (broken) return false;
    const uint64_t g = gen;
    if (++arrived == P) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return true;
    }
    static const int tmo = getenv("PQR_VGROUP_TIMEOUT") ? atoi(getenv("PQR_VGROUP_TIMEOUT")) : 300;
    cv.wait_for(lk, std::chrono::seconds(tmo), [&] { return gen != g || broken; });
    if (gen != g) return true;  // this barrier completed (a peer may have left right after it)
    broken = true;              // timeout, or a peer left before arriving
    cv.notify_all();
    return false;
  }
};

struct VirtualExchange : Exchange {
  VirtualGroup* g = nullptr;
  cudaEvent_t ready = nullptr, done = nullptr;
  VirtualExchange() { kind = kXVirtual; }
  ~VirtualExchange() override {
    if (g) g->leave();
  }
  int init(VirtualGroup* grp, int r) {
    g = grp;
    rank = r;
    nranks = grp->P;
    std::lock_guard<std::mutex> lk(g->mu);
    if (g->ready[r] || g->done[r]) return -1;  // PQR_EARG: rank already taken in this group
    if (cudaEventCreateWithFlags(&ready, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&done, cudaEventDisableTiming) != cudaSuccess)
      return -5;  // PQR_ECUDA
    g->ready[r] = ready;
    g->done[r] = done;
    return 0;
  }
  int allgather(const double* send, double* recv, size_t count, cudaStream_t st) override {
    if (cudaEventRecord(ready, st) != cudaSuccess) return -5;
    g->send[rank] = send;
    if (!g->barrier()) return -6;  // every rank has published its block and its event
    for (int j = 0; j < nranks; ++j) {
      if (j != rank && cudaStreamWaitEvent(st, g->ready[j], 0) != cudaSuccess) return -5;
      if (cudaMemcpyAsync(recv + (size_t)j * count, g->send[j], count * sizeof(double), cudaMemcpyDeviceToDevice,
                          st) != cudaSuccess)
        return -5;
    }
    if (cudaEventRecord(done, st) != cudaSuccess) return -5;
    if (!g->barrier()) return -6;  // every rank has enqueued its reads
    // this rank's later work (which may overwrite `send`) waits until every rank has read it
    for (int j = 0; j < nranks; ++j)
      if (j != rank && cudaStreamWaitEvent(st, g->done[j], 0) != cudaSuccess) return -5;
    ++calls;
    bytes += (int64_t)count * 8;
    return 0;
  }
};

}  // namespace pqr
