// common.cuh — device helpers shared by the libpqr kernels (sm_100a, fp64).
//
// The fp64 tensor-core instruction used throughout is the warp-level
// mma.sync.aligned.m8n8k4.row.col.f64 (SASS: DMMA.8).  On B200 its measured
// throughput equals the DFMA pipe's (37.0 vs 33.8 TFLOP/s fp64, see
// profiles/r01_microbench.md) but it issues 1/256 of the instructions and keeps
// the k-reduction inside the unit, which is what makes a one-warp-per-row-slab
// tall-skinny Gram / update fit in the register file.
//
// Fragment layout (PTX ISA, m8n8k4 .f64; lane l, g = l>>2, q = l&3):
//   A (8x4, row):  a0 = A[g][q]
//   B (4x8, col):  b0 = B[q][g]
//   C/D (8x8):     c0 = C[g][2q], c1 = C[g][2q+1]
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>
#include <unordered_map>

#define PQR_DEV __device__ __forceinline__
#define PQR_HOST_DEV __host__ __device__ __forceinline__

namespace pqr {

constexpr int kWarp = 32;

PQR_DEV void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// Streaming 16-byte load of two consecutive rows of one column (read-only path).
PQR_DEV double2 ld2(const double* p) { return __ldg(reinterpret_cast<const double2*>(p)); }
PQR_DEV double2 ld2_stream(const double* p) { return __ldcs(reinterpret_cast<const double2*>(p)); }

PQR_DEV double2 lds2(const double* p) { return *reinterpret_cast<const double2*>(p); }

PQR_DEV void st2(double* p, double x, double y) { *reinterpret_cast<double2*>(p) = make_double2(x, y); }

// Column pointer of A = [Q X] (Q: columns 0..k-1, X: columns k..m-1); nullptr past m.
PQR_DEV const double* col_ptr(const double* Q, int64_t ldq, const double* X, int64_t ldx, int k, int m, int j) {
  if (j < k) return Q + (int64_t)j * ldq;
  if (j < m) return X + (int64_t)(j - k) * ldx;
  return nullptr;
}

// Guarded two-row load for ragged tails: rows r, r+1 of column c (nullptr -> 0).
PQR_DEV double2 ld2_guard(const double* c, int64_t r, int64_t n) {
  double2 v = make_double2(0.0, 0.0);
  if (c) {
    if (r < n) v.x = __ldg(c + r);
    if (r + 1 < n) v.y = __ldg(c + r + 1);
  }
  return v;
}

}  // namespace pqr

// ---------------------------------------------------------------------------
// TMA bulk copies (cp.async.bulk, SASS UBLKCP) + mbarrier pipeline primitives
// ---------------------------------------------------------------------------
namespace pqr {

PQR_DEV uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

PQR_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
PQR_DEV void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
PQR_DEV void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

PQR_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
PQR_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
PQR_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// as mbar_wait, sleeping between polls (waits of a producer or an idle group: less power)
PQR_DEV void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  while (!ok) {
    __nanosleep(128);
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}
// global -> shared bulk copy completing on an mbarrier (bytes % 16 == 0, both addresses 16-B aligned)
PQR_DEV void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

}  // namespace pqr

// ---------------------------------------------------------------------------
// cp.async (LDGSTS) 16-byte global->shared copies with zero fill
// ---------------------------------------------------------------------------
namespace pqr {
// copies `src_bytes` (0, 8 or 16) bytes and zero-fills the rest of the 16-byte chunk
PQR_DEV void cp_async16(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)), "l"(src), "r"(src_bytes)
               : "memory");
}
// bulk prefetch of [p, p + bytes) into L2 (bytes % 16 == 0, p 16-B aligned)
PQR_DEV void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p), "r"(bytes) : "memory");
}
// cp.async 8-byte global->shared copy (LDGSTS, L1-allocating)
PQR_DEV void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
// L2 evict-last policy (small data re-read long after it is written, under a streaming load)
PQR_DEV uint64_t l2_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
PQR_DEV void st_l2pol(double* p, double v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;\n" ::"l"(p), "d"(v), "l"(pol) : "memory");
}
PQR_DEV void cp_async8_l2pol(void* dst, const void* src, uint64_t pol) {
  asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2;\n" ::"r"(smem_u32(dst)), "l"(src), "l"(pol)
               : "memory");
}
// as cp_async16 with a 32-bit shared-memory address
PQR_DEV void cp_async16_s(uint32_t dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
PQR_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
PQR_DEV void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
}  // namespace pqr

namespace pqr {
// wait until at most n of this thread's most recent cp.async groups are pending (n <= 14)
PQR_DEV void cp_async_wait_dyn(int n) {
  switch (n) {
    case 0: cp_async_wait<0>(); break;
    case 1: cp_async_wait<1>(); break;
    case 2: cp_async_wait<2>(); break;
    case 3: cp_async_wait<3>(); break;
    case 4: cp_async_wait<4>(); break;
    case 5: cp_async_wait<5>(); break;
    case 6: cp_async_wait<6>(); break;
    case 7: cp_async_wait<7>(); break;
    case 8: cp_async_wait<8>(); break;
    case 9: cp_async_wait<9>(); break;
    case 10: cp_async_wait<10>(); break;
    case 11: cp_async_wait<11>(); break;
    case 12: cp_async_wait<12>(); break;
    case 13: cp_async_wait<13>(); break;
    default: cp_async_wait<14>(); break;
  }
}
}  // namespace pqr

namespace pqr {
// the mbarrier receives one (non-incrementing) arrival once all of this thread's prior
// cp.async copies have landed
PQR_DEV void cp_async_mbar_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
}  // namespace pqr

namespace pqr {
// Grid reduction by the last CTA: W(j, c) = sum over the nb per-CTA partials (ms = m*s entries,
// column-major m x s each, at partials + b*ms).  Partial b goes to accumulator b % 4, the four
// are combined as (a0 + a1) + (a2 + a3): a fixed order, so results are bitwise reproducible.
// 16 independent L2 loads per thread are in flight per step (the reduction is latency-bound).
PQR_DEV void grid_sum_partials(const double* partials, int nb, int ms, int m, double* W, int ldw, int tid,
                               int nthr) {
  for (int e = tid; e < ms; e += nthr) {
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    int b = 0;
    for (; b + 16 <= nb; b += 16) {
      double v[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) v[u] = __ldcg(partials + (size_t)(b + u) * ms + e);
#pragma unroll
      for (int u = 0; u < 16; ++u) acc[u & 3] += v[u];
    }
    for (; b < nb; b += 4) {  // b is a multiple of 4 here: partial b + u goes to acc[u]
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (b + u < nb) acc[u] += __ldcg(partials + (size_t)(b + u) * ms + e);
    }
    const int jj = e % m, c = e / m;
    W[jj + (int64_t)c * ldw] = (acc[0] + acc[1]) + (acc[2] + acc[3]);
  }
}
PQR_DEV void grid_sum_partials(const double* partials, int nb, int ms, int m, double* W, int ldw) {
  grid_sum_partials(partials, nb, ms, m, W, ldw, threadIdx.x, blockDim.x);
}
}  // namespace pqr

namespace pqr {
// Host: raise a kernel's dynamic shared-memory limit to `bytes` once (cached per kernel, so
// repeated launches do not pay a cudaFuncSetAttribute call each).
template <typename K>
inline cudaError_t ensure_smem(K kern, size_t bytes) {
  static std::mutex mu;
  static std::unordered_map<const void*, size_t> done;
  const void* key = reinterpret_cast<const void*>(kern);
  std::lock_guard<std::mutex> lock(mu);
  auto it = done.find(key);
  if (it != done.end() && it->second >= bytes) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) done[key] = bytes;
  return e;
}
}  // namespace pqr
