// Microbenchmarks for design decisions (not part of the product path):
// HBM read / copy bandwidth, fp64 DFMA issue rate, fp64 DMMA (mma.sync f64) rates.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void k_read(const double2* __restrict__ a, size_t n2, double* out) {
  double2 acc = make_double2(0, 0);
  size_t stride = (size_t)gridDim.x * blockDim.x;
  #pragma unroll 8
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += stride) {
    double2 v = __ldcs(a + i); acc.x += v.x; acc.y += v.y;
  }
  if (acc.x == 1234.5) out[0] = acc.y;
}
__global__ void k_copy(const double2* __restrict__ a, double2* __restrict__ b, size_t n2) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  #pragma unroll 4
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += stride) b[i] = __ldcs(a + i);
}
__global__ void k_dfma(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
    x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
    x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
  }
  double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 1.2345) out[0] = s;
}
__device__ __forceinline__ void mma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__global__ void k_dmma884(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double d[8][2];
  #pragma unroll
  for (int j = 0; j < 8; ++j) d[j][0] = d[j][1] = 0;
  for (int i = 0; i < iters; ++i) {
    #pragma unroll
    for (int j = 0; j < 8; ++j) mma884(d[j][0], d[j][1], a, b);
  }
  double s = 0;
  #pragma unroll
  for (int j = 0; j < 8; ++j) s += d[j][0] + d[j][1];
  if (s == 1.2345) out[0] = s;
}
__device__ __forceinline__ void mma16816(double* d, const double* a, const double* b) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                 "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}
__global__ void k_dmma16816(double* out, int iters) {
  double a[8], b[4];
  #pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = (threadIdx.x + j) * 1e-3;
  #pragma unroll
  for (int j = 0; j < 4; ++j) b[j] = 1.0 - (threadIdx.x + j) * 1e-4;
  double d[4][4];
  #pragma unroll
  for (int j = 0; j < 4; ++j) d[j][0] = d[j][1] = d[j][2] = d[j][3] = 0;
  for (int i = 0; i < iters; ++i) {
    #pragma unroll
    for (int j = 0; j < 4; ++j) mma16816(d[j], a, b);
  }
  double s = 0;
  #pragma unroll
  for (int j = 0; j < 4; ++j) s += d[j][0] + d[j][1] + d[j][2] + d[j][3];
  if (s == 1.2345) out[0] = s;
}

// DFMA and DMMA issued together: do the two fp64 pipes add up?  (mode 0: every warp
// interleaves both; mode 1: even warps DMMA only, odd warps DFMA only)
__global__ void k_mixed(double* out, int iters, int mode) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double d[8][2];
  #pragma unroll
  for (int j = 0; j < 8; ++j) d[j][0] = d[j][1] = 0;
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  const int warp = threadIdx.x >> 5;
  const bool do_mma = mode == 0 || (warp & 1) == 0, do_fma = mode == 0 || (warp & 1) == 1;
  for (int i = 0; i < iters; ++i) {
    if (do_mma) {
      #pragma unroll
      for (int j = 0; j < 8; ++j) mma884(d[j][0], d[j][1], a, b);
    }
    if (do_fma) {
      #pragma unroll
      for (int r = 0; r < 8; ++r) {
        x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
        x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
      }
    }
  }
  double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  #pragma unroll
  for (int j = 0; j < 8; ++j) s += d[j][0] + d[j][1];
  if (s == 1.2345) out[0] = s;
}
__global__ void k_clock(long long* out, int iters, double a) {
  long long t0 = clock64();
  double x = threadIdx.x;
  for (int i = 0; i < iters; ++i) x = fma(x, a, 1e-9);
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (x == 1.2345) out[0] = 0;
}

int main() {
  int dev = 0; cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, dev));
  int sms = prop.multiProcessorCount;
  int l2 = 0; cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
  int smem = 0; cudaDeviceGetAttribute(&smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  printf("{\"name\":\"%s\",\"sms\":%d,\"l2_bytes\":%d,\"smem_optin\":%d,\"cc\":\"%d.%d\"}\n", prop.name, sms, l2, smem, prop.major, prop.minor);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  size_t bytes = (size_t)8 << 30;  // 8 GiB
  double *a, *b, *out; CK(cudaMalloc(&a, bytes)); CK(cudaMalloc(&b, bytes)); CK(cudaMalloc(&out, 64));
  CK(cudaMemset(a, 0, bytes)); CK(cudaMemset(b, 0, bytes));
  size_t n2 = bytes / 16;
  for (int occ : {4, 8, 16}) {
    float best = 1e30f;
    for (int r = 0; r < 6; ++r) {
      cudaEventRecord(e0); k_read<<<sms * occ, 256>>>((const double2*)a, n2, out); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (r && ms < best) best = ms;
    }
    printf("{\"test\":\"read\",\"ctas_per_sm\":%d,\"GBps\":%.1f}\n", occ, bytes / best / 1e6);
  }
  {
    float best = 1e30f;
    for (int r = 0; r < 6; ++r) {
      cudaEventRecord(e0); k_copy<<<sms * 8, 256>>>((const double2*)a, (double2*)b, n2 / 2); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (r && ms < best) best = ms;
    }
    printf("{\"test\":\"copy\",\"GBps\":%.1f}\n", bytes / best / 1e6);
  }
  // clock estimate
  {
    long long* clk; CK(cudaMalloc(&clk, sizeof(long long) * sms));
    int iters = 1 << 20;
    cudaEventRecord(e0); k_clock<<<sms, 32>>>(clk, iters, 0.999); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long h; cudaMemcpy(&h, clk, sizeof(h), cudaMemcpyDeviceToHost);
    printf("{\"test\":\"clock\",\"cycles\":%lld,\"ms\":%.3f,\"MHz\":%.0f}\n", h, ms, h / (ms * 1e3));
  }
  for (int threads : {256, 512}) {
    int iters = 1 << 14;
    float best = 1e30f;
    for (int r = 0; r < 4; ++r) {
      cudaEventRecord(e0); k_dfma<<<sms * 4, threads>>>(out, iters, 0.999, 1e-9); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (r && ms < best) best = ms;
    }
    double flops = 2.0 * 8 * iters * (double)sms * 4 * threads;
    printf("{\"test\":\"dfma\",\"threads\":%d,\"TFLOPs\":%.2f}\n", threads, flops / best / 1e9);
  }
  for (int threads : {128, 256, 512}) {
    int iters = 1 << 12;
    float best = 1e30f;
    for (int r = 0; r < 4; ++r) {
      cudaEventRecord(e0); k_dmma884<<<sms * 4, threads>>>(out, iters); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (r && ms < best) best = ms;
    }
    double flops = 2.0 * 256 * 8 * iters * (double)sms * 4 * (threads / 32);
    printf("{\"test\":\"dmma_m8n8k4\",\"threads\":%d,\"TFLOPs\":%.2f}\n", threads, flops / best / 1e9);
  }
  for (int threads : {128, 256, 512}) {
    int iters = 1 << 11;
    float best = 1e30f;
    for (int r = 0; r < 4; ++r) {
      cudaEventRecord(e0); k_dmma16816<<<sms * 4, threads>>>(out, iters); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (r && ms < best) best = ms;
    }
    double flops = 2.0 * 16 * 8 * 16 * 4 * iters * (double)sms * 4 * (threads / 32);
    printf("{\"test\":\"dmma_m16n8k16\",\"threads\":%d,\"TFLOPs\":%.2f}\n", threads, flops / best / 1e9);
  }
  for (int mode : {0, 1}) {
    int iters = 1 << 11, threads = 512;
    float best = 1e30f;
    for (int r = 0; r < 4; ++r) {
      cudaEventRecord(e0); k_mixed<<<sms * 2, threads>>>(out, iters, mode); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (r && ms < best) best = ms;
    }
    // per iteration and warp: 8 DMMA (2*256*8 flop) and/or 64 DFMA per lane (2*64*32 flop)
    double warps = (double)sms * 2 * (threads / 32);
    double per_warp = mode == 0 ? 2.0 * 256 * 8 + 2.0 * 64 * 32 : 0.5 * (2.0 * 256 * 8 + 2.0 * 64 * 32);
    printf("{\"test\":\"dmma+dfma\",\"mode\":%d,\"TFLOPs\":%.2f}\n", mode, per_warp * iters * warps / best / 1e9);
  }
  CK(cudaGetLastError());
  return 0;
}
