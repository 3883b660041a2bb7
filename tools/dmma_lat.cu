// DMMA (mma.sync m8n8k4 f64) latency and throughput vs. warps per SM sub-partition and
// independent accumulator chains per warp (tuning aid for the fused CholQR2 pass).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void mma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int C>
__global__ void k_chain(double* out, int iters, long long* cyc) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double d[C][2];
#pragma unroll
  for (int j = 0; j < C; ++j) d[j][0] = d[j][1] = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < C; ++j) mma884(d[j][0], d[j][1], a, b);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int j = 0; j < C; ++j) s += d[j][0] + d[j][1];
  if (s == 1.2345) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int C>
void run(int warps_per_sm, double* out, long long* cyc, int sms) {
  const int iters = 20000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  k_chain<C><<<sms, 32 * warps_per_sm>>>(out, 100, cyc);
  cudaEventRecord(e0);
  k_chain<C><<<sms, 32 * warps_per_sm>>>(out, iters, cyc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  const double flops = 512.0 * C * iters * warps_per_sm * sms;
  printf("{\"chains\":%d,\"warps_per_sm\":%d,\"TFLOPs\":%.2f,\"cycles_per_dmma_per_warp\":%.2f}\n", C, warps_per_sm,
         flops / ms / 1e9, (double)h / (iters * (double)C));
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; long long* cyc;
  cudaMalloc(&out, 8); cudaMalloc(&cyc, 8);
  for (int w : {4, 8, 16}) {
    run<1>(w, out, cyc, sms); run<2>(w, out, cyc, sms); run<4>(w, out, cyc, sms); run<8>(w, out, cyc, sms);
  }
  return 0;
}
