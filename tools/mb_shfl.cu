// microbenchmark: LDS.64 vs SHFL (64-bit) throughput and whether they share a pipe
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(double* out, int iters) {
  __shared__ double s[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) s[i] = i * 0.5;
  __syncthreads();
  double a0 = threadIdx.x, a1 = 1.0, a2 = 2.0, a3 = 3.0;
  const int lane = threadIdx.x & 31;
  int base = (threadIdx.x / 32) * 64 + lane;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      if (MODE == 0 || MODE == 2) {
        a0 += s[(base + r * 32) & 2047];
        a1 += s[(base + r * 32 + 1024) & 2047];
      }
      if (MODE == 1 || MODE == 2) {
        a2 += __shfl_sync(0xffffffff, a2, (lane + r + 1) & 31);
        a3 += __shfl_sync(0xffffffff, a3, (lane + 7 * r + 3) & 31);
      }
    }
    base += 3;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3;
}
int main() {
  double* o;
  cudaMalloc(&o, 148 * 8 * 1024 * 8);
  int dev; cudaGetDevice(&dev); int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4096, T = 512, B = 148 * 4;
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) k<0><<<B, T>>>(o, iters);
      if (mode == 1) k<1><<<B, T>>>(o, iters);
      if (mode == 2) k<2><<<B, T>>>(o, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double warp_ops = (double)B * T / 32 * iters * 8 * 2;   // per kind
      double cyc = ms * 1e-3 * 1.965e9;
      if (rep) printf("mode %d: %.3f ms, %.3f warp-ops(64b) per SM-cycle per kind\n", mode, ms, warp_ops / 148 / cyc);
    }
  }
  return 0;
}
