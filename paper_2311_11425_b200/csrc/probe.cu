// Measurement probe (not on the operator path): FP64 FMA peak of the device.
//
// bench.py reports the sweep's FP64 work against a MEASURED DFMA throughput
// (north_star: "FP64 pipe utilisation against peak").  Each thread runs 8
// independent dependent-FMA chains (enough ILP to cover the DFMA latency at
// 8+ warps per SM), the grid is a multiple of the SM count, and the result is
// stored so the compiler cannot drop the chains.  FLOPs = 2 x threads x 8 x iters.
#include <cuda_runtime.h>

#include "hv_common.h"
#include "hv_pow.cuh"

namespace {

__global__ void __launch_bounds__(256) dfma_probe_kernel(double* out, int64_t iters, double b, double c) {
  double a[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) a[r] = 1e-3 * (threadIdx.x + r);
  for (int64_t it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r) a[r] = fma(a[r], b, c);
  }
  double s = 0.0;
#pragma unroll
  for (int r = 0; r < 8; ++r) s += a[r];
  if (s == 12345.678) out[blockIdx.x * blockDim.x + threadIdx.x] = s;   // practically never true
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = s;
}

__global__ void pow_probe_kernel(int64_t n, const double* __restrict__ x, double y, double* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = hv::pow_pos(x[i], y);
}

// mismatches of hv::div_rcp against IEEE division over all (a_i, b_j) pairs of two arrays
__global__ void div_probe_kernel(int64_t n, const double* __restrict__ a, const double* __restrict__ b,
                                 unsigned long long* __restrict__ bad) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double bi = b[i], rb = __drcp_rn(bi);
  unsigned long long c = 0;
  for (int64_t j = 0; j < n; j += 97) {
    const double q0 = a[j] / bi, q1 = hv::div_rcp(a[j], bi, rb);
    if (__double_as_longlong(q0) != __double_as_longlong(q1)) ++c;
  }
  if (c) atomicAdd(bad, c);
}

}  // namespace

extern "C" int hv_probe_div(int64_t n, const double* d_a, const double* d_b, unsigned long long* d_bad, void* stream) {
  if (n <= 0 || !d_a || !d_b || !d_bad) HV_FAIL(HV_ERR_INVALID, "hv_probe_div: bad arguments");
  div_probe_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(n, d_a, d_b, d_bad);
  HV_LAUNCH_CHECK();
  return HV_OK;
}

extern "C" int hv_probe_pow(int64_t n, const double* d_x, double y, double* d_out, void* stream) {
  if (n <= 0 || !d_x || !d_out) HV_FAIL(HV_ERR_INVALID, "hv_probe_pow: bad arguments");
  pow_probe_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(n, d_x, y, d_out);
  HV_LAUNCH_CHECK();
  return HV_OK;
}

extern "C" int hv_probe_dfma(double* d_out, int64_t iters, int blocks, int threads, void* stream) {
  if (!d_out || iters <= 0 || blocks <= 0 || threads <= 0 || threads > 256)
    HV_FAIL(HV_ERR_INVALID, "hv_probe_dfma: bad arguments");
  dfma_probe_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>(d_out, iters, 0.999999, 1e-7);
  HV_LAUNCH_CHECK();
  return HV_OK;
}
