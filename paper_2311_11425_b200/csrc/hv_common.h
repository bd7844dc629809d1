// Shared helpers for the hv_b200 C-ABI library (host + device).
#pragma once
#include <cstdint>
#include <cstdio>
#include <string>

#include "../../include/hv_b200.h"

namespace hv {

// Thread-local last error string behind hv_last_error().
void set_error(const char* fmt, ...);

// Process-wide count of kernels launched by this library (hv_launch_count()).
void count_launch(int64_t k = 1);

}  // namespace hv

#define HV_FAIL(code, ...)            \
  do {                                \
    ::hv::set_error(__VA_ARGS__);     \
    return (code);                    \
  } while (0)

#define HV_CUDA_CHECK(expr)                                                              \
  do {                                                                                   \
    cudaError_t _e = (expr);                                                             \
    if (_e != cudaSuccess) {                                                             \
      (void)cudaGetLastError(); /* clear a non-sticky error so later launches are clean */ \
      HV_FAIL(HV_ERR_CUDA, "%s:%d %s -> %s", __FILE__, __LINE__, #expr, cudaGetErrorString(_e)); \
    }                                                                                    \
  } while (0)

#define HV_LAUNCH_CHECK()                                                                \
  do {                                                                                   \
    ::hv::count_launch();                                                                \
    cudaError_t _e = cudaGetLastError();                                                 \
    if (_e != cudaSuccess)                                                               \
      HV_FAIL(HV_ERR_CUDA, "%s:%d kernel launch -> %s", __FILE__, __LINE__, cudaGetErrorString(_e)); \
  } while (0)
