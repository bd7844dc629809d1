// C-ABI entry points of the hot path: hv_laplacian / hv_hyperdiffusion.
// hyperdiff.py:84-106 semantics; kernel selection (v1 element+CSR, or the tile
// sweep when the plan carries a tile map) happens here.
#include <cuda_runtime.h>

#include "hv_common.h"
#include "lap_common.cuh"

namespace {

__global__ void zero_cols_kernel(double* out, int64_t ng, int64_t ldo, unsigned keep_mask) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= ng * ldo) return;
  const int c = (int)(t % ldo);
  if (!((keep_mask >> c) & 1u)) out[t] = 0.0;
}

int check_plan(const hv_lap_plan* P) {
  if (!P) HV_FAIL(HV_ERR_INVALID, "null plan");
  if (P->N < 1 || P->N > 7) HV_FAIL(HV_ERR_UNSUPPORTED, "laplacian: degree %d not supported on the device (1..7)", P->N);
  if (P->nelem <= 0 || P->nglobal <= 0 || !P->d_gid || !P->d_off || !P->d_idx || !P->d_W || !P->d_Minv ||
      !P->d_work || !P->d_y)
    HV_FAIL(HV_ERR_INVALID, "incomplete laplacian plan");
  return HV_OK;
}

}  // namespace

extern "C" int hv_laplacian(const hv_lap_plan* P, const double* d_q, int64_t ldq, int nf, const int32_t* h_qf,
                            double* d_out, int64_t ldo, const int32_t* h_of, double scale, void* stream) {
  int rc = check_plan(P);
  if (rc) return rc;
  if (nf < 1 || nf > 5 || !d_q || !d_out || !h_qf || !h_of || ldq < 1 || ldo < 1)
    HV_FAIL(HV_ERR_INVALID, "hv_laplacian: bad arguments");
  hv::FieldMap qf{}, of{};
  for (int f = 0; f < nf; ++f) {
    if (h_qf[f] < 0 || h_qf[f] >= ldq || h_of[f] < 0 || h_of[f] >= ldo)
      HV_FAIL(HV_ERR_INVALID, "hv_laplacian: field index out of range");
    qf.f[f] = h_qf[f];
    of.f[f] = h_of[f];
  }
  return hv::laplacian_v1(P, d_q, ldq, nf, qf, d_out, ldo, of, scale, (cudaStream_t)stream);
}

extern "C" int hv_hyperdiffusion(const hv_lap_plan* P, const double* d_q, int64_t ldq, int nvar,
                                 const int32_t* h_vars, int alpha, double* d_out, int64_t ldo, void* stream) {
  int rc = check_plan(P);
  if (rc) return rc;
  if (alpha != 1 && alpha != 2) HV_FAIL(HV_ERR_INVALID, "alpha must be 1 or 2");
  if (nvar < 0 || nvar > 5 || !d_q || !d_out || ldo < 1 || ldo > 32 || ldq < 1)
    HV_FAIL(HV_ERR_INVALID, "hv_hyperdiffusion: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  unsigned keep = 0;
  hv::FieldMap qf{}, of{}, yf{};
  for (int v = 0; v < nvar; ++v) {
    if (h_vars[v] == 0) HV_FAIL(HV_ERR_INVALID, "hyper-diffusing density is out of scope");
    if (h_vars[v] < 0 || h_vars[v] >= ldq || h_vars[v] >= ldo) HV_FAIL(HV_ERR_INVALID, "variable index out of range");
    qf.f[v] = of.f[v] = h_vars[v];
    yf.f[v] = v;
    keep |= 1u << h_vars[v];
  }
  const int64_t tot = P->nglobal * ldo;
  zero_cols_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(d_out, P->nglobal, ldo, nvar ? keep : 0u);
  HV_LAUNCH_CHECK();
  if (nvar == 0) return HV_OK;
  const double sign = (alpha % 2 == 1) ? 1.0 : -1.0;  // (-1)^(alpha+1)
  if (alpha == 1) return hv::laplacian_v1(P, d_q, ldq, nvar, qf, d_out, ldo, of, sign, st);
  rc = hv::laplacian_v1(P, d_q, ldq, nvar, qf, P->d_y, nvar, yf, 1.0, st);
  if (rc) return rc;
  return hv::laplacian_v1(P, P->d_y, nvar, nvar, yf, d_out, ldo, of, sign, st);
}
