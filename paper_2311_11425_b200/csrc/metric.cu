// One-time setup kernels (sm_100a, fp64): element metric terms, lumped mass,
// column projection and the viscous metric / packed Laplacian metric.
//
// Reference: metrics.py:49-142, assembly.py:54-64, hyperdiff.py:54-81,
// euler.py:34-42.  The element metric kernel is rounding-faithful to numpy's
// einsum order (metric_math.h); the DSS sums run through the CSR map in flat
// order, reproducing np.add.at bit for bit.
#include <cuda_runtime.h>

#include <cmath>
#include <vector>

#include "hv_common.h"
#include "lap_common.cuh"
#include "metric_math.h"

namespace {

__device__ unsigned int g_setup_flags[4];  // [0]: J<=0, [1]: eig<=0, [2]: M<=0, [3]: mass==0

struct DMat {
  double v[81];
};

struct DevBarrier {
  __device__ void operator()() const { __syncthreads(); }
};

template <int n>
__global__ void __launch_bounds__(256) metric_kernel(int scheme, DMat Dm, const double* __restrict__ coords,
                                                     int64_t nelem, double* __restrict__ dx_out,
                                                     double* __restrict__ J_out, double* __restrict__ grad_out) {
  constexpr int nn = n * n * n;
  extern __shared__ double sm[];
  double* sD = sm;                 // n*n
  double* X = sD + n * n;          // 3 nn
  double* dx = X + 3 * nn;         // 9 nn
  double* J = dx + 9 * nn;         // nn
  double* A = J + nn;              // 9 nn
  double* grad = A + 9 * nn;       // 9 nn
  const int64_t e = blockIdx.x;
  if (e >= nelem) return;
  for (int t = threadIdx.x; t < n * n; t += blockDim.x) sD[t] = Dm.v[t];
  const double* ce = coords + e * 3 * nn;
  for (int t = threadIdx.x; t < 3 * nn; t += blockDim.x) X[t] = ce[t];
  __syncthreads();
  hv::element_metrics<n>(scheme, sD, X, dx, J, A, grad, threadIdx.x, blockDim.x, DevBarrier{});
  __syncthreads();
  for (int t = threadIdx.x; t < nn; t += blockDim.x) {
    J_out[e * nn + t] = J[t];
    if (!(J[t] > 0.0)) atomicOr(&g_setup_flags[0], 1u);
  }
  for (int t = threadIdx.x; t < 9 * nn; t += blockDim.x) {
    grad_out[e * 9 * nn + t] = grad[t];
    if (dx_out) dx_out[e * 9 * nn + t] = dx[t];
  }
}

__global__ void dss_csr_kernel(const double* __restrict__ fe, int ncomp, int64_t cstride,
                               const int64_t* __restrict__ off, const int32_t* __restrict__ idx, int64_t ng,
                               double* __restrict__ out) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= ng) return;
  const int64_t o0 = off[g], o1 = off[g + 1];
  for (int c = 0; c < ncomp; ++c) {
    double s = 0.0;
    for (int64_t o = o0; o < o1; ++o) s = __dadd_rn(s, fe[c * cstride + idx[o]]);
    out[g * ncomp + c] = s;
  }
}

// mass = DSS(w3 J); Jg = DSS((w3 J) J)/mass; gz_c = DSS((w3 J) grad[2][c])/mass
// (assembly.py:57-61, metrics.py:121-142), each sum sequential in flat order.
__global__ void mass_proj_kernel(int nn, const double* __restrict__ w3, const double* __restrict__ J,
                                 const double* __restrict__ grad, const int64_t* __restrict__ off,
                                 const int32_t* __restrict__ idx, int64_t ng, double* __restrict__ M,
                                 double* __restrict__ Minv, double* __restrict__ Jg, double* __restrict__ gz) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= ng) return;
  const int64_t o0 = off[g], o1 = off[g + 1];
  double m = 0.0, sj = 0.0, s0 = 0.0, s1 = 0.0, s2 = 0.0;
  for (int64_t o = o0; o < o1; ++o) {
    const int64_t p = idx[o];
    const int64_t e = p / nn, r = p % nn;
    const double Jp = J[p];
    const double wj = __dmul_rn(w3[r], Jp);
    m = __dadd_rn(m, wj);
    if (Jg) {
      sj = __dadd_rn(sj, __dmul_rn(wj, Jp));
      const double* gze = grad + (e * 9 + 6) * nn + r;   // grad[e][2][c][r]
      s0 = __dadd_rn(s0, __dmul_rn(wj, gze[0]));
      s1 = __dadd_rn(s1, __dmul_rn(wj, gze[nn]));
      s2 = __dadd_rn(s2, __dmul_rn(wj, gze[2 * nn]));
    }
  }
  M[g] = m;
  Minv[g] = __ddiv_rn(1.0, m);
  if (!(m > 0.0)) atomicOr(&g_setup_flags[2], 1u);
  if (m == 0.0) atomicOr(&g_setup_flags[3], 1u);
  if (Jg) {
    Jg[g] = __ddiv_rn(sj, m);
    gz[g * 3 + 0] = __ddiv_rn(s0, m);
    gz[g * 3 + 1] = __ddiv_rn(s1, m);
    gz[g * 3 + 2] = __ddiv_rn(s2, m);
  }
}

// Raw flat-order sums per node: [sum w3J, sum (w3J)J, sum (w3J) gz_c] (the numerators of
// GlobalMass / project_metrics_to_columns before any cross-rank addition).
__global__ void mass_proj_sums_kernel(int nn, const double* __restrict__ w3, const double* __restrict__ J,
                                      const double* __restrict__ grad, const int64_t* __restrict__ off,
                                      const int32_t* __restrict__ idx, int64_t ng, double* __restrict__ S) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= ng) return;
  double m = 0.0, sj = 0.0, s0 = 0.0, s1 = 0.0, s2 = 0.0;
  for (int64_t o = off[g]; o < off[g + 1]; ++o) {
    const int64_t p = idx[o];
    const int64_t e = p / nn, r = p % nn;
    const double Jp = J[p];
    const double wj = __dmul_rn(w3[r], Jp);
    m = __dadd_rn(m, wj);
    sj = __dadd_rn(sj, __dmul_rn(wj, Jp));
    const double* gze = grad + (e * 9 + 6) * nn + r;
    s0 = __dadd_rn(s0, __dmul_rn(wj, gze[0]));
    s1 = __dadd_rn(s1, __dmul_rn(wj, gze[nn]));
    s2 = __dadd_rn(s2, __dmul_rn(wj, gze[2 * nn]));
  }
  S[g * 5 + 0] = m;
  S[g * 5 + 1] = sj;
  S[g * 5 + 2] = s0;
  S[g * 5 + 3] = s1;
  S[g * 5 + 4] = s2;
}

__global__ void mass_proj_finalize_kernel(int64_t ng, const double* __restrict__ S, double* __restrict__ M,
                                          double* __restrict__ Minv, double* __restrict__ Jg, double* __restrict__ gz) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= ng) return;
  const double m = S[g * 5];
  M[g] = m;
  Minv[g] = __ddiv_rn(1.0, m);
  if (!(m > 0.0)) atomicOr(&g_setup_flags[2], 1u);
  if (m == 0.0) atomicOr(&g_setup_flags[3], 1u);
  if (Jg) {
    Jg[g] = __ddiv_rn(S[g * 5 + 1], m);
#pragma unroll
    for (int c = 0; c < 3; ++c) gz[g * 3 + c] = __ddiv_rn(S[g * 5 + 2 + c], m);
  }
}

// Cyclic Jacobi eigensolver for a symmetric 3x3 matrix; eigenvalues ascending,
// V columns = eigenvectors (LAPACK dsyevd's convention for ordering; signs and
// degenerate-eigenspace bases are arbitrary, the reference only relies on
// E^T E = I and the reconstruction).
__device__ void jacobi3(double a[3][3], double w[3], double V[3][3]) {
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) V[r][c] = (r == c) ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 32; ++sweep) {
    const double off = fabs(a[0][1]) + fabs(a[0][2]) + fabs(a[1][2]);
    const double diag = fabs(a[0][0]) + fabs(a[1][1]) + fabs(a[2][2]);
    if (off <= 1e-300 || off <= 1e-18 * diag) break;
#pragma unroll
    for (int pq = 0; pq < 3; ++pq) {
      const int p = (pq == 2) ? 1 : 0;
      const int q = (pq == 0) ? 1 : 2;
      const double apq = a[p][q];
      if (apq == 0.0) continue;
      const double theta = (a[q][q] - a[p][p]) / (2.0 * apq);
      const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
      const double c = 1.0 / sqrt(t * t + 1.0);
      const double s = t * c;
      const int r = 3 - p - q;
      const double arp = a[r][p], arq = a[r][q];
      a[p][p] -= t * apq;
      a[q][q] += t * apq;
      a[p][q] = a[q][p] = 0.0;
      a[r][p] = a[p][r] = c * arp - s * arq;
      a[r][q] = a[q][r] = s * arp + c * arq;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const double vkp = V[k][p], vkq = V[k][q];
        V[k][p] = c * vkp - s * vkq;
        V[k][q] = s * vkp + c * vkq;
      }
    }
  }
  w[0] = a[0][0];
  w[1] = a[1][1];
  w[2] = a[2][2];
  // ascending sort with the vectors
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2 - i; ++j)
      if (w[j] > w[j + 1]) {
        double tw = w[j]; w[j] = w[j + 1]; w[j + 1] = tw;
#pragma unroll
        for (int k = 0; k < 3; ++k) { double tv = V[k][j]; V[k][j] = V[k][j + 1]; V[k][j + 1] = tv; }
      }
}

struct ViscParams {
  int mode;
  double a[3];
  double b;
  double nu[3];
  double uscale;   // axis form: u = sqrt(uscale w3 Jg) e_3
};

// Per element node: G = grad grad^T -> eigh -> nu (hyperdiff.py:54-79) ->
// G_nu = sum_m (nu_m vals_m) e_m e_m^T (hyperdiff.py:80) -> W = w3 Jg[gid] G_nu.
__global__ void viscous_kernel(int nn, ViscParams P, const double* __restrict__ grad, int64_t nloc,
                               const double* __restrict__ w3, const double* __restrict__ Jg,
                               const int32_t* __restrict__ gid, double* __restrict__ Gnu_out,
                               double* __restrict__ lam_out, double* __restrict__ evec_out,
                               double* __restrict__ W_out, double* __restrict__ U_out) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= nloc) return;
  const int64_t e = p / nn, r = p % nn;
  double gr[3][3];
#pragma unroll
  for (int m = 0; m < 3; ++m)
#pragma unroll
    for (int c = 0; c < 3; ++c) gr[m][c] = grad[(e * 9 + m * 3 + c) * nn + r];
  double G[3][3];
#pragma unroll
  for (int m = 0; m < 3; ++m)
#pragma unroll
    for (int k = 0; k < 3; ++k) G[m][k] = gr[m][0] * gr[k][0] + gr[m][1] * gr[k][1] + gr[m][2] * gr[k][2];
  double vals[3], V[3][3];
  jacobi3(G, vals, V);
  if (!(vals[0] > 0.0)) atomicOr(&g_setup_flags[1], 1u);
  double lam[3], kv[3];
#pragma unroll
  for (int m = 0; m < 3; ++m) {
    lam[m] = 1.0 / vals[m];
    double nu;
    if (P.mode == 0) nu = (P.a[m] * lam[m]) / P.b;
    else nu = P.nu[m];
    kv[m] = nu * vals[m];
  }
  double Gn[3][3];
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int d = 0; d < 3; ++d) Gn[c][d] = kv[0] * V[c][0] * V[d][0] + kv[1] * V[c][1] * V[d][1] + kv[2] * V[c][2] * V[d][2];
  if (Gnu_out) {
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int d = 0; d < 3; ++d) Gnu_out[p * 9 + c * 3 + d] = Gn[c][d];
  }
  if (lam_out) {
#pragma unroll
    for (int m = 0; m < 3; ++m) lam_out[p * 3 + m] = lam[m];
  }
  if (evec_out) {
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int m = 0; m < 3; ++m) evec_out[p * 9 + c * 3 + m] = V[c][m];
  }
  if (U_out) {   // axis form (hv_viscous_axis): u = sqrt(uscale w3 Jg) e_3, e_3 = eigenvector of the largest eigenvalue
    const double su = sqrt(P.uscale * (w3[r] * Jg[gid[p]]));
#pragma unroll
    for (int c = 0; c < 3; ++c) U_out[c * nloc + p] = su * V[c][2];
  }
  if (W_out) {
    const double s = w3[r] * Jg[gid[p]];
    W_out[0 * nloc + p] = s * Gn[0][0];
    W_out[1 * nloc + p] = s * Gn[0][1];
    W_out[2 * nloc + p] = s * Gn[0][2];
    W_out[3 * nloc + p] = s * Gn[1][1];
    W_out[4 * nloc + p] = s * Gn[1][2];
    W_out[5 * nloc + p] = s * Gn[2][2];
  }
}

int reset_flags(cudaStream_t st) {
  void* ptr = nullptr;
  HV_CUDA_CHECK(cudaGetSymbolAddress(&ptr, g_setup_flags));
  HV_CUDA_CHECK(cudaMemsetAsync(ptr, 0, sizeof(unsigned int) * 4, st));
  return HV_OK;
}

int read_flags(cudaStream_t st, unsigned int out[4]) {
  HV_CUDA_CHECK(cudaMemcpyFromSymbolAsync(out, g_setup_flags, sizeof(unsigned int) * 4, 0,
                                          cudaMemcpyDeviceToHost, st));
  HV_CUDA_CHECK(cudaStreamSynchronize(st));
  return HV_OK;
}

template <int n>
int launch_metric(int scheme, const DMat& Dm, const double* coords, int64_t nelem, double* dx, double* J, double* grad,
                  cudaStream_t st) {
  constexpr int nn = n * n * n;
  const size_t smem = sizeof(double) * (n * n + 31 * nn);
  auto kern = metric_kernel<n>;
  if (smem > 48 * 1024) HV_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int threads = nn < 256 ? ((nn + 31) / 32) * 32 : 256;
  kern<<<(unsigned)nelem, threads, smem, st>>>(scheme, Dm, coords, nelem, dx, J, grad);
  HV_LAUNCH_CHECK();
  return HV_OK;
}

}  // namespace

extern "C" int hv_metric_terms(int scheme, int N, const double* h_D, const double* d_coords, int64_t nelem,
                               double* d_dxdxi, double* d_J, double* d_grad, void* stream) {
  if (scheme < 0 || scheme > 1) HV_FAIL(HV_ERR_INVALID, "unknown metric scheme %d", scheme);
  if (N < 1 || N > 8) HV_FAIL(HV_ERR_UNSUPPORTED, "polynomial degree %d not supported on the device (1..8)", N);
  if (!h_D || !d_coords || !d_J || !d_grad || nelem <= 0) HV_FAIL(HV_ERR_INVALID, "hv_metric_terms: null argument");
  cudaStream_t st = (cudaStream_t)stream;
  const int n = N + 1;
  DMat Dm;
  for (int t = 0; t < n * n; ++t) Dm.v[t] = h_D[t];
  int rc = reset_flags(st);
  if (rc) return rc;
  switch (n) {
    case 2: rc = launch_metric<2>(scheme, Dm, d_coords, nelem, d_dxdxi, d_J, d_grad, st); break;
    case 3: rc = launch_metric<3>(scheme, Dm, d_coords, nelem, d_dxdxi, d_J, d_grad, st); break;
    case 4: rc = launch_metric<4>(scheme, Dm, d_coords, nelem, d_dxdxi, d_J, d_grad, st); break;
    case 5: rc = launch_metric<5>(scheme, Dm, d_coords, nelem, d_dxdxi, d_J, d_grad, st); break;
    case 6: rc = launch_metric<6>(scheme, Dm, d_coords, nelem, d_dxdxi, d_J, d_grad, st); break;
    case 7: rc = launch_metric<7>(scheme, Dm, d_coords, nelem, d_dxdxi, d_J, d_grad, st); break;
    case 8: rc = launch_metric<8>(scheme, Dm, d_coords, nelem, d_dxdxi, d_J, d_grad, st); break;
    default: rc = launch_metric<9>(scheme, Dm, d_coords, nelem, d_dxdxi, d_J, d_grad, st); break;
  }
  if (rc) return rc;
  unsigned int f[4];
  rc = read_flags(st, f);
  if (rc) return rc;
  if (f[0]) HV_FAIL(HV_ERR_DEGENERATE, "inverted element: J <= 0");
  return HV_OK;
}

extern "C" int hv_dss_csr(const double* d_fe, int ncomp, int64_t cstride, const int64_t* d_off, const int32_t* d_idx,
                          int64_t nglobal, double* d_out, void* stream) {
  if (!d_fe || !d_off || !d_idx || !d_out || ncomp < 1 || nglobal <= 0) HV_FAIL(HV_ERR_INVALID, "hv_dss_csr: bad args");
  const int T = 256;
  dss_csr_kernel<<<(unsigned)((nglobal + T - 1) / T), T, 0, (cudaStream_t)stream>>>(d_fe, ncomp, cstride, d_off, d_idx,
                                                                                   nglobal, d_out);
  HV_LAUNCH_CHECK();
  return HV_OK;
}

extern "C" int hv_mass_and_projection(int N, const double* d_w3, const double* d_J, const double* d_grad,
                                      int64_t nelem, const int64_t* d_off, const int32_t* d_idx, int64_t nglobal,
                                      double* d_M, double* d_Minv, double* d_Jg, double* d_gz, void* stream) {
  if (N < 1 || !d_w3 || !d_J || !d_off || !d_idx || !d_M || !d_Minv || nelem <= 0 || nglobal <= 0)
    HV_FAIL(HV_ERR_INVALID, "hv_mass_and_projection: bad args");
  if (d_Jg && (!d_gz || !d_grad)) HV_FAIL(HV_ERR_INVALID, "hv_mass_and_projection: projection needs grad and gz");
  cudaStream_t st = (cudaStream_t)stream;
  int rc = reset_flags(st);
  if (rc) return rc;
  const int n = N + 1, nn = n * n * n;
  const int T = 256;
  mass_proj_kernel<<<(unsigned)((nglobal + T - 1) / T), T, 0, st>>>(nn, d_w3, d_J, d_grad, d_off, d_idx, nglobal, d_M,
                                                                   d_Minv, d_Jg, d_gz);
  HV_LAUNCH_CHECK();
  unsigned int f[4];
  rc = read_flags(st, f);
  if (rc) return rc;
  if (d_Jg && f[3]) HV_FAIL(HV_ERR_DEGENERATE, "zero mass-matrix entry in projection");
  if (f[2]) HV_FAIL(HV_ERR_DEGENERATE, "non-positive mass-matrix entry (inverted element?)");
  return HV_OK;
}

extern "C" int hv_viscous_metric(int N, int mode, const double* h_a, double b, const double* h_nu,
                                 const double* d_grad, int64_t nelem, const double* d_w3, const double* d_Jg,
                                 const int32_t* d_gid32, double* d_Gnu, double* d_lam, double* d_evecs, double* d_W,
                                 void* stream) {
  if (N < 1 || mode < 0 || mode > 2 || !d_grad || nelem <= 0) HV_FAIL(HV_ERR_INVALID, "hv_viscous_metric: bad args");
  if (d_W && (!d_w3 || !d_Jg || !d_gid32)) HV_FAIL(HV_ERR_INVALID, "hv_viscous_metric: packing needs w3, Jg, gid");
  ViscParams P{};
  P.mode = mode;
  if (mode == 0) {
    if (!h_a || !(b > 0)) HV_FAIL(HV_ERR_INVALID, "scaled viscosities need dt > 0");
    for (int m = 0; m < 3; ++m) P.a[m] = h_a[m];
    P.b = b;
  } else {
    if (!h_nu) HV_FAIL(HV_ERR_INVALID, "constant/anisotropic mode needs nu");
    for (int m = 0; m < 3; ++m) P.nu[m] = h_nu[m];
  }
  cudaStream_t st = (cudaStream_t)stream;
  int rc = reset_flags(st);
  if (rc) return rc;
  const int n = N + 1, nn = n * n * n;
  const int64_t nloc = nelem * nn;
  const int T = 128;
  viscous_kernel<<<(unsigned)((nloc + T - 1) / T), T, 0, st>>>(nn, P, d_grad, nloc, d_w3, d_Jg, d_gid32, d_Gnu, d_lam,
                                                              d_evecs, d_W, nullptr);
  HV_LAUNCH_CHECK();
  unsigned int f[4];
  rc = read_flags(st, f);
  if (rc) return rc;
  if (f[1]) HV_FAIL(HV_ERR_DEGENERATE, "degenerate element: non-positive metric eigenvalue");
  return HV_OK;
}

// isotropic form: s[p] = scale * w3 * Jg[gid[p]]
__global__ void iso_kernel(int nn, const double* __restrict__ w3, const double* __restrict__ Jg,
                           const int32_t* __restrict__ gid, int64_t nloc, double scale, double* __restrict__ S) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p < nloc) S[p] = scale * (w3[p % nn] * Jg[gid[p]]);
}

extern "C" int hv_viscous_axis(int N, const double* d_grad, int64_t nelem, const double* d_w3, const double* d_Jg,
                               const int32_t* d_gid32, int ncomp, double scale, double* d_U, void* stream) {
  if (N < 1 || !d_grad || nelem <= 0 || !d_w3 || !d_Jg || !d_gid32 || !d_U || (ncomp != 1 && ncomp != 3))
    HV_FAIL(HV_ERR_INVALID, "hv_viscous_axis: bad args");
  if (ncomp == 1) {
    const int n = N + 1, nn = n * n * n;
    const int64_t nloc = nelem * nn;
    iso_kernel<<<(unsigned)((nloc + 255) / 256), 256, 0, (cudaStream_t)stream>>>(nn, d_w3, d_Jg, d_gid32, nloc, scale,
                                                                               d_U);
    HV_LAUNCH_CHECK();
    return HV_OK;
  }
  ViscParams P{};
  P.mode = 1;   // the eigenvectors only; nu unused
  P.uscale = scale > 0.0 ? scale : 1.0;
  cudaStream_t st = (cudaStream_t)stream;
  int rc = reset_flags(st);
  if (rc) return rc;
  const int n = N + 1, nn = n * n * n;
  const int64_t nloc = nelem * nn;
  const int T = 128;
  viscous_kernel<<<(unsigned)((nloc + T - 1) / T), T, 0, st>>>(nn, P, d_grad, nloc, d_w3, d_Jg, d_gid32, nullptr,
                                                              nullptr, nullptr, nullptr, d_U);
  HV_LAUNCH_CHECK();
  unsigned int f[4];
  rc = read_flags(st, f);
  if (rc) return rc;
  if (f[1]) HV_FAIL(HV_ERR_DEGENERATE, "degenerate element: non-positive metric eigenvalue");
  return HV_OK;
}

extern "C" int hv_mass_proj_sums(int N, const double* d_w3, const double* d_J, const double* d_grad, int64_t nelem,
                                 const int64_t* d_off, const int32_t* d_idx, int64_t nglobal, double* d_S, void* stream) {
  if (N < 1 || !d_w3 || !d_J || !d_grad || !d_off || !d_idx || !d_S || nelem <= 0 || nglobal <= 0)
    HV_FAIL(HV_ERR_INVALID, "hv_mass_proj_sums: bad args");
  const int n = N + 1, nn = n * n * n, T = 256;
  mass_proj_sums_kernel<<<(unsigned)((nglobal + T - 1) / T), T, 0, (cudaStream_t)stream>>>(nn, d_w3, d_J, d_grad, d_off,
                                                                                         d_idx, nglobal, d_S);
  HV_LAUNCH_CHECK();
  return HV_OK;
}

extern "C" int hv_mass_proj_finalize(int64_t nglobal, const double* d_S, double* d_M, double* d_Minv, double* d_Jg,
                                     double* d_gz, void* stream) {
  if (nglobal <= 0 || !d_S || !d_M || !d_Minv || (d_Jg && !d_gz)) HV_FAIL(HV_ERR_INVALID, "hv_mass_proj_finalize: bad args");
  cudaStream_t st = (cudaStream_t)stream;
  int rc = reset_flags(st);
  if (rc) return rc;
  const int T = 256;
  mass_proj_finalize_kernel<<<(unsigned)((nglobal + T - 1) / T), T, 0, st>>>(nglobal, d_S, d_M, d_Minv, d_Jg, d_gz);
  HV_LAUNCH_CHECK();
  unsigned int f[4];
  rc = read_flags(st, f);
  if (rc) return rc;
  if (d_Jg && f[3]) HV_FAIL(HV_ERR_DEGENERATE, "zero mass-matrix entry in projection");
  if (f[2]) HV_FAIL(HV_ERR_DEGENERATE, "non-positive mass-matrix entry (inverted element?)");
  return HV_OK;
}

// ---------------------------------------------------------------------------
// Element derivative primitives (assembly.elem_deriv / weak_deriv_acc, assembly.py:29-51):
// strong: out[e, .., i, ..] = sum_a D[i, a] f[e, .., a, ..] along axis;
// weak:   out[e, .., i, ..] = -sum_a D[a, i] (w3 f)[e, .., a, ..]   (w3 multiplied first, as the
// reference's wf = weights3 * f).  One thread per element node.
namespace {

template <int n>
__global__ void elem_deriv_kernel(hv::DTab<n> Dt, const double* __restrict__ w3, int64_t nelem,
                                  const double* __restrict__ f, int axis, int weak, double* __restrict__ out) {
  constexpr int nn = n * n * n;
  const int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (id >= nelem * nn) return;
  const int64_t e = id / nn;
  const int t = (int)(id % nn);
  const int i = t / (n * n), j = (t / n) % n, k = t % n;
  const int ii = (axis == 0) ? i : (axis == 1) ? j : k;
  const int stride = (axis == 0) ? n * n : (axis == 1) ? n : 1;
  const double* fe = f + e * nn + (t - ii * stride);
  double s = 0.0;
#pragma unroll
  for (int a = 0; a < n; ++a) {
    const double v = fe[a * stride];
    if (weak) s += Dt.D[a][ii] * (w3[t - ii * stride + a * stride] * v);
    else s += Dt.D[ii][a] * v;
  }
  out[id] = weak ? -s : s;
}

template <int n>
int run_elem_deriv(const double* hD, const double* w3, int64_t nelem, const double* f, int axis, int weak,
                   double* out, cudaStream_t st) {
  hv::DTab<n> Dt;
  hv::fill_dtab(Dt, hD);
  const int64_t tot = nelem * n * n * n;
  elem_deriv_kernel<n><<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(Dt, w3, nelem, f, axis, weak, out);
  HV_LAUNCH_CHECK();
  return HV_OK;
}

}  // namespace

extern "C" int hv_elem_deriv(int N, const double* h_D, const double* d_w3, int64_t nelem, const double* d_f, int axis,
                             int weak, double* d_out, void* stream) {
  if (N < 1 || N > 7 || !h_D || nelem <= 0 || !d_f || !d_out || axis < 0 || axis > 2 || (weak && !d_w3))
    HV_FAIL(HV_ERR_INVALID, "hv_elem_deriv: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  switch (N + 1) {
    case 2: return run_elem_deriv<2>(h_D, d_w3, nelem, d_f, axis, weak, d_out, st);
    case 3: return run_elem_deriv<3>(h_D, d_w3, nelem, d_f, axis, weak, d_out, st);
    case 4: return run_elem_deriv<4>(h_D, d_w3, nelem, d_f, axis, weak, d_out, st);
    case 5: return run_elem_deriv<5>(h_D, d_w3, nelem, d_f, axis, weak, d_out, st);
    case 6: return run_elem_deriv<6>(h_D, d_w3, nelem, d_f, axis, weak, d_out, st);
    case 7: return run_elem_deriv<7>(h_D, d_w3, nelem, d_f, axis, weak, d_out, st);
    default: return run_elem_deriv<8>(h_D, d_w3, nelem, d_f, axis, weak, d_out, st);
  }
}
