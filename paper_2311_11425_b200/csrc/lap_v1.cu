// Hot path, first correct version (v1): element kernel + CSR DSS kernel.
//
// laplacian_apply (hyperdiff.py:84-94) for nf fields in one pass:
//   K1 lap_elem_v1: one CTA per element; gather q (nf fields), strong
//      derivatives, contraction with the packed metric W = w3 Jg G_nu,
//      weak derivatives; writes the element accumulator (nf, nloc).
//   K2 dss_minv_v1: one thread per global node; sums the accumulator over
//      the CSR map in flat order (== np.add.at), multiplies by Minv and scale.
// The optimised hot path (tile sweep with on-chip DSS) lives in lap_tile.cu;
// v1 stays as the cross-check and the generic fallback layout.
#include <cuda_runtime.h>

#include "hv_common.h"
#include "lap_common.cuh"

namespace {

template <int n, int NF>
__global__ void __launch_bounds__(512) lap_elem_v1(hv::DTab<n> Dt, const int32_t* __restrict__ gid,
                                                   const double* __restrict__ W, int64_t nloc,
                                                   const double* __restrict__ q, int64_t ldq, hv::FieldMap fm,
                                                   double* __restrict__ work) {
  constexpr int nn = n * n * n;
  extern __shared__ double smem_v1[];
  double(*sq)[nn] = reinterpret_cast<double(*)[nn]>(smem_v1);
  double(*sf)[NF][nn] = reinterpret_cast<double(*)[NF][nn]>(smem_v1 + NF * nn);
  double(*sD)[n] = reinterpret_cast<double(*)[n]>(smem_v1 + 4 * NF * nn);   // D: thread-varying rows
  const int64_t e = blockIdx.x;
  const int t = threadIdx.x;
  for (int x = t; x < n * n; x += blockDim.x) sD[x / n][x % n] = Dt.D[x / n][x % n];
  const bool act = t < nn;
  const int i = t / (n * n), j = (t / n) % n, k = t % n;
  const int64_t p = e * nn + t;
  if (act) {
    const int64_t g = gid[p];
#pragma unroll
    for (int f = 0; f < NF; ++f) sq[f][t] = q[g * ldq + fm.f[f]];
  }
  __syncthreads();
  if (act) {
    const double w00 = W[0 * nloc + p], w01 = W[1 * nloc + p], w02 = W[2 * nloc + p];
    const double w11 = W[3 * nloc + p], w12 = W[4 * nloc + p], w22 = W[5 * nloc + p];
#pragma unroll
    for (int f = 0; f < NF; ++f) {
      double d0 = 0.0, d1 = 0.0, d2 = 0.0;
#pragma unroll
      for (int a = 0; a < n; ++a) {
        d0 += sD[i][a] * sq[f][(a * n + j) * n + k];
        d1 += sD[j][a] * sq[f][(i * n + a) * n + k];
        d2 += sD[k][a] * sq[f][(i * n + j) * n + a];
      }
      sf[0][f][t] = w00 * d0 + w01 * d1 + w02 * d2;
      sf[1][f][t] = w01 * d0 + w11 * d1 + w12 * d2;
      sf[2][f][t] = w02 * d0 + w12 * d1 + w22 * d2;
    }
  }
  __syncthreads();
  if (act) {
#pragma unroll
    for (int f = 0; f < NF; ++f) {
      double s = 0.0;
#pragma unroll
      for (int a = 0; a < n; ++a) {
        s += sD[a][i] * sf[0][f][(a * n + j) * n + k];
        s += sD[a][j] * sf[1][f][(i * n + a) * n + k];
        s += sD[a][k] * sf[2][f][(i * n + j) * n + a];
      }
      work[f * nloc + p] = -s;
    }
  }
}

template <int NF>
__global__ void dss_minv_v1(const double* __restrict__ work, int64_t nloc, const int64_t* __restrict__ off,
                            const int32_t* __restrict__ idx, const double* __restrict__ Minv, int64_t ng,
                            double scale, double* __restrict__ out, int64_t ldo, hv::FieldMap fm, int accumulate) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= ng) return;
  const int64_t o0 = off[g], o1 = off[g + 1];
  double s[NF];
#pragma unroll
  for (int f = 0; f < NF; ++f) s[f] = 0.0;
  for (int64_t o = o0; o < o1; ++o) {
    const int64_t pp = idx[o];
#pragma unroll
    for (int f = 0; f < NF; ++f) s[f] += work[f * nloc + pp];
  }
  const double mi = Minv[g] * scale;
#pragma unroll
  for (int f = 0; f < NF; ++f) {
    double* o = out + g * ldo + fm.f[f];
    *o = accumulate ? *o + s[f] * mi : s[f] * mi;
  }
}

template <int n, int NF>
int run_v1(const hv_lap_plan* P, const double* q, int64_t ldq, const hv::FieldMap& qf, double* out, int64_t ldo,
           const hv::FieldMap& of, double scale, int accumulate, cudaStream_t st) {
  constexpr int nn = n * n * n;
  const int64_t nloc = P->nelem * nn;
  hv::DTab<n> Dt;
  hv::fill_dtab(Dt, P->D);
  const int threads = ((nn + 31) / 32) * 32;
  const size_t smem = sizeof(double) * (4 * NF * nn + n * n);
  auto kern = lap_elem_v1<n, NF>;
  if (smem > 48 * 1024) HV_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<(unsigned)P->nelem, threads, smem, st>>>(Dt, P->d_gid, P->d_W, nloc, q, ldq, qf, P->d_work);
  HV_LAUNCH_CHECK();
  const int T = 256;
  dss_minv_v1<NF><<<(unsigned)((P->nglobal + T - 1) / T), T, 0, st>>>(P->d_work, nloc, P->d_off, P->d_idx, P->d_Minv,
                                                                    P->nglobal, scale, out, ldo, of, accumulate);
  HV_LAUNCH_CHECK();
  return HV_OK;
}

template <int n>
int run_v1_nf(int nf, const hv_lap_plan* P, const double* q, int64_t ldq, const hv::FieldMap& qf, double* out,
              int64_t ldo, const hv::FieldMap& of, double scale, int acc, cudaStream_t st) {
  switch (nf) {
    case 1: return run_v1<n, 1>(P, q, ldq, qf, out, ldo, of, scale, acc, st);
    case 2: return run_v1<n, 2>(P, q, ldq, qf, out, ldo, of, scale, acc, st);
    case 3: return run_v1<n, 3>(P, q, ldq, qf, out, ldo, of, scale, acc, st);
    case 4: return run_v1<n, 4>(P, q, ldq, qf, out, ldo, of, scale, acc, st);
    default: return run_v1<n, 5>(P, q, ldq, qf, out, ldo, of, scale, acc, st);
  }
}

}  // namespace

namespace hv {

int dss_minv_accumulate(const double* work, int64_t nloc, const int64_t* off, const int32_t* idx, const double* Minv,
                        int64_t ng, double* out, int64_t ldo, int nf, bool accumulate, cudaStream_t st) {
  FieldMap fm{};
  for (int f = 0; f < 5; ++f) fm.f[f] = f;
  const int T = 256;
  const unsigned G = (unsigned)((ng + T - 1) / T);
  if (nf != 5) HV_FAIL(HV_ERR_UNSUPPORTED, "dss_minv_accumulate: nf=%d", nf);
  dss_minv_v1<5><<<G, T, 0, st>>>(work, nloc, off, idx, Minv, ng, 1.0, out, ldo, fm, accumulate ? 1 : 0);
  HV_LAUNCH_CHECK();
  return HV_OK;
}

int laplacian_v1(const hv_lap_plan* P, const double* q, int64_t ldq, int nf, const FieldMap& qf, double* out,
                 int64_t ldo, const FieldMap& of, double scale, int acc, cudaStream_t st) {
  switch (P->N) {
    case 1: return run_v1_nf<2>(nf, P, q, ldq, qf, out, ldo, of, scale, acc, st);
    case 2: return run_v1_nf<3>(nf, P, q, ldq, qf, out, ldo, of, scale, acc, st);
    case 3: return run_v1_nf<4>(nf, P, q, ldq, qf, out, ldo, of, scale, acc, st);
    case 4: return run_v1_nf<5>(nf, P, q, ldq, qf, out, ldo, of, scale, acc, st);
    case 5: return run_v1_nf<6>(nf, P, q, ldq, qf, out, ldo, of, scale, acc, st);
    case 6: return run_v1_nf<7>(nf, P, q, ldq, qf, out, ldo, of, scale, acc, st);
    case 7: return run_v1_nf<8>(nf, P, q, ldq, qf, out, ldo, of, scale, acc, st);
    default: HV_FAIL(HV_ERR_UNSUPPORTED, "laplacian: degree %d not supported (1..7)", P->N);
  }
}

}  // namespace hv
