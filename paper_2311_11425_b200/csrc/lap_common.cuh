// Small shared device types for the hot-path kernels.
#pragma once
#include <cuda_runtime.h>

#include "hv_common.h"

namespace hv {

template <int F>
struct Vec {
  double v[F];
};


// (n x n) LGL derivative matrix passed by value (kernel-parameter constant bank,
// broadcast to every thread): D[i][a] = d psi_a / d xi at node i (basis.py:77-87).
template <int n>
struct DTab {
  double D[n][n];
};

template <int n>
inline void fill_dtab(DTab<n>& t, const double* Drow) {
  for (int i = 0; i < n; ++i)
    for (int a = 0; a < n; ++a) t.D[i][a] = Drow[i * n + a];
}

// D plus its even-odd form and that of -D^T (the plane kernel's line contractions, lap_plane.cu).
// The LGL derivative matrix is centro-antisymmetric (A[N-i][N-a] = -A[i][a] for A = D and A = -D^T),
// so y = A x follows from the top rows only: with xd_a = x_a - x_{N-a}, xs_a = x_a + x_{N-a} (a < M = n/2),
//   e_i = sum_a ce[i][a] xd_a,  o_i = sum_a co[i][a] xs_a + cm[i] x_M (n odd),
//   y_i = e_i + o_i,  y_{N-i} = e_i - o_i  (i < M),  y_M = sum_a ce[M][a] xd_a  (n odd),
// ce = (A[i][a] - A[i][N-a]) / 2, co = (A[i][a] + A[i][N-a]) / 2, cm = A[i][M]: n^2 - n + (n odd) line
// FMAs + adds instead of n^2 (20 instead of 25 at n = 5).  Index 0: A = D, index 1: A = -D^T.
template <int n>
struct DTabEO : DTab<n> {
  double ce[2][(n + 1) / 2][n / 2 > 0 ? n / 2 : 1], co[2][n / 2 > 0 ? n / 2 : 1][n / 2 > 0 ? n / 2 : 1],
      cm[2][n / 2 > 0 ? n / 2 : 1];
};

template <int n>
inline void fill_dtab_eo(DTabEO<n>& t, const double* Drow) {
  fill_dtab<n>(t, Drow);
  constexpr int N = n - 1, M = n / 2;
  for (int w = 0; w < 2; ++w) {
    auto A = [&](int i, int a) { return w == 0 ? Drow[i * n + a] : -Drow[a * n + i]; };
    for (int i = 0; i < (n + 1) / 2; ++i)
      for (int a = 0; a < M; ++a) {
        t.ce[w][i][a] = 0.5 * (A(i, a) - A(i, N - a));
        if (i < M) t.co[w][i][a] = 0.5 * (A(i, a) + A(i, N - a));
      }
    for (int i = 0; i < M; ++i) t.cm[w][i] = (n % 2) ? A(i, M) : 0.0;
  }
}

// y = A x with A = D (W = 0) or -D^T (W = 1), even-odd form (DTabEO)
template <int n, int W>
__device__ __forceinline__ void eo_mv(const DTabEO<n>& Dt, const double (&x)[n], double (&y)[n]) {
  constexpr int N = n - 1, M = n / 2;
  double xd[M], xs[M];
#pragma unroll
  for (int a = 0; a < M; ++a) {
    xd[a] = x[a] - x[N - a];
    xs[a] = x[a] + x[N - a];
  }
#pragma unroll
  for (int i = 0; i < M; ++i) {
    double e = Dt.ce[W][i][0] * xd[0], o = Dt.co[W][i][0] * xs[0];
#pragma unroll
    for (int a = 1; a < M; ++a) {
      e = fma(Dt.ce[W][i][a], xd[a], e);
      o = fma(Dt.co[W][i][a], xs[a], o);
    }
    if constexpr (n % 2 == 1) o = fma(Dt.cm[W][i], x[M], o);
    y[i] = e + o;
    y[N - i] = e - o;
  }
  if constexpr (n % 2 == 1) {
    double e = Dt.ce[W][M][0] * xd[0];
#pragma unroll
    for (int a = 1; a < M; ++a) e = fma(Dt.ce[W][M][a], xd[a], e);
    y[M] = e;
  }
}

// eo_mv with the outputs stored as they are formed (out[i * stride]): fewer live registers
template <int n, int W>
__device__ __forceinline__ void eo_mv_st(const DTabEO<n>& Dt, const double (&x)[n], double* out, int stride) {
  constexpr int N = n - 1, M = n / 2;
  double xd[M], xs[M];
#pragma unroll
  for (int a = 0; a < M; ++a) {
    xd[a] = x[a] - x[N - a];
    xs[a] = x[a] + x[N - a];
  }
  double xm = 0.0;
  if constexpr (n % 2 == 1) xm = x[M];
#pragma unroll
  for (int i = 0; i < M; ++i) {
    double e = Dt.ce[W][i][0] * xd[0], o = Dt.co[W][i][0] * xs[0];
#pragma unroll
    for (int a = 1; a < M; ++a) {
      e = fma(Dt.ce[W][i][a], xd[a], e);
      o = fma(Dt.co[W][i][a], xs[a], o);
    }
    if constexpr (n % 2 == 1) o = fma(Dt.cm[W][i], xm, o);
    out[i * stride] = e + o;
    out[(N - i) * stride] = e - o;
  }
  if constexpr (n % 2 == 1) {
    double e = Dt.ce[W][M][0] * xd[0];
#pragma unroll
    for (int a = 1; a < M; ++a) e = fma(Dt.ce[W][M][a], xd[a], e);
    out[M * stride] = e;
  }
}

// eo_mv_st with the coefficients read from shared memory (a copy of DTabEO's ce[W], co[W], cm[W] in
// that order, eo_smem_fill): kernels whose loops would otherwise hoist the constant-bank coefficients
// into registers and spill them
template <int n>
struct EOSmem {
  static constexpr int M = n / 2 > 0 ? n / 2 : 1, CE = ((n + 1) / 2) * M, CO = M * M, PER = CE + CO + M;
};
template <int n>
__device__ __forceinline__ void eo_smem_fill(const DTabEO<n>& Dt, double* cf, int tid, int nthr) {
  using E = EOSmem<n>;
  for (int x = tid; x < 2 * E::PER; x += nthr) {
    const int w = x / E::PER, r = x % E::PER;
    double v;
    if (r < E::CE) v = Dt.ce[w][r / E::M][r % E::M];
    else if (r < E::CE + E::CO) v = Dt.co[w][(r - E::CE) / E::M][(r - E::CE) % E::M];
    else v = Dt.cm[w][r - E::CE - E::CO];
    cf[x] = v;
  }
}
template <int n, int W>
__device__ __forceinline__ void eo_mv_st_s(const double* cf0, const double (&x)[n], double* out, int stride) {
  using E = EOSmem<n>;
  constexpr int N = n - 1, M = n / 2;
  const double* ce = cf0 + W * E::PER;
  const double* co = ce + E::CE;
  const double* cm = co + E::CO;
  double xd[M], xs[M];
#pragma unroll
  for (int a = 0; a < M; ++a) {
    xd[a] = x[a] - x[N - a];
    xs[a] = x[a] + x[N - a];
  }
  double xm = 0.0;
  if constexpr (n % 2 == 1) xm = x[M];
#pragma unroll
  for (int i = 0; i < M; ++i) {
    double e = ce[i * M] * xd[0], o = co[i * M] * xs[0];
#pragma unroll
    for (int a = 1; a < M; ++a) {
      e = fma(ce[i * M + a], xd[a], e);
      o = fma(co[i * M + a], xs[a], o);
    }
    if constexpr (n % 2 == 1) o = fma(cm[i], xm, o);
    out[i * stride] = e + o;
    out[(N - i) * stride] = e - o;
  }
  if constexpr (n % 2 == 1) {
    double e = ce[M * M] * xd[0];
#pragma unroll
    for (int a = 1; a < M; ++a) e = fma(ce[M * M + a], xd[a], e);
    out[M * stride] = e;
  }
}

// Up to five (state column) indices.
struct FieldMap {
  int f[5];
};

int laplacian_v1(const hv_lap_plan* P, const double* q, int64_t ldq, int nf, const FieldMap& qf, double* out,
                 int64_t ldo, const FieldMap& of, double scale, int accumulate, cudaStream_t st);

}  // namespace hv
