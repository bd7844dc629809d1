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

// Up to five (state column) indices.
struct FieldMap {
  int f[5];
};

int laplacian_v1(const hv_lap_plan* P, const double* q, int64_t ldq, int nf, const FieldMap& qf, double* out,
                 int64_t ldo, const FieldMap& of, double scale, int accumulate, cudaStream_t st);

}  // namespace hv
