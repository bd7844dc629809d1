// Rounding-faithful element metric arithmetic, shared by the sm_100a kernel
// and a host build used only by the CPU test suite to pin the operation order
// against the reference (tests/test_metric_order.py).
//
// Every product/sum is rounded individually (no FMA contraction) and follows
// the exact order numpy 2.3's einsum kernels use for the reference calls
// (re-verified by the CPU tests):
//   strong derivative along axis 0 or 1 ("ia,eajk->eijk", "ja,eiak->eijk"):
//       s = (((0 + p_0) + p_1) + ...) + p_N            with p_a = D[i,a] f_a
//   strong derivative along axis 2 ("ka,eija->eijk", contiguous reduction):
//       numpy's 2-lane sum: lanes L0/L1 accumulate even/odd terms, blocks of
//       8 terms visited in the order a+6,a+4,a+2,a (a+7,...,a+1), then the
//       tail pairs ascending, result L0 + L1.
//   _jacobian / _cross: the expression trees of metrics.py:57-76 left to right.
#pragma once

#ifdef __CUDACC__
#define HV_HD __host__ __device__ __forceinline__
#else
#define HV_HD inline
#endif

#if defined(__CUDA_ARCH__)
#define HV_MUL(a, b) __dmul_rn((a), (b))
#define HV_ADD(a, b) __dadd_rn((a), (b))
#define HV_SUB(a, b) __dsub_rn((a), (b))
#define HV_DIV(a, b) __ddiv_rn((a), (b))
#else
// host build is compiled with -ffp-contract=off
#define HV_MUL(a, b) ((a) * (b))
#define HV_ADD(a, b) ((a) + (b))
#define HV_SUB(a, b) ((a) - (b))
#define HV_DIV(a, b) ((a) / (b))
#endif

namespace hv {

// f points at one element scalar field (n*n*n, k fastest); D is row-major n x n.
template <int n>
HV_HD double strong_deriv_exact(const double* __restrict__ D, const double* __restrict__ f, int i, int j, int k,
                                int axis) {
  if (axis == 0) {
    double s = 0.0;
#pragma unroll
    for (int a = 0; a < n; ++a) s = HV_ADD(s, HV_MUL(D[i * n + a], f[(a * n + j) * n + k]));
    return s;
  }
  if (axis == 1) {
    double s = 0.0;
#pragma unroll
    for (int a = 0; a < n; ++a) s = HV_ADD(s, HV_MUL(D[j * n + a], f[(i * n + a) * n + k]));
    return s;
  }
  const double* row = D + k * n;
  const double* line = f + (i * n + j) * n;
  double L0 = 0.0, L1 = 0.0;
  int a = 0;
#pragma unroll
  for (; a + 8 <= n; a += 8) {
#pragma unroll
    for (int t = 3; t >= 0; --t) {
      L0 = HV_ADD(HV_MUL(row[a + 2 * t], line[a + 2 * t]), L0);
      L1 = HV_ADD(HV_MUL(row[a + 2 * t + 1], line[a + 2 * t + 1]), L1);
    }
  }
#pragma unroll
  for (; a < n; a += 2) {
    L0 = HV_ADD(HV_MUL(row[a], line[a]), L0);
    if (a + 1 < n) L1 = HV_ADD(HV_MUL(row[a + 1], line[a + 1]), L1);
  }
  return HV_ADD(L0, L1);
}

// J = a0 (b1 c2 - b2 c1) - a1 (b0 c2 - b2 c0) + a2 (b0 c1 - b1 c0)   (metrics.py:57-64)
// x[c][m] = dx_c / dxi^m ; a = column 0, b = column 1, c = column 2.
HV_HD double jacobian_exact(const double x[3][3]) {
  const double t0 = HV_MUL(x[0][0], HV_SUB(HV_MUL(x[1][1], x[2][2]), HV_MUL(x[2][1], x[1][2])));
  const double t1 = HV_MUL(x[1][0], HV_SUB(HV_MUL(x[0][1], x[2][2]), HV_MUL(x[2][1], x[0][2])));
  const double t2 = HV_MUL(x[2][0], HV_SUB(HV_MUL(x[0][1], x[1][2]), HV_MUL(x[1][1], x[0][2])));
  return HV_ADD(HV_SUB(t0, t1), t2);
}

// (u x v) in the component order of metrics.py:67-76
HV_HD void cross_exact(const double u[3], const double v[3], double out[3]) {
  out[0] = HV_SUB(HV_MUL(u[1], v[2]), HV_MUL(u[2], v[1]));
  out[1] = HV_SUB(HV_MUL(u[2], v[0]), HV_MUL(u[0], v[2]));
  out[2] = HV_SUB(HV_MUL(u[0], v[1]), HV_MUL(u[1], v[0]));
}

#ifdef __CUDACC__
#pragma nv_exec_check_disable
#endif
// Full metric terms of one element (curl-invariant: scheme 0; cross-product: 1).
// X: (3, nn) coordinates; scratch A: (3 dir, 3 comp, nn); outputs dx (3 c, 3 m, nn),
// J (nn), grad (3 i, 3 c, nn).  Node-parallel over `node` in [first, nn) step `stride`
// with barrier callbacks between the phases (device: __syncthreads; host: no-op).
template <int n, class Barrier>
HV_HD void element_metrics(int scheme, const double* __restrict__ D, const double* __restrict__ X, double* dx,
                           double* J, double* A, double* grad, int first, int stride, Barrier bar) {
  constexpr int nn = n * n * n;
  for (int node = first; node < nn; node += stride) {
    const int i = node / (n * n), j = (node / n) % n, k = node % n;
    double x[3][3];
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int m = 0; m < 3; ++m) {
        x[c][m] = strong_deriv_exact<n>(D, X + c * nn, i, j, k, m);
        dx[(c * 3 + m) * nn + node] = x[c][m];
      }
    J[node] = jacobian_exact(x);
    if (scheme == 0) {
      const double pos[3] = {X[node], X[nn + node], X[2 * nn + node]};
#pragma unroll
      for (int m = 0; m < 3; ++m) {
        const double u[3] = {x[0][m], x[1][m], x[2][m]};
        double cr[3];
        cross_exact(u, pos, cr);
#pragma unroll
        for (int c = 0; c < 3; ++c) A[(m * 3 + c) * nn + node] = cr[c];
      }
    }
  }
  bar();
  for (int node = first; node < nn; node += stride) {
    const int i = node / (n * n), j = (node / n) % n, k = node % n;
    const double Jn = J[node];
#pragma unroll
    for (int ii = 0; ii < 3; ++ii) {
      const int jj = (ii + 1) % 3, kk = (ii + 2) % 3;
      if (scheme == 0) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double t1 = strong_deriv_exact<n>(D, A + (jj * 3 + c) * nn, i, j, k, kk);
          const double t2 = strong_deriv_exact<n>(D, A + (kk * 3 + c) * nn, i, j, k, jj);
          grad[(ii * 3 + c) * nn + node] = HV_DIV(HV_MUL(0.5, HV_SUB(t1, t2)), Jn);
        }
      } else {
        const double u[3] = {dx[(0 * 3 + jj) * nn + node], dx[(1 * 3 + jj) * nn + node], dx[(2 * 3 + jj) * nn + node]};
        const double v[3] = {dx[(0 * 3 + kk) * nn + node], dx[(1 * 3 + kk) * nn + node], dx[(2 * 3 + kk) * nn + node]};
        double cr[3];
        cross_exact(u, v, cr);
#pragma unroll
        for (int c = 0; c < 3; ++c) grad[(ii * 3 + c) * nn + node] = HV_DIV(cr[c], Jn);
      }
    }
  }
}

}  // namespace hv
