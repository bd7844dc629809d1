// Compressible-Euler right-hand side on the device (sets 2NC / 2C / 3C).
//
// Reference: EulerOps._precompute (euler.py:39-59), rhs_full / rhs_horizontal
// (euler.py:111-134), _contravariant (148-154), _acc_advective (159-189),
// _acc_flux (191-224), pressure (state.py:84-101).
//
// euler_setup  (once per EulerOps): per element node the 13-15 doubles the RHS
//              reads -- grad xi, grad eta (element), grad zeta (projected,
//              gathered), Jg (projected, gathered), dPhi_m (strong derivative of
//              the gathered geopotential), flux mask, Phi (3C), rhat.
// euler_elem   one CTA per element, one thread per node: gathers the 5 fields,
//              EOS, contravariant velocities, all fluxes of the requested
//              directions into shared memory, then every node forms its weak /
//              strong line sums, geopotential and Coriolis terms -> element
//              accumulator (5 fields).
// DSS + Minv   the flat-order CSR sum of lap_v1 (dss_minv_v1), optionally
//              accumulating into the output (S + H_nu in one buffer).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>

#include "hv_common.h"
#include "hv_pow.cuh"
#include "lap_common.cuh"
#include "lap_tile.cuh"

namespace hv {
int slot_fixup(const TileArgs& A, int F, cudaStream_t st);
int dss_minv_accumulate(const double* work, int64_t nloc, const int64_t* off, const int32_t* idx, const double* Minv,
                        int64_t ng, double* out, int64_t ldo, int nf, bool accumulate, cudaStream_t st);
}

namespace {

// metric record per element node (component-major, nloc stride)
enum { M_GXI = 0, M_GETA = 3, M_GZETA = 6, M_JG = 9, M_DPHI = 10, M_MASK = 13, M_PHI = 14, M_RHAT = 15, M_NCOMP = 18 };

struct EulerConsts {
  double P_A, R, gamma, omega;
  int set;       // 0 = 2NC, 1 = 2C, 2 = 3C
  int dirs;      // bit mask of reference directions
  int coriolis;  // 0 = rhat, 1 = zetahat
};

template <int n>
__global__ void __launch_bounds__(512) euler_setup_kernel(hv::DTab<n> Dt, int64_t nelem, const int32_t* __restrict__ gid,
                                                          const double* __restrict__ grad, const double* __restrict__ Jg,
                                                          const double* __restrict__ gz, const double* __restrict__ Phi_g,
                                                          const double* __restrict__ mask_g,
                                                          const double* __restrict__ coords, int sphere,
                                                          double* __restrict__ Mout) {
  constexpr int nn = n * n * n;
  __shared__ double sPhi[nn];
  const int64_t e = blockIdx.x;
  const int t = threadIdx.x;
  const int64_t nloc = nelem * nn;
  const int64_t p = e * nn + t;
  const int i = t / (n * n), j = (t / n) % n, k = t % n;
  int g = 0;
  if (t < nn) {
    g = gid[p];
    sPhi[t] = Phi_g[g];
  }
  __syncthreads();
  if (t >= nn) return;
  for (int c = 0; c < 3; ++c) {
    Mout[(M_GXI + c) * nloc + p] = grad[(e * 9 + 0 * 3 + c) * nn + t];
    Mout[(M_GETA + c) * nloc + p] = grad[(e * 9 + 1 * 3 + c) * nn + t];
    Mout[(M_GZETA + c) * nloc + p] = gz[(int64_t)g * 3 + c];
  }
  Mout[M_JG * nloc + p] = Jg[g];
  // dPhi_m = strong derivative of the gathered geopotential (euler.py:58-59)
  double d0 = 0.0, d1 = 0.0, d2 = 0.0;
#pragma unroll
  for (int a = 0; a < n; ++a) {
    d0 += Dt.D[i][a] * sPhi[(a * n + j) * n + k];
    d1 += Dt.D[j][a] * sPhi[(i * n + a) * n + k];
    d2 += Dt.D[k][a] * sPhi[(i * n + j) * n + a];
  }
  Mout[(M_DPHI + 0) * nloc + p] = d0;
  Mout[(M_DPHI + 1) * nloc + p] = d1;
  Mout[(M_DPHI + 2) * nloc + p] = d2;
  Mout[M_MASK * nloc + p] = mask_g[g];
  Mout[M_PHI * nloc + p] = sPhi[t];
  // rhat: element coordinates / |x| on the sphere, zhat in the box (euler.py:48-55)
  if (sphere) {
    const double x = coords[(e * 3 + 0) * nn + t], y = coords[(e * 3 + 1) * nn + t], z = coords[(e * 3 + 2) * nn + t];
    const double r = sqrt(x * x + y * y + z * z);
    Mout[(M_RHAT + 0) * nloc + p] = x / r;
    Mout[(M_RHAT + 1) * nloc + p] = y / r;
    Mout[(M_RHAT + 2) * nloc + p] = z / r;
  } else {
    Mout[(M_RHAT + 0) * nloc + p] = 0.0;
    Mout[(M_RHAT + 1) * nloc + p] = 0.0;
    Mout[(M_RHAT + 2) * nloc + p] = 1.0;
  }
}

// One element's RHS accumulator at node t (all threads of the CTA call it: it holds a CTA
// barrier).  Phase 1: gather, EOS, contravariant velocities, fluxes into shared memory;
// phase 2: weak / strong line sums, geopotential, Coriolis -> acc[5] (valid for t < n^3).
template <int n>
__device__ __forceinline__ void euler_node_acc(const hv::DTab<n>& Dt, const EulerConsts& K, int64_t nelem,
                                               int64_t e, int t, const int32_t* __restrict__ gid,
                                               const double* __restrict__ w3, const double* __restrict__ Mt,
                                               const double* __restrict__ q, int64_t ldq, double* sm,
                                               double (&acc)[5], int& g_out, int layer, int nlay,
                                               const double* __restrict__ sD) {
  constexpr int nn = n * n * n;
  // 2C / 3C: per direction m: [0] w3*F_rho, [1] w3*F_thermo (weak), [2..4] momentum fluxes (strong)
  // 2NC: [0..2] w3*F_rho per m (weak), [3..7] u, v, w, theta, P (strong derivatives)
  const bool act = t < nn;
  const int64_t nloc = nelem * nn;
  const int64_t p = e * nn + (act ? t : 0);
  const int i = t / (n * n), j = (t / n) % n, k = t % n;
  double qv[5] = {0, 0, 0, 0, 0}, gm[3][3] = {}, Jg = 0, mask = 0, dphi[3] = {}, phi = 0, P = 0, un[3] = {};
  if (act) {
    const int g = gid[p];
    g_out = g;
#pragma unroll
    for (int f = 0; f < 5; ++f) qv[f] = q[(int64_t)g * ldq + f];
#pragma unroll
    for (int m = 0; m < 3; ++m)
#pragma unroll
      for (int c = 0; c < 3; ++c) gm[m][c] = Mt[(m * 3 + c) * nloc + p];
    Jg = Mt[M_JG * nloc + p];
    // flux mask (mesh.py:141-143): zero on the bottom and top levels of every column, i.e. at
    // k = 0 of the first layer and k = N of the last one (derived, not read from the record)
    mask = ((layer == 0 && k == 0) || (layer == nlay - 1 && k == n - 1)) ? 0.0 : 1.0;
#pragma unroll
    for (int m = 0; m < 3; ++m) dphi[m] = Mt[(M_DPHI + m) * nloc + p];
    if (K.set == 2) phi = Mt[M_PHI * nloc + p];   // the geopotential enters the 3C pressure only
    const double rho = qv[0];
    // EOS (state.py:84-101), reference expression order
    if (K.set == 0) P = K.P_A * hv::pow_pos(qv[0] * K.R * qv[4] / K.P_A, K.gamma);
    else if (K.set == 1) P = K.P_A * hv::pow_pos(K.R * qv[4] / K.P_A, K.gamma);
    else {
      const double ke = 0.5 * (qv[1] * qv[1] + qv[2] * qv[2] + qv[3] * qv[3]) / rho;
      P = (K.gamma - 1.0) * (qv[4] - ke - rho * phi);
    }
    // contravariant velocities (euler.py:148-154)
#pragma unroll
    for (int m = 0; m < 3; ++m) {
      double s = gm[m][0] * qv[1] + gm[m][1] * qv[2] + gm[m][2] * qv[3];
      if (K.set != 0) s = s / rho;
      un[m] = (m == 2) ? s * mask : s;
    }
  }
  const double w = act ? w3[t] : 0.0;
  const double wj = w * Jg;
#pragma unroll
  for (int f = 0; f < 5; ++f) acc[f] = 0.0;
  if (K.set != 0) {
    const double tflux = (K.set == 1) ? qv[4] / qv[0] : (qv[4] + P) / qv[0];
    double* s = sm;  // [m][5][nn]
    if (act) {
#pragma unroll
      for (int m = 0; m < 3; ++m) {
        const double jun = Jg * un[m];
        s[(m * 5 + 0) * nn + t] = w * (jun * qv[0]);
        s[(m * 5 + 1) * nn + t] = w * (jun * qv[0] * tflux);
#pragma unroll
        for (int c = 0; c < 3; ++c) s[(m * 5 + 2 + c) * nn + t] = Jg * (qv[1 + c] * un[m] + P * gm[m][c]);
      }
    }
    __syncthreads();
    if (act) {
#pragma unroll
      for (int m = 0; m < 3; ++m) {
        if (!((K.dirs >> m) & 1)) continue;
        double wk0 = 0.0, wk4 = 0.0, st[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int a = 0; a < n; ++a) {
          const int o = (m == 0) ? (a * n + j) * n + k : (m == 1) ? (i * n + a) * n + k : (i * n + j) * n + a;
          const int ii = (m == 0) ? i : (m == 1) ? j : k;
          // D from shared memory: the lanes of a warp index it with different ii (LDC would serialise)
          const double dw = sD[a * n + ii], ds = sD[n * n + a * n + ii];   // D, D^T: lanes vary ii
          wk0 += dw * s[(m * 5 + 0) * nn + o];
          wk4 += dw * s[(m * 5 + 1) * nn + o];
#pragma unroll
          for (int c = 0; c < 3; ++c) st[c] += ds * s[(m * 5 + 2 + c) * nn + o];
        }
        acc[0] += wk0;   // acc -= weak = acc + sum_a D[a,i] (w3 F)_a
        acc[4] += wk4;
#pragma unroll
        for (int c = 0; c < 3; ++c) acc[1 + c] -= w * st[c];
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double sg = 0.0;
#pragma unroll
        for (int m = 0; m < 3; ++m)
          if ((K.dirs >> m) & 1) sg += dphi[m] * gm[m][c];
        acc[1 + c] -= wj * qv[0] * sg;
      }
    }
  } else {
    double* s = sm;  // [0..2]: w3*Jg*rho*un_m ; [3..7]: u, v, w, theta, P
    if (act) {
#pragma unroll
      for (int m = 0; m < 3; ++m) s[m * nn + t] = w * (Jg * qv[0] * un[m]);
#pragma unroll
      for (int f = 0; f < 4; ++f) s[(3 + f) * nn + t] = qv[1 + f];
      s[7 * nn + t] = P;
    }
    __syncthreads();
    if (act) {
      double adv[4] = {0, 0, 0, 0}, pg[3] = {0, 0, 0};
#pragma unroll
      for (int m = 0; m < 3; ++m) {
        if (!((K.dirs >> m) & 1)) continue;
        double wk0 = 0.0, dd[5] = {0, 0, 0, 0, 0};
#pragma unroll
        for (int a = 0; a < n; ++a) {
          const int o = (m == 0) ? (a * n + j) * n + k : (m == 1) ? (i * n + a) * n + k : (i * n + j) * n + a;
          const int ii = (m == 0) ? i : (m == 1) ? j : k;
          const double dw = sD[a * n + ii], ds = sD[n * n + a * n + ii];   // D, D^T: lanes vary ii
          wk0 += dw * s[m * nn + o];
#pragma unroll
          for (int f = 0; f < 5; ++f) dd[f] += ds * s[(3 + f) * nn + o];
        }
        acc[0] += wk0;
#pragma unroll
        for (int f = 0; f < 4; ++f) adv[f] += un[m] * dd[f];
        const double pm = dd[4] / qv[0] + dphi[m];
#pragma unroll
        for (int c = 0; c < 3; ++c) pg[c] += pm * gm[m][c];
      }
#pragma unroll
      for (int f = 0; f < 4; ++f) acc[1 + f] -= wj * adv[f];
#pragma unroll
      for (int c = 0; c < 3; ++c) acc[1 + c] -= wj * pg[c];
    }
  }
  if (!act) return;
  // Coriolis 2 omega e x u (euler.py:183-188, 217-223)
  if (K.omega > 0.0) {
    double ev[3];
    if (K.coriolis == 0) {
#pragma unroll
      for (int c = 0; c < 3; ++c) ev[c] = Mt[(M_RHAT + c) * nloc + p];
    } else {
      const double zn = sqrt(gm[2][0] * gm[2][0] + gm[2][1] * gm[2][1] + gm[2][2] * gm[2][2]);
#pragma unroll
      for (int c = 0; c < 3; ++c) ev[c] = gm[2][c] / zn;
    }
    const double ux = qv[1], uy = qv[2], uz = qv[3];
    const double cx = ev[1] * uz - ev[2] * uy, cy = ev[2] * ux - ev[0] * uz, cz = ev[0] * uy - ev[1] * ux;
    acc[1] -= wj * 2.0 * K.omega * cx;
    acc[2] -= wj * 2.0 * K.omega * cy;
    acc[3] -= wj * 2.0 * K.omega * cz;
  }
}

template <int n>
__global__ void __launch_bounds__(512, (n >= 8 ? 2 : 1)) euler_elem_kernel(hv::DTab<n> Dt, EulerConsts K, int64_t nelem,
                                                         const int32_t* __restrict__ gid, const double* __restrict__ w3,
                                                         const double* __restrict__ Mt, const double* __restrict__ q,
                                                         int64_t ldq, double* __restrict__ work,
                                                         const int32_t* __restrict__ elem_layer, int nlay) {
  constexpr int nn = n * n * n;
  extern __shared__ double sm[];
  const int64_t e = blockIdx.x;
  const int t = threadIdx.x;
  double* sD = sm + 15 * nn;                      // D then D^T (n x n each)
  for (int x = t; x < n * n; x += blockDim.x) {
    sD[x] = Dt.D[x / n][x % n];
    sD[n * n + x] = Dt.D[x % n][x / n];
  }
  double acc[5];
  int g = 0;
  euler_node_acc<n>(Dt, K, nelem, e, t, gid, w3, Mt, q, ldq, sm, acc, g, elem_layer[e], nlay, sD);
  if (t >= nn) return;
  const int64_t nloc = nelem * nn;
  const int64_t p = e * nn + t;
#pragma unroll
  for (int f = 0; f < 5; ++f) work[f * nloc + p] = acc[f];
}

// Column sweep of the Euler RHS on single-column tiles (the N = 7 tile plan, tiles.py): one
// CTA per element column walks the layers; each layer's element accumulator comes from
// euler_node_acc, then the DSS happens on chip: the top level is carried (shared memory,
// double-buffered by layer parity) into the next layer's bottom level, nodes of the column's
// interior (tile-owned) columns get Minv * acc written (or added) to the output row, nodes on
// the element's side faces (shared with neighbouring columns) write 5-wide partial rows that
// slot_fixup sums in fixed order.  Replaces the element kernel + CSR DSS round trip of the
// (5 x nloc) work array.
template <int n>
__global__ void __launch_bounds__(512, (n >= 8 ? 2 : 1)) euler_tile_kernel(hv::DTab<n> Dt, EulerConsts K, int64_t nelem,
                                                         const int32_t* __restrict__ gid, const double* __restrict__ w3,
                                                         const double* __restrict__ Mt, const double* __restrict__ q,
                                                         int64_t ldq, hv::TileArgs A,
                                                         const int32_t* __restrict__ elem) {
  constexpr int nn = n * n * n, N = n - 1;
  extern __shared__ double sm[];
  double* s_carry = sm + 15 * nn;                 // [2][n*n][5]
  int* s_code = reinterpret_cast<int*>(s_carry + 2 * n * n * 5);   // [n*n]
  double* sD = s_carry + 2 * n * n * 5 + (n * n + 1) / 2;           // D then D^T (n x n each)
  const int64_t tl = blockIdx.x;
  const int t = threadIdx.x;
  for (int x = t; x < n * n; x += blockDim.x) {
    sD[x] = Dt.D[x / n][x % n];
    sD[n * n + x] = Dt.D[x % n][x / n];
  }
  const int i = t / (n * n), j = (t / n) % n, k = t % n;
  const int nlay = A.nlay;
  if (t < n * n) s_code[t] = A.code[tl * n * n + t];
  const double* Mt_t = A.Mt + tl * (int64_t)nlay * (((nn + 1) & ~1));
  for (int l = 0; l < nlay; ++l) {
    const int64_t e = elem[tl * nlay + l];
    double acc[5];
    int g = 0;
    euler_node_acc<n>(Dt, K, nelem, e, t, gid, w3, Mt, q, ldq, sm, acc, g, l, nlay, sD);
    if (t < nn) {
      double* cw = s_carry + (l & 1) * n * n * 5 + (i * n + j) * 5;
      const double* cr = s_carry + ((l + 1) & 1) * n * n * 5 + (i * n + j) * 5;
      if (k == 0 && l > 0) {
#pragma unroll
        for (int f = 0; f < 5; ++f) acc[f] = cr[f] + acc[f];   // previous layer's top first
      }
      if (k == N && l < nlay - 1) {
#pragma unroll
        for (int f = 0; f < 5; ++f) cw[f] = acc[f];
      } else {
        const int cd = s_code[i * n + j];
        const int z = l * N + k;
        if (cd < 0) {
          const double m = A.scale * Mt_t[(int64_t)l * ((nn + 1) & ~1) + t];
          double* o = A.out + (int64_t)g * A.ldo;
#pragma unroll
          for (int f = 0; f < 5; ++f) o[f] = A.accumulate ? o[f] + m * acc[f] : m * acc[f];
        } else {
          double* o = A.part + ((int64_t)cd * A.n_z + z) * 5;
#pragma unroll
          for (int f = 0; f < 5; ++f) o[f] = acc[f];
        }
      }
    }
    // the next layer's phase-1 barrier orders the carry / scratch reuse
  }
}

// Column sweep of the 2C / 3C Euler RHS with line tasks (N = 7 single-column tiles; 2NC keeps
// euler_tile_kernel).  Per layer:
//   phase 1  thread = node: gather q, metric record, EOS, contravariant velocities -> the 15 fluxes
//            (3 directions x [w3 F_rho, w3 F_thermo, 3 momentum]) into shared arrays; the geopotential
//            (and Coriolis) terms of the node stay in registers
//   phase 2  thread = (direction, flux, line): the whole line in registers, one even-odd product
//            (-D^T for the weak rho / thermo fluxes, D for the strong momentum fluxes, DTabEO), the
//            results back in place -- one shared load and store per node and flux instead of 8 x 7
//            loads per node and direction in euler_tile_kernel's per-node line sums
//   phase 3  thread = node: sum the directions, the element accumulator (euler.py:191-224), then the
//            same on-chip DSS / carry / partial rows as euler_tile_kernel
// Flux arrays: node (i, j, k) at i*PI + j*n + k with PI = n*n + 1, so the half-warps of phase 1 / 3 and
// of the i- and k-direction lines hit 16 distinct banks (the j-direction lines: 2-way).
// A row of 5 doubles at element offset 5 r of a 16-byte aligned array (state / output rows, 5-wide
// partial rows): 40 bytes, 16-byte aligned when r is even, 8 bytes past that when r is odd -- one
// 8-byte and two 16-byte accesses instead of five 8-byte ones, the same instructions for both parities
__device__ __forceinline__ void ld_row5(const double* row, bool odd, double (&v)[5]) {
  const double a = row[odd ? 0 : 4];
  const double2 b = *reinterpret_cast<const double2*>(row + (odd ? 1 : 0));
  const double2 c = *reinterpret_cast<const double2*>(row + (odd ? 3 : 2));
  v[0] = odd ? a : b.x;
  v[1] = odd ? b.x : b.y;
  v[2] = odd ? b.y : c.x;
  v[3] = odd ? c.x : c.y;
  v[4] = odd ? c.y : a;
}
__device__ __forceinline__ void st_row5(double* row, bool odd, const double (&v)[5]) {
  row[odd ? 0 : 4] = odd ? v[0] : v[4];
  *reinterpret_cast<double2*>(row + (odd ? 1 : 0)) = odd ? make_double2(v[1], v[2]) : make_double2(v[0], v[1]);
  *reinterpret_cast<double2*>(row + (odd ? 3 : 2)) = odd ? make_double2(v[3], v[4]) : make_double2(v[2], v[3]);
}

template <int n>
struct ElinesCfg {
  static constexpr int nn = n * n * n, PI = n * n + 1, FS = ((n - 1) * PI + (n - 1) * n + n + 1) & ~1;
  static constexpr int NL = n * n;                    // lines per direction and flux
  static constexpr int OFF_C = 15 * FS;               // carry [2][n*n][5]
  static constexpr int OFF_CF = OFF_C + 2 * n * n * 5;   // even-odd coefficients (hv::EOSmem)
  static constexpr int OFF_CODE = OFF_CF + 2 * hv::EOSmem<n>::PER;
  static constexpr int OFF_EL = OFF_CODE + (n * n + 1) / 2;   // element of every layer of the column (int, <= 256 layers)
  // staged variant (bulk copies need 16-byte multiples: even n): the next layer's grad xi / eta / zeta
  // and Jg rows (10 x n^3 doubles) and its gids, one mbarrier
  static constexpr bool STG = (n % 2 == 0) && (n * n * n * 4) % 16 == 0;
  static constexpr int NST = 10;
  static constexpr int OFF_ST = (OFF_EL + 128 + 1) & ~1;
  static constexpr int OFF_G = OFF_ST + (STG ? NST * nn : 0);
  static constexpr int OFF_BAR = OFF_G + (STG ? (nn + 1) / 2 : 0);
  static constexpr size_t SMEM = sizeof(double) * (OFF_BAR + (STG ? 2 : 0));
};

// NPT nodes per thread (blockDim = n^3 / NPT): NPT = 2 gives each thread twice the registers (2 x 256
// threads x 128 at N = 7) so that both nodes' phase-1 loads are in flight together
// FAST: the configuration of config 4 fixed at compile time (set 2C, all three directions, no Coriolis):
// no runtime branches on K.set / K.dirs / K.omega in the phases
template <int n, int NPT, bool FAST = false>
__global__ void __launch_bounds__(n * n * n / NPT, (n >= 8 ? 2 : 1)) euler_lines_kernel(hv::DTabEO<n> Dt, EulerConsts Kin,
                                                          int64_t nelem, const int32_t* __restrict__ gid,
                                                          const double* __restrict__ w3,
                                                          const double* __restrict__ Mt, const double* __restrict__ q,
                                                          int64_t ldq, hv::TileArgs A,
                                                          const int32_t* __restrict__ elem) {
  using C = ElinesCfg<n>;
  constexpr int nn = C::nn, N = n - 1, PI = C::PI, FS = C::FS, NB = nn / NPT;
  static_assert(nn % NPT == 0, "nodes per thread");
  struct KC {   // the constants the phases branch on: compile-time in the FAST variant
    double P_A, R, gamma, omega;
    int set, dirs, coriolis;
  };
  const KC K = FAST ? KC{Kin.P_A, Kin.R, Kin.gamma, 0.0, 1, 7, 0}
                    : KC{Kin.P_A, Kin.R, Kin.gamma, Kin.omega, Kin.set, Kin.dirs, Kin.coriolis};
  extern __shared__ double sm[];
  double* s_f = sm;                                      // [15][FS] fluxes, then line results
  double* s_carry = sm + C::OFF_C;                       // [2][n*n][5]
  int* s_code = reinterpret_cast<int*>(sm + C::OFF_CODE);
  double* s_cf = sm + C::OFF_CF;
  const int64_t tl = blockIdx.x;
  const int t0 = threadIdx.x;
  hv::eo_smem_fill<n>(Dt, s_cf, t0, blockDim.x);   // visible after the first layer's phase-1 barrier
  const int nlay = A.nlay;
  const int64_t nloc = nelem * nn;
  for (int x = t0; x < n * n; x += blockDim.x) s_code[x] = A.code[tl * n * n + x];
  // the column's elements in shared memory and the next layer's gids in registers: a layer's phase 1
  // then starts with the q-row loads instead of the chain elem -> gid -> q row
  int* s_el = reinterpret_cast<int*>(sm + C::OFF_EL);
  for (int x = t0; x < nlay; x += blockDim.x) s_el[x] = elem[tl * nlay + x];
  const double* Mt_t = A.Mt + tl * (int64_t)nlay * (((nn + 1) & ~1));
  constexpr bool STG = C::STG;
  // 16-byte row accesses (ld_row5 / st_row5) when the rows are 5 wide and the arrays 16-byte aligned
  const bool vq = ldq == 5 && (reinterpret_cast<uintptr_t>(q) & 15) == 0;
  const bool vo = A.ldo == 5 && (reinterpret_cast<uintptr_t>(A.out) & 15) == 0 && (reinterpret_cast<uintptr_t>(A.part) & 15) == 0;
  const double* s_m = sm + C::OFF_ST;                    // [NST][nn] staged record rows of the current layer
  const int* s_g = reinterpret_cast<const int*>(sm + C::OFF_G);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + C::OFF_BAR);
  // layer le's rows 0..9 of the record (grad xi, eta, zeta; Jg) and gids -> the stage: 11 bulk copies on
  // one mbarrier phase, ~43 KB in flight per CTA while the previous layer's phases 2 and 3 run (the
  // per-thread loads they replace kept ~4 loads in flight per thread: latency-bound at 2.9 TB/s)
  auto issue_stage = [&](int64_t en) {
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(bar);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"((uint32_t)(C::NST * nn * 8 + nn * 4))
                 : "memory");
#pragma unroll 1
    for (int c = 0; c < C::NST; ++c)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       (uint32_t)__cvta_generic_to_shared(s_m + c * nn)),
                   "l"(Mt + c * nloc + en * nn), "r"((uint32_t)(nn * 8)), "r"(b)
                   : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(s_g)),
                 "l"(gid + en * nn), "r"((uint32_t)(nn * 4)), "r"(b)
                 : "memory");
  };
  if constexpr (STG) {
    if (t0 == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
  }
  const double rPA = __drcp_rn(K.P_A);                   // quotients by P_A and rho: hv::div_rcp (hv_pow.cuh)
  double w[NPT];
  int gnx[NPT];                                          // gids of the next layer's nodes (unstaged variant)
#pragma unroll
  for (int jn = 0; jn < NPT; ++jn) {
    w[jn] = (t0 + jn * NB < nn) ? w3[t0 + jn * NB] : 0.0;
    gnx[jn] = (!STG && t0 + jn * NB < nn) ? gid[(int64_t)elem[tl * nlay] * nn + t0 + jn * NB] : 0;
  }
  __syncthreads();
  if constexpr (STG) {
    if (t0 == 0) issue_stage(s_el[0]);
  }
  auto wait_stage = [&](int le) {   // layer le's stage has landed
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(bar), par = (uint32_t)(le & 1);
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                   : "=r"(done)
                   : "r"(b), "r"(par)
                   : "memory");
  };
  // staged variant: a layer's gids and q rows are read at the END of the previous layer's phase 3 (the stage
  // has landed by then), so the q-row loads fly across the layer barrier instead of heading phase 1
  int gq[NPT];
  double qn[NPT][5];
  auto load_q = [&]() {
#pragma unroll
    for (int jn = 0; jn < NPT; ++jn) {
      const int t = t0 + jn * NB;
      gq[jn] = 0;
#pragma unroll
      for (int f = 0; f < 5; ++f) qn[jn][f] = 0.0;
      if (t >= nn) continue;
      const int g = s_g[t];
      gq[jn] = g;
      if (vq) {   // raw pieces (ld_row5's loads); the parity selects wait for the data, so they happen in phase 1
        const double* row = q + (int64_t)g * 5;
        const bool odd = g & 1;
        qn[jn][0] = row[odd ? 0 : 4];
        const double2 b = *reinterpret_cast<const double2*>(row + (odd ? 1 : 0));
        const double2 c = *reinterpret_cast<const double2*>(row + (odd ? 3 : 2));
        qn[jn][1] = b.x;
        qn[jn][2] = b.y;
        qn[jn][3] = c.x;
        qn[jn][4] = c.y;
      } else {
#pragma unroll
        for (int f = 0; f < 5; ++f) qn[jn][f] = q[(int64_t)g * ldq + f];
      }
    }
  };
  if constexpr (STG) {
    wait_stage(0);
    load_q();
  }
  for (int l = 0; l < nlay; ++l) {
    const int64_t e = s_el[l];
    double extra[NPT][3];                                // geopotential + Coriolis terms of acc[1..3]
    int gn[NPT];
    // ---- phase 1 (euler_node_acc's fluxes, reference expression order), node t = t0 + jn * NB
#pragma unroll
    for (int jn = 0; jn < NPT; ++jn) {
      const int t = t0 + jn * NB;
      const bool act = t < nn;
      const int k = t % n;
      const int na = (t / (n * n)) * PI + ((t / n) % n) * n + k;
      const int64_t p = e * nn + (act ? t : 0);
      extra[jn][0] = extra[jn][1] = extra[jn][2] = 0.0;
      gn[jn] = 0;
      if (!act) continue;
      const int g = STG ? gq[jn] : gnx[jn];
      gn[jn] = g;
      if (!STG && l + 1 < nlay) gnx[jn] = gid[(int64_t)s_el[l + 1] * nn + t];
      double qv[5];
      if constexpr (STG) {
        const bool odd = vq && (g & 1);                  // ld_row5's selects on load_q's raw pieces
        qv[0] = (!vq || odd) ? qn[jn][0] : qn[jn][1];
        qv[1] = !vq ? qn[jn][1] : (odd ? qn[jn][1] : qn[jn][2]);
        qv[2] = !vq ? qn[jn][2] : (odd ? qn[jn][2] : qn[jn][3]);
        qv[3] = !vq ? qn[jn][3] : (odd ? qn[jn][3] : qn[jn][4]);
        qv[4] = !vq ? qn[jn][4] : (odd ? qn[jn][4] : qn[jn][0]);
      } else if (vq) {
        ld_row5(q + (int64_t)g * 5, g & 1, qv);
      } else {
#pragma unroll
        for (int f = 0; f < 5; ++f) qv[f] = q[(int64_t)g * ldq + f];
      }
      const double Jg = STG ? s_m[9 * nn + t] : Mt[9 * nloc + p];
      const double mask = ((l == 0 && k == 0) || (l == nlay - 1 && k == n - 1)) ? 0.0 : 1.0;
      const double rho = qv[0];
      double P;
      if (K.set == 1) {
        P = K.P_A * hv::pow_pos(hv::div_rcp(K.R * qv[4], K.P_A, rPA), K.gamma);
      } else {
        const double phi = Mt[14 * nloc + p];
        const double ke = 0.5 * (qv[1] * qv[1] + qv[2] * qv[2] + qv[3] * qv[3]) / rho;
        P = (K.gamma - 1.0) * (qv[4] - ke - rho * phi);
      }
      const double rrho = __drcp_rn(rho);   // the node's four quotients by rho: div_rcp
      const double tflux = (K.set == 1) ? hv::div_rcp(qv[4], rho, rrho) : hv::div_rcp(qv[4] + P, rho, rrho);
      double sg[3] = {0.0, 0.0, 0.0};
      // one direction at a time: grad xi^m (3 doubles) live only inside its iteration
#pragma unroll
      for (int m = 0; m < 3; ++m) {
        double gm[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) gm[c] = STG ? s_m[(m * 3 + c) * nn + t] : Mt[(m * 3 + c) * nloc + p];
        double un = hv::div_rcp(gm[0] * qv[1] + gm[1] * qv[2] + gm[2] * qv[3], rho, rrho);
        if (m == 2) un = un * mask;
        const double jun = Jg * un;
        s_f[(m * 5 + 0) * FS + na] = w[jn] * (jun * qv[0]);
        s_f[(m * 5 + 1) * FS + na] = w[jn] * (jun * qv[0] * tflux);
#pragma unroll
        for (int c = 0; c < 3; ++c) s_f[(m * 5 + 2 + c) * FS + na] = Jg * (qv[1 + c] * un + P * gm[c]);
        if ((K.dirs >> m) & 1) {
          const double dphi = Mt[(10 + m) * nloc + p];
#pragma unroll
          for (int c = 0; c < 3; ++c) sg[c] += dphi * gm[c];
        }
      }
      const double wj = w[jn] * Jg;
#pragma unroll
      for (int c = 0; c < 3; ++c) extra[jn][c] = wj * qv[0] * sg[c];
      if (K.omega > 0.0) {   // Coriolis 2 omega e x u (euler.py:183-188, 217-223)
        double ev[3];
        if (K.coriolis == 0) {
#pragma unroll
          for (int c = 0; c < 3; ++c) ev[c] = Mt[(15 + c) * nloc + p];
        } else {
          double gz[3];
#pragma unroll
          for (int c = 0; c < 3; ++c) gz[c] = STG ? s_m[(6 + c) * nn + t] : Mt[(6 + c) * nloc + p];
          const double zn = sqrt(gz[0] * gz[0] + gz[1] * gz[1] + gz[2] * gz[2]);
#pragma unroll
          for (int c = 0; c < 3; ++c) ev[c] = gz[c] / zn;
        }
        const double ux = qv[1], uy = qv[2], uz = qv[3];
        const double cx = ev[1] * uz - ev[2] * uy, cy = ev[2] * ux - ev[0] * uz, cz = ev[0] * uy - ev[1] * ux;
        extra[jn][0] += wj * 2.0 * K.omega * cx;
        extra[jn][1] += wj * 2.0 * K.omega * cy;
        extra[jn][2] += wj * 2.0 * K.omega * cz;
      }
    }
    __syncthreads();
    // the next layer's element record: the staged rows (grad xi / eta / zeta, Jg) and gids by bulk copy into
    // the stage, free now that every thread is past its phase-1 reads; the rows phase 1 and 3 load
    // directly (dPhi_m, M^-1; everything in the unstaged variant) -> L2, so that those loads wait for L2
    // rather than DRAM
    if constexpr (STG) {
      if (t0 == 32 && l + 1 < nlay) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue_stage(s_el[l + 1]);
      }
    }
    if (l + 1 < nlay && t0 < 16) {
      const int64_t en = s_el[l + 1];
      const void* src = nullptr;
      uint32_t bytes = nn * 8;
      if (t0 < 13) { if (!STG || t0 >= C::NST) src = Mt + t0 * nloc + en * nn; }
      else if (t0 == 13) { if (!STG) { src = gid + en * nn; bytes = nn * 4; } }
      else if (t0 == 14) { src = Mt_t + (int64_t)(l + 1) * ((nn + 1) & ~1); bytes = ((nn + 1) & ~1) * 8; }
      if (src && (bytes & 15) == 0 && (reinterpret_cast<uintptr_t>(src) & 15) == 0)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
    }
    // ---- phase 2: line tasks (direction m, flux x, line); warp-uniform (m, x)
#pragma unroll 1
    for (int T = t0; T < 15 * C::NL; T += blockDim.x) {
      const int m = T / (5 * C::NL), x = (T / C::NL) % 5, lam = T % C::NL;
      if (!((K.dirs >> m) & 1)) continue;
      int base, stride;
      if (m == 0) { base = (lam / n) * n + lam % n; stride = PI; }          // line (j, k)
      else if (m == 1) { base = (lam / n) * PI + lam % n; stride = n; }     // line (i, k)
      else { base = (lam % n) * PI + (lam / n) * n; stride = 1; }           // line (i, j)
      double* fl = s_f + (m * 5 + x) * FS + base;
      double xl[n];
#pragma unroll
      for (int a = 0; a < n; ++a) xl[a] = fl[a * stride];
      if (x < 2) hv::eo_mv_st_s<n, 1>(s_cf, xl, fl, stride);   // -D^T (weak), in place
      else hv::eo_mv_st_s<n, 0>(s_cf, xl, fl, stride);         // D (strong), in place
    }
    __syncthreads();
    // ---- phase 3: element accumulator, then the column DSS
    if constexpr (STG) {   // the next layer's q rows towards L1 / L2 now (its gids have landed); loaded at the end of the phase
      if (l + 1 < nlay) {
        wait_stage(l + 1);
#pragma unroll
        for (int jn = 0; jn < NPT; ++jn)
          if (t0 + jn * NB < nn)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(q + (int64_t)s_g[t0 + jn * NB] * ldq + 2));
      }
    }
#pragma unroll
    for (int jn = 0; jn < NPT; ++jn) {
      const int t = t0 + jn * NB;
      if (t >= nn) continue;
      const int i = t / (n * n), j = (t / n) % n, k = t % n;
      const int na = i * PI + j * n + k;
      // where this node's result goes -- the final row M^-1 acc of a node the column owns, or the raw sums
      // into its 5-wide partial row (perimeter nodes; slot_fixup sums them) -- and the global loads of the
      // store (M^-1, the row's previous value when accumulating) first: they fly during the sums below
      const bool carry_up = (k == N && l < nlay - 1);       // top level: carried into the next layer
      const int cd = s_code[i * n + j];
      const bool fin = cd < 0;
      const int64_t ro = fin ? (int64_t)gn[jn] : (int64_t)cd * A.n_z + l * N + k;
      double* o = fin ? A.out + ro * A.ldo : A.part + ro * 5;
      const double mraw = (fin && !carry_up) ? Mt_t[(int64_t)l * ((nn + 1) & ~1) + t] : 1.0;
      // the row's previous value as ld_row5's raw pieces (the parity selects, which wait for the data, at the use)
      const bool oodd = ro & 1;
      double pa = 0.0;
      double2 pb = make_double2(0.0, 0.0), pc = make_double2(0.0, 0.0);
      if (vo && A.accumulate && fin && !carry_up) {
        pa = o[oodd ? 0 : 4];
        pb = *reinterpret_cast<const double2*>(o + (oodd ? 1 : 0));
        pc = *reinterpret_cast<const double2*>(o + (oodd ? 3 : 2));
      }
      double acc[5];
      double r[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int m = 0; m < 3; ++m)
        if ((K.dirs >> m) & 1) {
#pragma unroll
          for (int x = 0; x < 5; ++x) r[x] += s_f[(m * 5 + x) * FS + na];
        }
      acc[0] = -r[0];                                   // acc -= weak = acc + sum_a D[a,i] (w3 F)_a
      acc[4] = -r[1];
#pragma unroll
      for (int c = 0; c < 3; ++c) acc[1 + c] = -(w[jn] * r[2 + c]) - extra[jn][c];
      double* cw = s_carry + (l & 1) * n * n * 5 + (i * n + j) * 5;
      const double* cr = s_carry + ((l + 1) & 1) * n * n * 5 + (i * n + j) * 5;
      if (k == 0 && l > 0) {
#pragma unroll
        for (int f = 0; f < 5; ++f) acc[f] = cr[f] + acc[f];   // previous layer's top first
      }
      if (carry_up) {
#pragma unroll
        for (int f = 0; f < 5; ++f) cw[f] = acc[f];
      } else {
        const double mi = fin ? A.scale * mraw : 1.0;
        double v[5];
#pragma unroll
        for (int f = 0; f < 5; ++f) v[f] = fin ? mi * acc[f] : acc[f];
        if (vo) {
          if (A.accumulate && fin) {
            v[0] = (oodd ? pa : pb.x) + v[0];
            v[1] = (oodd ? pb.x : pb.y) + v[1];
            v[2] = (oodd ? pb.y : pc.x) + v[2];
            v[3] = (oodd ? pc.x : pc.y) + v[3];
            v[4] = (oodd ? pc.y : pa) + v[4];
          }
          st_row5(o, oodd, v);
        } else {
#pragma unroll
          for (int f = 0; f < 5; ++f) o[f] = (A.accumulate && fin) ? o[f] + v[f] : v[f];
        }
      }
    }
    if constexpr (STG) {
      if (l + 1 < nlay) {
        wait_stage(l + 1);
        load_q();
      }
    }
    // no barrier here: phase 3 reads and the next layer's phase 1 writes only the thread's OWN node's
    // entries of the flux arrays, and a carry slot is rewritten two barriers after its last read
  }
}

template <int n>
int run_lines(const double* Drow, const EulerConsts& K, int64_t nelem, const int32_t* gid, const double* w3,
              const double* Mt, const double* q, int64_t ldq, const hv::TileArgs& A, const int32_t* elem,
              cudaStream_t st) {
  hv::DTabEO<n> Dt;
  hv::fill_dtab_eo(Dt, Drow);
  using C = ElinesCfg<n>;
  // one node per thread; HV_EULER_NPT=2 at N = 7: two (2 x 256 threads x 120 registers: both nodes' loads in
  // flight together, but half the warps -- c4 Euler sweep 2.26 -> 2.87 ms, not taken)
  const char* ev = getenv("HV_EULER_NPT");
  if (n == 8 && ev && atoi(ev) == 2) {
    auto kern = euler_lines_kernel<n, (n == 8 ? 2 : 1)>;
    HV_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
    kern<<<(unsigned)A.ntiles, C::nn / (n == 8 ? 2 : 1), C::SMEM, st>>>(Dt, K, nelem, gid, w3, Mt, q, ldq, A, elem);
  } else {
    const bool fast = n == 8 && K.set == 1 && K.dirs == 7 && !(K.omega > 0.0);
    auto kern = fast ? euler_lines_kernel<n, 1, true> : euler_lines_kernel<n, 1, false>;
    HV_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
    kern<<<(unsigned)A.ntiles, ((C::nn + 31) / 32) * 32, C::SMEM, st>>>(Dt, K, nelem, gid, w3, Mt, q, ldq, A, elem);
  }
  HV_LAUNCH_CHECK();
  return HV_OK;
}

template <int n>
int run_tile(const double* Drow, const EulerConsts& K, int64_t nelem, const int32_t* gid, const double* w3,
             const double* Mt, const double* q, int64_t ldq, const hv::TileArgs& A, const int32_t* elem,
             cudaStream_t st) {
  // 2C / 3C at N >= 4: the line-task kernel (HV_EULER_LINES=0 keeps the per-node line sums)
  if constexpr (n >= 5) {
    const char* ev = getenv("HV_EULER_LINES");
    if (K.set != 0 && A.nlay <= 256 && !(ev && atoi(ev) == 0)) return run_lines<n>(Drow, K, nelem, gid, w3, Mt, q, ldq, A, elem, st);
  }
  hv::DTab<n> Dt;
  hv::fill_dtab(Dt, Drow);
  constexpr int nn = n * n * n;
  const size_t smem = sizeof(double) * (15 * nn + 2 * n * n * 5 + (n * n + 1) / 2 + 2 * n * n);
  auto kern = euler_tile_kernel<n>;
  HV_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<(unsigned)A.ntiles, ((nn + 31) / 32) * 32, smem, st>>>(Dt, K, nelem, gid, w3, Mt, q, ldq, A, elem);
  HV_LAUNCH_CHECK();
  return HV_OK;
}

template <int n>
int run_setup(const double* Drow, int64_t nelem, const int32_t* gid, const double* grad, const double* Jg,
              const double* gz, const double* Phi_g, const double* mask_g, const double* coords, int sphere,
              double* Mout, cudaStream_t st) {
  hv::DTab<n> Dt;
  hv::fill_dtab(Dt, Drow);
  constexpr int nn = n * n * n;
  euler_setup_kernel<n><<<(unsigned)nelem, ((nn + 31) / 32) * 32, 0, st>>>(Dt, nelem, gid, grad, Jg, gz, Phi_g, mask_g,
                                                                           coords, sphere, Mout);
  HV_LAUNCH_CHECK();
  return HV_OK;
}

template <int n>
int run_elem(const double* Drow, const EulerConsts& K, int64_t nelem, const int32_t* gid, const double* w3,
             const double* Mt, const double* q, int64_t ldq, double* work, const int32_t* elem_layer, int nlay,
             cudaStream_t st) {
  hv::DTab<n> Dt;
  hv::fill_dtab(Dt, Drow);
  constexpr int nn = n * n * n;
  const size_t smem = sizeof(double) * (15 * nn + 2 * n * n);
  auto kern = euler_elem_kernel<n>;
  if (smem > 48 * 1024) HV_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<(unsigned)nelem, ((nn + 31) / 32) * 32, smem, st>>>(Dt, K, nelem, gid, w3, Mt, q, ldq, work, elem_layer, nlay);
  HV_LAUNCH_CHECK();
  return HV_OK;
}

}  // namespace

extern "C" int hv_euler_setup(int N, const double* h_D, int64_t nelem, const int32_t* d_gid, const double* d_grad,
                              const double* d_Jg, const double* d_gz, const double* d_Phi_g, const double* d_mask_g,
                              const double* d_coords, int sphere, double* d_M, void* stream) {
  if (N < 1 || N > 7 || !h_D || nelem <= 0 || !d_gid || !d_grad || !d_Jg || !d_gz || !d_Phi_g || !d_mask_g ||
      !d_coords || !d_M)
    HV_FAIL(HV_ERR_INVALID, "hv_euler_setup: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  switch (N + 1) {
    case 2: return run_setup<2>(h_D, nelem, d_gid, d_grad, d_Jg, d_gz, d_Phi_g, d_mask_g, d_coords, sphere, d_M, st);
    case 3: return run_setup<3>(h_D, nelem, d_gid, d_grad, d_Jg, d_gz, d_Phi_g, d_mask_g, d_coords, sphere, d_M, st);
    case 4: return run_setup<4>(h_D, nelem, d_gid, d_grad, d_Jg, d_gz, d_Phi_g, d_mask_g, d_coords, sphere, d_M, st);
    case 5: return run_setup<5>(h_D, nelem, d_gid, d_grad, d_Jg, d_gz, d_Phi_g, d_mask_g, d_coords, sphere, d_M, st);
    case 6: return run_setup<6>(h_D, nelem, d_gid, d_grad, d_Jg, d_gz, d_Phi_g, d_mask_g, d_coords, sphere, d_M, st);
    case 7: return run_setup<7>(h_D, nelem, d_gid, d_grad, d_Jg, d_gz, d_Phi_g, d_mask_g, d_coords, sphere, d_M, st);
    default: return run_setup<8>(h_D, nelem, d_gid, d_grad, d_Jg, d_gz, d_Phi_g, d_mask_g, d_coords, sphere, d_M, st);
  }
}

extern "C" int hv_euler_rhs(int N, const double* h_D, int set_id, int dirs, int coriolis, double P_A, double R,
                            double gamma, double omega, int64_t nelem, int64_t nglobal, const int32_t* d_gid,
                            const int32_t* d_elem_layer, int nlay,
                            const double* d_w3, const double* d_M, const int64_t* d_off, const int32_t* d_idx,
                            const double* d_Minv, const double* d_q, int64_t ldq, double* d_work, double* d_out,
                            int64_t ldo, int accumulate, void* stream) {
  if (N < 1 || N > 7 || set_id < 0 || set_id > 2 || dirs <= 0 || dirs > 7 || !d_q || !d_out || !d_work || ldq < 5 ||
      ldo < 5 || !d_elem_layer || nlay < 1)
    HV_FAIL(HV_ERR_INVALID, "hv_euler_rhs: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  EulerConsts K{P_A, R, gamma, omega, set_id, dirs, coriolis};
  int rc;
  switch (N + 1) {
    case 2: rc = run_elem<2>(h_D, K, nelem, d_gid, d_w3, d_M, d_q, ldq, d_work, d_elem_layer, nlay, st); break;
    case 3: rc = run_elem<3>(h_D, K, nelem, d_gid, d_w3, d_M, d_q, ldq, d_work, d_elem_layer, nlay, st); break;
    case 4: rc = run_elem<4>(h_D, K, nelem, d_gid, d_w3, d_M, d_q, ldq, d_work, d_elem_layer, nlay, st); break;
    case 5: rc = run_elem<5>(h_D, K, nelem, d_gid, d_w3, d_M, d_q, ldq, d_work, d_elem_layer, nlay, st); break;
    case 6: rc = run_elem<6>(h_D, K, nelem, d_gid, d_w3, d_M, d_q, ldq, d_work, d_elem_layer, nlay, st); break;
    case 7: rc = run_elem<7>(h_D, K, nelem, d_gid, d_w3, d_M, d_q, ldq, d_work, d_elem_layer, nlay, st); break;
    default: rc = run_elem<8>(h_D, K, nelem, d_gid, d_w3, d_M, d_q, ldq, d_work, d_elem_layer, nlay, st); break;
  }
  if (rc) return rc;
  const int n = N + 1;
  return hv::dss_minv_accumulate(d_work, nelem * n * n * n, d_off, d_idx, d_Minv, nglobal, d_out, ldo, 5,
                                 accumulate != 0, st);
}

// ---------------------------------------------------------------------------
// V(q): the vertical (zeta) operator evaluated column by column
// (EulerOps.rhs_vertical / column_apply / _col_acc, euler.py:61-94,138-144,231-272).
// One thread per column walks its layers bottom to top with the layer's zeta
// line in registers; the shared node between layers is summed as the
// reference's _col_assemble does (previous top first), then divided by the
// column mass DSS(w_z J).
namespace {

template <int n>
__global__ void euler_vertical_kernel(hv::DTab<n> Dt, EulerConsts K, hv::DTab<n> Wz, int64_t ncol, int nlay, int n_z,
                                      const int32_t* __restrict__ col_gid, const double* __restrict__ Jg,
                                      const double* __restrict__ gz, const double* __restrict__ mask_g,
                                      const double* __restrict__ Phi_g, const double* __restrict__ q, int64_t ldq,
                                      double* __restrict__ out, int64_t ldo, int accumulate) {
  constexpr int N = n - 1;
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= ncol) return;
  const int32_t* cg = col_gid + c * (int64_t)n_z;
  double carry[5] = {0, 0, 0, 0, 0}, carry_m = 0.0;
  auto emit = [&](int g, const double* a, double m) {
    double* o = out + (int64_t)g * ldo;
#pragma unroll
    for (int f = 0; f < 5; ++f) o[f] = accumulate ? o[f] + a[f] / m : a[f] / m;
  };
  for (int l = 0; l < nlay; ++l) {
    int g[n];
    double qv[n][5], J[n], z[n][3], msk[n], phi[n], P[n], uz[n], tf[n];
#pragma unroll
    for (int i = 0; i < n; ++i) {
      g[i] = cg[l * N + i];
#pragma unroll
      for (int f = 0; f < 5; ++f) qv[i][f] = q[(int64_t)g[i] * ldq + f];
      J[i] = Jg[g[i]];
#pragma unroll
      for (int d = 0; d < 3; ++d) z[i][d] = gz[(int64_t)g[i] * 3 + d];
      msk[i] = mask_g[g[i]];
      phi[i] = Phi_g[g[i]];
      const double rho = qv[i][0];
      if (K.set == 0) {
        P[i] = K.P_A * hv::pow_pos(qv[i][0] * K.R * qv[i][4] / K.P_A, K.gamma);
        uz[i] = msk[i] * (qv[i][1] * z[i][0] + qv[i][2] * z[i][1] + qv[i][3] * z[i][2]);
        tf[i] = 0.0;
      } else {
        if (K.set == 1) {
          P[i] = K.P_A * hv::pow_pos(K.R * qv[i][4] / K.P_A, K.gamma);
        } else {
          const double ke = 0.5 * (qv[i][1] * qv[i][1] + qv[i][2] * qv[i][2] + qv[i][3] * qv[i][3]) / rho;
          P[i] = (K.gamma - 1.0) * (qv[i][4] - ke - rho * phi[i]);
        }
        uz[i] = msk[i] * (qv[i][1] * z[i][0] + qv[i][2] * z[i][1] + qv[i][3] * z[i][2]) / rho;
        tf[i] = (K.set == 1) ? qv[i][4] / rho : (qv[i][4] + P[i]) / rho;
      }
    }
    double acc[n][5], ms[n];
#pragma unroll
    for (int i = 0; i < n; ++i) {
      const double wj = Wz.D[0][i] * J[i];
      ms[i] = wj;
      double dphi = 0.0;
#pragma unroll
      for (int a = 0; a < n; ++a) dphi += Dt.D[i][a] * phi[a];
      if (K.set == 0) {
        double a0 = 0.0, dP = 0.0, du[4] = {0, 0, 0, 0};
#pragma unroll
        for (int a = 0; a < n; ++a) {
          a0 += Dt.D[a][i] * (Wz.D[0][a] * (J[a] * qv[a][0] * uz[a]));
          dP += Dt.D[i][a] * P[a];
#pragma unroll
          for (int f = 0; f < 4; ++f) du[f] += Dt.D[i][a] * qv[a][1 + f];
        }
        acc[i][0] = a0;
#pragma unroll
        for (int cc = 0; cc < 3; ++cc)
          acc[i][1 + cc] = -wj * (uz[i] * du[cc] + (z[i][cc] / qv[i][0]) * dP + z[i][cc] * dphi);
        acc[i][4] = -wj * uz[i] * du[3];
      } else {
        double a0 = 0.0, a4 = 0.0, dm[3] = {0, 0, 0};
#pragma unroll
        for (int a = 0; a < n; ++a) {
          const double jru = J[a] * qv[a][0] * uz[a];
          a0 += Dt.D[a][i] * (Wz.D[0][a] * jru);
          a4 += Dt.D[a][i] * (Wz.D[0][a] * (jru * tf[a]));
#pragma unroll
          for (int cc = 0; cc < 3; ++cc) dm[cc] += Dt.D[i][a] * (J[a] * (qv[a][1 + cc] * uz[a] + P[a] * z[a][cc]));
        }
        acc[i][0] = a0;
        acc[i][4] = a4;
#pragma unroll
        for (int cc = 0; cc < 3; ++cc) acc[i][1 + cc] = -Wz.D[0][i] * dm[cc] - wj * qv[i][0] * dphi * z[i][cc];
      }
    }
    // column DSS: node 0 of this layer is node N of the previous one
    if (l > 0) {
#pragma unroll
      for (int f = 0; f < 5; ++f) acc[0][f] = carry[f] + acc[0][f];
      ms[0] = carry_m + ms[0];
    }
#pragma unroll
    for (int i = 0; i < N; ++i) emit(g[i], acc[i], ms[i]);
#pragma unroll
    for (int f = 0; f < 5; ++f) carry[f] = acc[N][f];
    carry_m = ms[N];
    if (l == nlay - 1) emit(g[N], acc[N], ms[N]);
  }
}

template <int n>
int run_vertical(const double* Drow, const double* w, const EulerConsts& K, int64_t ncol, int nlay, int n_z,
                 const int32_t* col_gid, const double* Jg, const double* gz, const double* mask, const double* Phi,
                 const double* q, int64_t ldq, double* out, int64_t ldo, int accumulate, cudaStream_t st) {
  hv::DTab<n> Dt, Wz{};
  hv::fill_dtab(Dt, Drow);
  for (int i = 0; i < n; ++i) Wz.D[0][i] = w[i];
  const int T = 128;
  euler_vertical_kernel<n><<<(unsigned)((ncol + T - 1) / T), T, 0, st>>>(Dt, K, Wz, ncol, nlay, n_z, col_gid, Jg, gz,
                                                                         mask, Phi, q, ldq, out, ldo, accumulate);
  HV_LAUNCH_CHECK();
  return HV_OK;
}

}  // namespace

extern "C" int hv_euler_vertical(int N, const double* h_D, const double* h_w, int set_id, double P_A, double R,
                                 double gamma, int64_t ncol, int nlay, int n_z, const int32_t* d_col_gid,
                                 const double* d_Jg, const double* d_gz, const double* d_mask_g,
                                 const double* d_Phi_g, const double* d_q, int64_t ldq, double* d_out, int64_t ldo,
                                 int accumulate, void* stream) {
  if (N < 1 || N > 7 || !h_D || !h_w || set_id < 0 || set_id > 2 || ncol <= 0 || nlay <= 0 || n_z != nlay * N + 1 ||
      !d_col_gid || !d_Jg || !d_gz || !d_mask_g || !d_Phi_g || !d_q || !d_out || ldq < 5 || ldo < 5)
    HV_FAIL(HV_ERR_INVALID, "hv_euler_vertical: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  EulerConsts K{P_A, R, gamma, 0.0, set_id, 4, 0};
  switch (N + 1) {
    case 2: return run_vertical<2>(h_D, h_w, K, ncol, nlay, n_z, d_col_gid, d_Jg, d_gz, d_mask_g, d_Phi_g, d_q, ldq, d_out, ldo, accumulate, st);
    case 3: return run_vertical<3>(h_D, h_w, K, ncol, nlay, n_z, d_col_gid, d_Jg, d_gz, d_mask_g, d_Phi_g, d_q, ldq, d_out, ldo, accumulate, st);
    case 4: return run_vertical<4>(h_D, h_w, K, ncol, nlay, n_z, d_col_gid, d_Jg, d_gz, d_mask_g, d_Phi_g, d_q, ldq, d_out, ldo, accumulate, st);
    case 5: return run_vertical<5>(h_D, h_w, K, ncol, nlay, n_z, d_col_gid, d_Jg, d_gz, d_mask_g, d_Phi_g, d_q, ldq, d_out, ldo, accumulate, st);
    case 6: return run_vertical<6>(h_D, h_w, K, ncol, nlay, n_z, d_col_gid, d_Jg, d_gz, d_mask_g, d_Phi_g, d_q, ldq, d_out, ldo, accumulate, st);
    case 7: return run_vertical<7>(h_D, h_w, K, ncol, nlay, n_z, d_col_gid, d_Jg, d_gz, d_mask_g, d_Phi_g, d_q, ldq, d_out, ldo, accumulate, st);
    default: return run_vertical<8>(h_D, h_w, K, ncol, nlay, n_z, d_col_gid, d_Jg, d_gz, d_mask_g, d_Phi_g, d_q, ldq, d_out, ldo, accumulate, st);
  }
}

// ---------------------------------------------------------------------------
// Diagnostics (EulerOps.diagnostics, euler.py:421-456): quadrature-weighted global
// integrals (M-weighted sums) and the surface-pressure minimum / vertical-velocity
// maximum.  Two-stage deterministic reduction: a fixed grid of DIAG_BLOCKS blocks writes
// partials, one block combines them in block order (run-to-run bitwise reproducible).
namespace {

constexpr int DIAG_BLOCKS = 592, DIAG_T = 256;
// partial layout per block: 5 sums (mass, e_int, e_kin, e_pot, e_tot3C), max |w|, min P_surface
constexpr int DIAG_NP = 7;

__device__ __forceinline__ void block_reduce(double (&v)[DIAG_NP], double* sh) {
  const int t = threadIdx.x;
#pragma unroll
  for (int k = 0; k < DIAG_NP; ++k) sh[k * DIAG_T + t] = v[k];
  __syncthreads();
  for (int s = DIAG_T / 2; s > 0; s >>= 1) {
    if (t < s) {
#pragma unroll
      for (int k = 0; k < 5; ++k) sh[k * DIAG_T + t] += sh[k * DIAG_T + t + s];
      sh[5 * DIAG_T + t] = fmax(sh[5 * DIAG_T + t], sh[5 * DIAG_T + t + s]);
      sh[6 * DIAG_T + t] = fmin(sh[6 * DIAG_T + t], sh[6 * DIAG_T + t + s]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int k = 0; k < DIAG_NP; ++k) v[k] = sh[k * DIAG_T];
}

__global__ void __launch_bounds__(DIAG_T) diag_partial_kernel(EulerConsts K, double c_v, int sphere, int64_t ng,
                                                              const double* __restrict__ q,
                                                              const double* __restrict__ Mm,
                                                              const double* __restrict__ Phi,
                                                              const double* __restrict__ xg, int64_t ncol, int n_z,
                                                              const int32_t* __restrict__ col_gid,
                                                              double* __restrict__ part) {
  __shared__ double sh[DIAG_NP * DIAG_T];
  double v[DIAG_NP] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, INFINITY};
  for (int64_t g = blockIdx.x * (int64_t)DIAG_T + threadIdx.x; g < ng; g += (int64_t)DIAG_BLOCKS * DIAG_T) {
    const double* r = q + g * 5;
    const double rho = r[0], m = Mm[g], phi = Phi[g];
    double P;
    if (K.set == 0) P = K.P_A * hv::pow_pos(rho * K.R * r[4] / K.P_A, K.gamma);
    else if (K.set == 1) P = K.P_A * hv::pow_pos(K.R * r[4] / K.P_A, K.gamma);
    else {
      const double kk = 0.5 * (r[1] * r[1] + r[2] * r[2] + r[3] * r[3]) / rho;
      P = (K.gamma - 1.0) * (r[4] - kk - rho * phi);
    }
    const double T = P / (rho * K.R);
    const double u2 = r[1] * r[1] + r[2] * r[2] + r[3] * r[3];
    const double ke = (K.set == 0) ? 0.5 * rho * u2 : 0.5 * u2 / rho;
    double wv;
    if (!sphere) {
      wv = (K.set == 0) ? fabs(r[3]) : fabs(r[3] / rho);
    } else {
      const double x = xg[g * 3], y = xg[g * 3 + 1], z = xg[g * 3 + 2];
      const double nr = sqrt(x * x + y * y + z * z);
      const double s = (K.set == 0) ? 1.0 : rho;
      wv = fabs((r[1] / s) * (x / nr) + (r[2] / s) * (y / nr) + (r[3] / s) * (z / nr));
    }
    v[0] += m * rho;
    v[1] += m * rho * c_v * T;
    v[2] += m * ke;
    v[3] += m * rho * phi;
    v[4] += m * r[4];
    v[5] = fmax(v[5], wv);
  }
  for (int64_t c = blockIdx.x * (int64_t)DIAG_T + threadIdx.x; c < ncol; c += (int64_t)DIAG_BLOCKS * DIAG_T) {
    const int64_t g = col_gid[c * n_z];
    const double* r = q + g * 5;
    double P;
    if (K.set == 0) P = K.P_A * hv::pow_pos(r[0] * K.R * r[4] / K.P_A, K.gamma);
    else if (K.set == 1) P = K.P_A * hv::pow_pos(K.R * r[4] / K.P_A, K.gamma);
    else {
      const double kk = 0.5 * (r[1] * r[1] + r[2] * r[2] + r[3] * r[3]) / r[0];
      P = (K.gamma - 1.0) * (r[4] - kk - r[0] * Phi[g]);
    }
    v[6] = fmin(v[6], P);
  }
  block_reduce(v, sh);
  if (threadIdx.x == 0)
#pragma unroll
    for (int k = 0; k < DIAG_NP; ++k) part[k * DIAG_BLOCKS + blockIdx.x] = v[k];
}

__global__ void __launch_bounds__(DIAG_T) diag_final_kernel(const double* __restrict__ part, int set,
                                                            double* __restrict__ out) {
  __shared__ double sh[DIAG_NP * DIAG_T];
  double v[DIAG_NP] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, INFINITY};
  for (int b = threadIdx.x; b < DIAG_BLOCKS; b += DIAG_T) {
#pragma unroll
    for (int k = 0; k < 5; ++k) v[k] += part[k * DIAG_BLOCKS + b];
    v[5] = fmax(v[5], part[5 * DIAG_BLOCKS + b]);
    v[6] = fmin(v[6], part[6 * DIAG_BLOCKS + b]);
  }
  block_reduce(v, sh);
  if (threadIdx.x == 0) {
    // mass, energy_internal, energy_kinetic, energy_potential, energy_total, p_surface_min, w_vertical_max
    double e_int = v[1], e_tot;
    if (set == 2) {
      e_tot = v[4];
      e_int = e_tot - v[2] - v[3];
    } else {
      e_tot = e_int + v[2] + v[3];
    }
    out[0] = v[0];
    out[1] = e_int;
    out[2] = v[2];
    out[3] = v[3];
    out[4] = e_tot;
    out[5] = v[6];
    out[6] = v[5];
  }
}

}  // namespace

extern "C" int hv_euler_diagnostics(int set_id, double P_A, double R, double gamma, double c_v, int sphere,
                                    int64_t ng, const double* d_q, const double* d_M, const double* d_Phi_g,
                                    const double* d_xg, int64_t ncol, int n_z, const int32_t* d_col_gid,
                                    double* d_work, double* d_out, void* stream) {
  if (set_id < 0 || set_id > 2 || ng <= 0 || ncol <= 0 || n_z <= 0 || !d_q || !d_M || !d_Phi_g || !d_col_gid ||
      !d_work || !d_out || (sphere && !d_xg))
    HV_FAIL(HV_ERR_INVALID, "hv_euler_diagnostics: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  EulerConsts K{P_A, R, gamma, 0.0, set_id, 0, 0};
  diag_partial_kernel<<<DIAG_BLOCKS, DIAG_T, 0, st>>>(K, c_v, sphere, ng, d_q, d_M, d_Phi_g, d_xg, ncol, n_z,
                                                      d_col_gid, d_work);
  HV_LAUNCH_CHECK();
  diag_final_kernel<<<1, DIAG_T, 0, st>>>(d_work, set_id, d_out);
  HV_LAUNCH_CHECK();
  return HV_OK;
}

extern "C" int hv_euler_rhs_tiles(const hv_lap_plan* P, const int32_t* d_elem, const double* d_w3, int set_id,
                                  int dirs, int coriolis, double P_A, double R, double gamma, double omega,
                                  const double* d_M, const double* d_q, int64_t ldq, double* d_out, int64_t ldo,
                                  int accumulate, void* stream) {
  if (!P || !P->d_gt || !P->d_Mt || !P->d_part || !d_elem || !d_w3 || P->TX != 1 || P->TY != 1 || set_id < 0 ||
      set_id > 2 || dirs <= 0 || dirs > 7 || !d_q || !d_out || ldq < 5 || ldo < 5 || !d_M || P->N < 1 || P->N > 7)
    HV_FAIL(HV_ERR_INVALID, "hv_euler_rhs_tiles: needs a single-column tile plan and valid arguments");
  cudaStream_t st = (cudaStream_t)stream;
  EulerConsts K{P_A, R, gamma, omega, set_id, dirs, coriolis};
  hv::TileArgs A{};
  A.TX = 1; A.TY = 1; A.nlay = P->nlay; A.n_z = P->n_z;
  A.ntiles = P->ntiles; A.nslot = P->nslot; A.tile0 = 0; A.tile1 = P->ntiles;
  A.gt = P->d_gt; A.code = P->d_code; A.tmeta = P->d_tmeta;
  A.slot_col = P->d_slot_col; A.slot_row0 = P->d_slot_row0; A.slot_nc = P->d_slot_nc; A.col_gid = P->d_col_gid;
  A.Mt = P->d_Mt; A.Minv = P->d_Minv; A.Ms = P->d_Ms; A.q = d_q; A.ldq = ldq; A.ldo = ldo;
  for (int f = 0; f < 5; ++f) A.of.f[f] = f;
  A.zero_mask = 0; A.accumulate = accumulate; A.scale = 1.0; A.out = d_out; A.part = P->d_part;
  int rc;
#define HV_ET(NN_) \
  case NN_: rc = run_tile<NN_>(P->D, K, P->nelem, P->d_gid, d_w3, d_M, d_q, ldq, A, d_elem, st); break;
  switch (P->N + 1) {
    HV_ET(2) HV_ET(3) HV_ET(4) HV_ET(5) HV_ET(6) HV_ET(7) HV_ET(8)
    default: HV_FAIL(HV_ERR_UNSUPPORTED, "hv_euler_rhs_tiles: N=%d", P->N);
  }
#undef HV_ET
  if (rc) return rc;
  return hv::slot_fixup(A, 5, st);   // shared side-face nodes: fixed-order sums of the partial rows
}

// ---------------------------------------------------------------- slab Euler RHS (parallel.py)
namespace {

// out[g, f] (+)= Minv[g] * raw[g, f]: the division by the global mass after the slab-face sums of
// the raw DSS rows were completed across ranks (euler.py:101-103 with the DSS split over slabs);
// explicit __dmul_rn / __dadd_rn: the same rounding as the single-GPU DSS kernel's Minv * sum
// followed by the accumulate
__global__ void rows_minv_kernel(double* __restrict__ out, int64_t ldo, const double* __restrict__ raw,
                                 int64_t ldr, const double* __restrict__ Minv, int64_t ng, int nf, int accumulate) {
  const int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (id >= ng * nf) return;
  const int64_t g = id / nf;
  const int f = (int)(id - g * nf);
  const double v = __dmul_rn(__ldg(Minv + g), __ldg(raw + g * ldr + f));
  out[g * ldo + f] = accumulate ? __dadd_rn(out[g * ldo + f], v) : v;
}

}  // namespace

extern "C" int hv_rows_minv(double* d_out, int64_t ldo, const double* d_raw, int64_t ldr, const double* d_Minv,
                            int64_t ng, int nf, int accumulate, void* stream) {
  if (!d_out || !d_raw || !d_Minv || ng < 0 || nf < 1 || ldo < nf || ldr < nf)
    HV_FAIL(HV_ERR_INVALID, "hv_rows_minv: bad arguments");
  if (ng == 0) return HV_OK;
  const int64_t tot = ng * nf;
  rows_minv_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, (cudaStream_t)stream>>>(d_out, ldo, d_raw, ldr, d_Minv, ng,
                                                                                     nf, accumulate);
  HV_LAUNCH_CHECK();
  return HV_OK;
}
