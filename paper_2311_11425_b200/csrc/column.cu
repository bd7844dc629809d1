// LHEVI column systems on the device.
//
// hv_column_jacobian  band batch of I - lam dV/dq (EulerOps.column_jacobian /
//                     _col_dacc, euler.py:274-417): one CTA per column walks its
//                     layers bottom to top; the layer's node data go to shared
//                     memory, then every thread adds its block entries
//                     (-lam dacc / Mrow) into the LAPACK band (ncol, 2kl+ku+1, M).
//                     Layers run in order, so the node shared by two layers
//                     accumulates exactly as the reference's loop does.
// hv_band_lu_factor   batched band LU with partial pivoting (linalg.py:112-163):
//                     one warp per system, a sliding window of band columns in
//                     shared memory (kl+ku+1 live columns + a chunk being
//                     retired), chunked coalesced row loads / stores.  Same
//                     elementary operations as the reference (multiplier =
//                     a / pivot; update = a - (m * u), no FMA contraction), so
//                     the pivots and factors follow the reference bit for bit
//                     for a bitwise-equal input band.
// hv_band_solve       forward (pivot swaps + L) and backward (U) substitution
//                     (linalg.py:166-194), one warp per system.
#include <cuda_runtime.h>

#include <cstdlib>

#include <cmath>

#include "hv_common.h"
#include "hv_pow.cuh"
#include "lap_common.cuh"

namespace {

struct ColConsts {
  double P_A, R, gamma, lam;
  int set;  // 0 = 2NC, 1 = 2C, 2 = 3C
};

// per layer node data in shared memory
template <int n>
struct LayerNodes {
  double q[5][n], J[n], z[3][n], mask[n], phi[n], P[n], dP[5][n], mass[n];
  double dphi[n], dPz[n], dfld[3][n], dth[n];   // Dz contractions along the layer
};

template <int n>
__global__ void __launch_bounds__(256) column_jacobian_kernel(hv::DTab<n> Dt, hv::DTab<n> Wz, ColConsts K,
                                                              int nlay, int n_z, const int32_t* __restrict__ col_gid,
                                                              const double* __restrict__ qcol,
                                                              const double* __restrict__ Jg,
                                                              const double* __restrict__ gz,
                                                              const double* __restrict__ mask_g,
                                                              const double* __restrict__ Phi_g,
                                                              double* __restrict__ band) {
  constexpr int N = n - 1;
  constexpr int NV = 5;
  constexpr int KL = NV * n - 1, KU = KL, D0 = KL + KU, R = 2 * KL + KU + 1;
  __shared__ LayerNodes<n> L;
  // band columns of the current layer, [R][TW]: the layer's block entries accumulate here (no global
  // read-modify-write); after the layer its first TW - NV columns are final and leave with coalesced
  // row segments, the last NV (the node shared with the next layer) move to the front
  constexpr int TW = NV * n;
  __shared__ double T[R][TW];
  const int64_t c = blockIdx.x;
  const int t = threadIdx.x;
  const int64_t M = (int64_t)NV * n_z;
  double* bc = band + c * R * M;
  // D and the zeta weights in shared memory: the entry loop indexes them with thread-varying
  // (i, a) (constant-bank loads would serialise across the warp)
  __shared__ double sDm[n][n], sw[n];
  for (int x = t; x < n * n; x += blockDim.x) sDm[x / n][x % n] = Dt.D[x / n][x % n];
  if (t < n) sw[t] = Wz.D[0][t];
  const double* w = sw;
  for (int e = t; e < R * TW; e += blockDim.x) T[e / TW][e % TW] = (e / TW == D0) ? 1.0 : 0.0;   // band = I
  __syncthreads();
  const int32_t* cg = col_gid + c * (int64_t)n_z;
  const double* qc = qcol + c * (int64_t)n_z * NV;
  // node data of the whole column, once, by n_z threads (not n threads per layer): state, J, grad
  // zeta, mask, Phi, P, dP/dq (state.py:104-125) and the column mass DSS(w_z J) (euler.py:76-78:
  // at a node shared by two layers the lower layer's top weight first)
  extern __shared__ double colsm[];
  double* cq = colsm;                    // [5][n_z]
  double* cJ = cq + NV * n_z;
  double* cz = cJ + n_z;                 // [3][n_z]
  double* cmask = cz + 3 * n_z;
  double* cphi = cmask + n_z;
  double* cP = cphi + n_z;
  double* cdP = cP + n_z;                // [5][n_z]
  double* cmass = cdP + NV * n_z;
  double* cder = cmass + n_z;            // [6][nlay * n]: Dz of Phi, P, U, V, W, Theta per layer node
  for (int z = t; z < n_z; z += blockDim.x) {
    const int g = cg[z];
    double qv[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) cq[v * n_z + z] = qv[v] = qc[(int64_t)z * NV + v];
    const double J = Jg[g];
    cJ[z] = J;
#pragma unroll
    for (int d = 0; d < 3; ++d) cz[d * n_z + z] = gz[(int64_t)g * 3 + d];
    cmask[z] = mask_g[g];
    const double phi = Phi_g[g];
    cphi[z] = phi;
    double m = 0.0;
    const int i = (z == n_z - 1) ? N : z % N;
    if (i == 0 && z > 0) m = m + w[N] * J;
    m = m + w[i] * J;
    cmass[z] = m;
    const double rho = qv[0];
    double P;
    if (K.set == 0) P = K.P_A * hv::pow_pos(rho * K.R * qv[4] / K.P_A, K.gamma);
    else if (K.set == 1) P = K.P_A * hv::pow_pos(K.R * qv[4] / K.P_A, K.gamma);
    else {
      const double ke = 0.5 * (qv[1] * qv[1] + qv[2] * qv[2] + qv[3] * qv[3]) / rho;
      P = (K.gamma - 1.0) * (qv[4] - ke - rho * phi);
    }
    cP[z] = P;
    double dp[NV];
    if (K.set == 0) {
      dp[0] = K.gamma * P / rho;
      dp[1] = dp[2] = dp[3] = 0.0;
      dp[4] = K.gamma * P / qv[4];
    } else if (K.set == 1) {
      dp[0] = dp[1] = dp[2] = dp[3] = 0.0;
      dp[4] = K.gamma * P / qv[4];
    } else {
      const double g1 = K.gamma - 1.0;
      const double ke2 = qv[1] * qv[1] + qv[2] * qv[2] + qv[3] * qv[3];
      dp[0] = g1 * (0.5 * ke2 / (rho * rho) - phi);
      dp[1] = -g1 * qv[1] / rho;
      dp[2] = -g1 * qv[2] / rho;
      dp[3] = -g1 * qv[3] / rho;
      dp[4] = g1;
    }
#pragma unroll
    for (int v = 0; v < NV; ++v) cdP[v * n_z + z] = dp[v];
  }
  __syncthreads();
  for (int x = t; x < nlay * n; x += blockDim.x) {   // strong zeta derivatives along each layer
    const int l = x / n, i = x % n, z0 = l * N;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0, a4 = 0.0, a5 = 0.0;
#pragma unroll
    for (int a = 0; a < n; ++a) {
      const double d = sDm[i][a];
      a0 += d * cphi[z0 + a];
      a1 += d * cP[z0 + a];
      a2 += d * cq[1 * n_z + z0 + a];
      a3 += d * cq[2 * n_z + z0 + a];
      a4 += d * cq[3 * n_z + z0 + a];
      a5 += d * cq[4 * n_z + z0 + a];
    }
    const int nl = nlay * n;
    cder[0 * nl + x] = a0;
    cder[1 * nl + x] = a1;
    cder[2 * nl + x] = a2;
    cder[3 * nl + x] = a3;
    cder[4 * nl + x] = a4;
    cder[5 * nl + x] = a5;
  }
  __syncthreads();
  for (int l = 0; l < nlay; ++l) {
    // this layer's node view (parallel copy of the column arrays)
    const int z0 = l * N, nl = nlay * n;
    for (int x = t; x < 24 * n; x += blockDim.x) {
      const int f = x / n, i = x % n, z = z0 + i, li = l * n + i;
      double v;
      if (f < 5) v = cq[f * n_z + z];
      else if (f == 5) v = cJ[z];
      else if (f < 9) v = cz[(f - 6) * n_z + z];
      else if (f == 9) v = cmask[z];
      else if (f == 10) v = cphi[z];
      else if (f == 11) v = cP[z];
      else if (f < 17) v = cdP[(f - 12) * n_z + z];
      else if (f == 17) v = cmass[z];
      else v = cder[(f - 18) * nl + li];
      (&L.q[0][0])[f * n + i] = v;   // LayerNodes is 24 consecutive [n] arrays in this order
    }
    __syncthreads();
    // block entries (i, vi, a, va)
    for (int e = t; e < NV * n * NV * n; e += blockDim.x) {
      const int va = e % NV, a = (e / NV) % n, vi = (e / (NV * n)) % NV, i = e / (NV * n * NV);
      const double rho_i = L.q[0][i], rho_a = L.q[0][a];
      const double wj_i = w[i] * L.J[i];
      double B = 0.0;
      if (K.set == 0) {
        const double uz_i = L.mask[i] * (L.q[1][i] * L.z[0][i] + L.q[2][i] * L.z[1][i] + L.q[3][i] * L.z[2][i]);
        const double uz_a = L.mask[a] * (L.q[1][a] * L.z[0][a] + L.q[2][a] * L.z[1][a] + L.q[3][a] * L.z[2][a]);
        if (vi == 0) {
          if (va == 0) B = (w[a] * sDm[a][i]) * (L.J[a] * uz_a);
          else if (va <= 3) B = (w[a] * sDm[a][i]) * (L.J[a] * (L.mask[a] * rho_a * L.z[va - 1][a]));
        } else if (vi <= 3) {
          const double zc = L.z[vi - 1][i];
          if (va == 0) {
            const double dg = (i == a) ? (wj_i * (-zc / (rho_i * rho_i)) * L.dPz[i]) : 0.0;
            B = -(dg + ((wj_i * zc / rho_i) * sDm[i][a]) * L.dP[0][a]);
          } else if (va <= 3) {
            const double dg = (i == a) ? (wj_i * L.mask[i] * L.z[va - 1][i] * L.dfld[vi - 1][i]) : 0.0;
            B = (va == vi) ? -(dg + (wj_i * uz_i) * sDm[i][a]) : -dg;
          } else {
            B = -(((wj_i * zc / rho_i) * sDm[i][a]) * L.dP[4][a]);
          }
        } else {
          if (va >= 1 && va <= 3) B = (i == a) ? -(wj_i * L.mask[i] * L.z[va - 1][i] * L.dth[i]) : 0.0;
          else if (va == 4) B = -((wj_i * uz_i) * sDm[i][a]);
        }
      } else {
        const bool three = (K.set == 2);
        const double Uz_a = L.mask[a] * (L.q[1][a] * L.z[0][a] + L.q[2][a] * L.z[1][a] + L.q[3][a] * L.z[2][a]);
        const double uz_a = Uz_a / rho_a;
        const double dUz_a = (va >= 1 && va <= 3) ? L.mask[a] * L.z[va - 1][a] : 0.0;
        if (vi == 0) {
          B = (w[a] * sDm[a][i]) * (L.J[a] * dUz_a);
        } else if (vi == 4) {
          const double T5 = L.q[4][a];
          double dF;
          if (!three) {
            if (va == 0) dF = -T5 * Uz_a / (rho_a * rho_a);
            else if (va <= 3) dF = L.mask[a] * L.z[va - 1][a] * T5 / rho_a;
            else dF = uz_a;
          } else {
            const double EP = T5 + L.P[a];
            if (va == 0) dF = -EP * Uz_a / (rho_a * rho_a) + uz_a * L.dP[0][a];
            else if (va <= 3) dF = L.mask[a] * L.z[va - 1][a] * EP / rho_a + uz_a * L.dP[va][a];
            else dF = uz_a * (1.0 + L.dP[4][a]);
          }
          B = (w[a] * sDm[a][i]) * (L.J[a] * dF);
        } else {
          const int comp = vi;
          const double zc_a = L.z[comp - 1][a];
          const double Uc = L.q[comp][a];
          double df;
          if (va == 0) df = L.J[a] * (-Uc * Uz_a / (rho_a * rho_a) + zc_a * L.dP[0][a]);
          else if (va == 4) df = L.J[a] * zc_a * L.dP[4][a];
          else {
            double d = Uc * dUz_a / rho_a + zc_a * L.dP[va][a];
            if (va == comp) d = d + uz_a;
            df = L.J[a] * d;
          }
          B = -((w[i] * sDm[i][a]) * df);
          if (va == 0 && i == a) B = B + -(wj_i * L.dphi[i] * L.z[comp - 1][i]);
        }
      }
      const double contrib = (-K.lam * B) / L.mass[i];
      const int row = NV * i + vi, col = NV * a + va;   // layer-local: band row D0 + row - col
      T[D0 + row - col][col] = T[D0 + row - col][col] + contrib;
    }
    __syncthreads();
    // columns NV*l*N .. + wout are final: all R band rows, row segments of wout doubles
    const int wout = (l == nlay - 1) ? TW : TW - NV;
    const int64_t c0 = (int64_t)NV * l * N;
    for (int e = t; e < R * wout; e += blockDim.x) {
      const int r = e / wout, k = e - r * wout;
      bc[(int64_t)r * M + c0 + k] = T[r][k];
    }
    __syncthreads();
    if (l < nlay - 1) {
      for (int e = t; e < R * NV; e += blockDim.x) {   // shared node's columns to the front (TW >= 2 NV)
        const int r = e / NV, k = e % NV;
        T[r][k] = T[r][TW - NV + k];
      }
      __syncthreads();
      for (int e = t; e < R * (TW - NV); e += blockDim.x) {   // the next layer's new columns: identity
        const int r = e / (TW - NV), k = NV + e % (TW - NV);
        T[r][k] = (r == D0) ? 1.0 : 0.0;
      }
    }
    __syncthreads();
  }
}

template <int n>
int run_jacobian(const double* hD, const double* hw, const ColConsts& K, int64_t ncol, int nlay, int n_z,
                 const int32_t* col_gid, const double* qcol, const double* Jg, const double* gz, const double* mask,
                 const double* Phi, double* band, cudaStream_t st) {
  hv::DTab<n> Dt, Wz{};
  hv::fill_dtab(Dt, hD);
  for (int i = 0; i < n; ++i) Wz.D[0][i] = hw[i];
  const size_t smem = sizeof(double) * ((size_t)18 * n_z + (size_t)6 * nlay * n);   // column node arrays
  auto kern = column_jacobian_kernel<n>;
  if (smem > 160 * 1024) HV_FAIL(HV_ERR_UNSUPPORTED, "hv_column_jacobian: column too tall (n_z=%d)", n_z);
  HV_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<(unsigned)ncol, 256, smem, st>>>(Dt, Wz, K, nlay, n_z, col_gid, qcol, Jg, gz, mask, Phi, band);
  HV_LAUNCH_CHECK();
  return HV_OK;
}

// ---------------------------------------------------------------- band LU / solve
constexpr int CH = 4;    // LU: columns per retire / load chunk (small window: more systems per SM)
constexpr int CHS = 8;   // solve: columns per streamed chunk

struct BandDims {
  int kl, ku, R, M, WC, RS;   // window columns WC = kl + ku + 1 + CH, padded row stride RS (even)
};

__device__ __forceinline__ double dsub_mul(double a, double m, double u) { return __dsub_rn(a, __dmul_rn(m, u)); }

__global__ void band_lu_kernel(BandDims B, int64_t nb, double* __restrict__ data, int32_t* __restrict__ ipiv,
                               int32_t* __restrict__ info) {
  extern __shared__ double win_all[];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t s = (int64_t)blockIdx.x * (blockDim.x / 32) + warp;
  if (s >= nb) return;
  double* win = win_all + (size_t)warp * B.R * B.RS;
  double* g = data + s * (int64_t)B.R * B.M;
  const int d = B.kl + B.ku;
  auto slot = [&](int col) { return col % B.WC; };
  // chunk transfers: the (row, column) elements of the chunk spread over the lanes, eight
  // independent loads in flight per lane
  auto load_cols = [&](int c0, int c1) {     // columns [c0, c1) -> window
    const int w = c1 - c0, tot = B.R * w;
    for (int e0 = 0; e0 < tot; e0 += 32 * 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + u * 32 + lane;
        v[u] = (e < tot) ? g[(int64_t)(e / w) * B.M + c0 + e % w] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + u * 32 + lane;
        if (e < tot) win[(e / w) * B.RS + slot(c0 + e % w)] = v[u];
      }
    }
  };
  auto store_cols = [&](int c0, int c1) {
    const int w = c1 - c0, tot = B.R * w;
    for (int e = lane; e < tot; e += 32) {
      const int r = e / w, c = e - r * w;
      g[(int64_t)r * B.M + c0 + c] = win[r * B.RS + slot(c0 + c)];
    }
  };
  // the next chunk is prefetched into registers one chunk ahead (R * CH <= 32 * PFN)
  constexpr int PFN = 16;
  double pf[PFN];
  int pf_c0 = 0, pf_w = 0;
  auto prefetch = [&](int c0, int c1) {
    pf_c0 = c0;
    pf_w = c1 - c0;
    const int tot = B.R * pf_w;
#pragma unroll
    for (int u = 0; u < PFN; ++u) {
      const int e = u * 32 + lane;
      const int r = (pf_w == CH) ? e / CH : e / pf_w, c = (pf_w == CH) ? e % CH : e % pf_w;
      pf[u] = (e < tot) ? g[(int64_t)r * B.M + c0 + c] : 0.0;
    }
  };
  auto commit = [&]() {
    const int tot = B.R * pf_w;
#pragma unroll
    for (int u = 0; u < PFN; ++u) {
      const int e = u * 32 + lane;
      const int r = (pf_w == CH) ? e / CH : e / pf_w, c = (pf_w == CH) ? e % CH : e % pf_w;
      if (e < tot) win[r * B.RS + slot(pf_c0 + c)] = pf[u];
    }
  };
  int loaded = min(B.M, B.WC);
  load_cols(0, loaded);
  if (loaded < B.M) prefetch(loaded, min(B.M, loaded + CH));
  int stored = 0;
  __syncwarp();
  for (int j = 0; j < B.M; ++j) {
    const int jmax = min(B.M - 1, j + B.ku + B.kl);
    if (jmax >= loaded) {   // retire finished columns [stored, j), bring in the prefetched chunk
      store_cols(stored, j);
      stored = j;
      __syncwarp();
      commit();
      loaded = pf_c0 + pf_w;
      if (loaded < B.M) prefetch(loaded, min(B.M, loaded + CH));
      __syncwarp();
    }
    const int lm = min(B.kl, B.M - 1 - j);
    const int sj = j % B.WC;                                          // window slot of column j
    auto sl = [&](int col) { const int t = sj + (col - j); return t >= B.WC ? t - B.WC : t; };
    // pivot: first index of the largest |candidate| (np.argmax)
    double best = -1.0;
    int bi = 0;
    for (int r = lane; r <= lm; r += 32) {
      const double v = fabs(win[(d + r) * B.RS + sj]);
      if (v > best) { best = v; bi = r; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    const int prel = bi;
    const double piv = win[(d + prel) * B.RS + sj];
    if (piv == 0.0) {
      if (lane == 0) info[s] = j + 1;
      store_cols(stored, loaded);
      return;
    }
    if (lane == 0) ipiv[s * B.M + j] = j + prel;
    if (prel != 0) {
      for (int col = j + lane; col <= jmax; col += 32) {
        const int off = d + j - col;
        double* a = win + off * B.RS + sl(col);
        double* b = win + (off + prel) * B.RS + sl(col);
        const double tmp = *a;
        *a = *b;
        *b = tmp;
      }
    }
    __syncwarp();
    if (lm > 0) {
      // lanes own the rows below the pivot: multiplier in a register, then the row update
      // in batches of 8 columns (all loads of a batch before its stores)
      const double pv = win[d * B.RS + sj];
      for (int i0 = 0; i0 < lm; i0 += 32) {
        const int i = i0 + lane;
        const bool act = i < lm;
        double m = 0.0;
        if (act) {
          m = win[(d + 1 + i) * B.RS + sj] / pv;
          win[(d + 1 + i) * B.RS + sj] = m;
        }
        for (int c0 = j + 1; c0 <= jmax; c0 += 8) {
          double u[8], a[8];
          int so[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int col = c0 + k;
            const int off = d + j - col;
            const bool ok = act && col <= jmax;
            so[k] = off * B.RS + sl(col);
            u[k] = ok ? win[so[k]] : 0.0;
            a[k] = ok ? win[so[k] + (1 + i) * B.RS] : 0.0;
          }
#pragma unroll
          for (int k = 0; k < 8; ++k)
            if (act && c0 + k <= jmax) win[so[k] + (1 + i) * B.RS] = dsub_mul(a[k], m, u[k]);
        }
      }
      __syncwarp();
    }
  }
  __syncwarp();
  store_cols(stored, B.M);
  if (lane == 0) info[s] = 0;
}

// Block-per-system band LU (default): the same sliding window and elementary operations as
// band_lu_kernel (bitwise the same factors), with NT threads per system instead of one warp, so
// the per-column critical path (pivot, swap, multipliers, rank-1 update) is spread out:
// thread t updates window column j + 1 + (t % CW) for the rows i = t / CW, t / CW + G, ...
// (CW = kl + ku update columns, G = NT / CW row groups); every warp finds the pivot redundantly
// (read-only).  Two CTA barriers per column: (1) the row swap of columns j+1..jmax and the
// multipliers of column j (computed from the pre-swap column into a side buffer, so the slower
// warps' pivot search is never disturbed) run together; (2) the rank-1 update, while the
// multiplier threads write column j's final values (pivot, multipliers) into the window.  RS is
// even here: the column-walking update and swap (stride RS - 1, odd) hit distinct banks.
template <int PFN>
__global__ void __launch_bounds__(128) band_lu_block_kernel(BandDims B, int64_t nb, double* __restrict__ data,
                                                           int32_t* __restrict__ ipiv, int32_t* __restrict__ info) {
  extern __shared__ double win[];
  double* mb = win + (size_t)B.R * B.RS;   // [kl] multipliers of the current column
  const int t = threadIdx.x, NT = blockDim.x, lane = t % 32;
  const int64_t s = blockIdx.x;
  if (s >= nb) return;
  double* g = data + s * (int64_t)B.R * B.M;
  const int d = B.kl + B.ku;
  // phase-2 mapping: column j+1 by warp 0 (one row per lane; look-ahead pivot search right after),
  // columns j+2..jmax by (column, row group) threads
  const int CB = max(1, d - 1), G = max(1, NT / CB);
  const int tc = t % CB, tr = t / CB;
  int* s_prel = reinterpret_cast<int*>(mb + B.kl + 1);   // pivot row (relative) of the next column
  // first index of the largest |candidate| of column `col` (window slot sc), rows 0..lm; warp 0
  auto find_pivot = [&](int sc, int lm_) {
    double best = -1.0;
    int bi = 0;
    for (int r = lane; r <= lm_; r += 32) {
      const double v = fabs(win[(d + r) * B.RS + sc]);
      if (v > best) { best = v; bi = r; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    if (lane == 0) *s_prel = bi;
  };
  // window slot of column c0 + c for c < WC, given s0 = slot(c0) (no integer division in the loops)
  auto wrap = [&](int q) { return q >= B.WC ? q - B.WC : q; };
  auto load_cols = [&](int c0, int c1) {   // once, c0 = 0: slots = columns
    const int w = c1 - c0, tot = B.R * w;
    for (int e = t; e < tot; e += NT) {
      const int r = e / w, c = e - r * w;
      win[r * B.RS + c0 + c] = g[(int64_t)r * B.M + c0 + c];
    }
  };
  auto store_cols = [&](int c0, int c1) {   // w = c1 - c0 <= WC columns
    const int w = c1 - c0, tot = B.R * w;
    const int s0 = c0 % B.WC;
    if (w == CH) {
      for (int e = t; e < tot; e += NT) {
        const int r = e / CH, c = e % CH;
        g[(int64_t)r * B.M + c0 + c] = win[r * B.RS + wrap(s0 + c)];
      }
    } else {
      for (int e = t; e < tot; e += NT) {
        const int r = e / w, c = e - r * w;
        g[(int64_t)r * B.M + c0 + c] = win[r * B.RS + wrap(s0 + c)];
      }
    }
  };
  // the next chunk is prefetched into registers (R * CH <= NT * PFN, checked by the launcher)
  double pf[PFN];
  int pf_c0 = 0, pf_w = 0;
  auto prefetch = [&](int c0, int c1) {
    pf_c0 = c0;
    pf_w = c1 - c0;
    const int tot = B.R * pf_w;
#pragma unroll
    for (int u = 0; u < PFN; ++u) {
      const int e = u * NT + t;
      const int r = (pf_w == CH) ? e / CH : e / pf_w, c = (pf_w == CH) ? e % CH : e % pf_w;
      pf[u] = (e < tot) ? g[(int64_t)r * B.M + c0 + c] : 0.0;
    }
  };
  auto commit = [&]() {
    const int tot = B.R * pf_w;
    const int s0 = pf_c0 % B.WC;
#pragma unroll
    for (int u = 0; u < PFN; ++u) {
      const int e = u * NT + t;
      const int r = (pf_w == CH) ? e / CH : e / pf_w, c = (pf_w == CH) ? e % CH : e % pf_w;
      if (e < tot) win[r * B.RS + wrap(s0 + c)] = pf[u];
    }
  };
  int loaded = min(B.M, B.WC);
  load_cols(0, loaded);
  if (loaded < B.M) prefetch(loaded, min(B.M, loaded + CH));
  int stored = 0;
  int sj = 0;                    // window slot of column j (j % WC, kept incrementally)
  __syncthreads();
  if (t < 32) find_pivot(0, min(B.kl, B.M - 1));
  __syncthreads();
  for (int j = 0; j < B.M; ++j, sj = wrap(sj + 1)) {
    const int jmax = min(B.M - 1, j + B.ku + B.kl);
    if (jmax >= loaded) {   // retire finished columns [stored, j), bring in the prefetched chunk
      store_cols(stored, j);
      stored = j;
      __syncthreads();
      commit();
      loaded = pf_c0 + pf_w;
      if (loaded < B.M) prefetch(loaded, min(B.M, loaded + CH));
      __syncthreads();
    }
    const int lm = min(B.kl, B.M - 1 - j);
    auto sl = [&](int col) { return wrap(sj + (col - j)); };
    const int prel = *s_prel;    // found during the previous column's update (look-ahead)
    const double piv = win[(d + prel) * B.RS + sj];
    if (piv == 0.0) {
      if (t == 0) info[s] = j + 1;
      __syncthreads();
      store_cols(stored, loaded);
      return;
    }
    if (t == 0) ipiv[s * B.M + j] = j + prel;
    const int ncol = jmax - j;   // update columns j + 1 .. jmax
    // phase 1: row swap in columns j+1..jmax (threads from the top), multipliers of column j
    // from its pre-swap values (threads from the bottom) -- disjoint data
    double mcol = 0.0;           // this thread's final column-j value (written in phase 2)
    if (prel != 0)
      for (int c = 1 + t; c <= ncol; c += NT) {
        const int col = j + c, off = d + j - col;
        double* x = win + off * B.RS + sl(col);
        double* y = x + prel * B.RS;
        const double tmp = *x;
        *x = *y;
        *y = tmp;
      }
    const int tm = NT - 1 - t;   // multiplier / column-j thread: tm < lm (row j+1+tm), tm == lm (pivot row)
    if (tm < lm) {
      // after the swap, row j + 1 + tm holds the old row j value if j + 1 + tm == j + prel
      const double v = (tm + 1 == prel) ? win[d * B.RS + sj] : win[(d + 1 + tm) * B.RS + sj];
      mcol = v / piv;
      mb[tm] = mcol;
    }
    __syncthreads();
    // phase 2: rank-1 update of columns j+1..jmax; column j gets its pivot and multipliers
    if (tm < lm) win[(d + 1 + tm) * B.RS + sj] = mcol;
    else if (tm == lm) win[d * B.RS + sj] = piv;
    if (t < 32 && ncol >= 1) {   // column j+1 first, then its pivot (the next step's critical path)
      const int so = (d - 1) * B.RS + sl(j + 1);
      const double u = win[so];
      for (int i = lane; i < lm; i += 32) {
        double* ap = win + so + (1 + i) * B.RS;
        *ap = dsub_mul(*ap, mb[i], u);
      }
      __syncwarp();
      find_pivot(sl(j + 1), min(B.kl, B.M - 2 - j));
    }
    if (tr < G && 1 + tc < ncol) {
      const int col = j + 2 + tc;
      const int so = (d + j - col) * B.RS + sl(col);
      const double u = win[so];
      // rows in batches of four: loads of a batch before its stores
      for (int i0 = tr; i0 < lm; i0 += 4 * G) {
        double a[4], m[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int i = i0 + k * G;
          a[k] = (i < lm) ? win[so + (1 + i) * B.RS] : 0.0;
          m[k] = (i < lm) ? mb[i] : 0.0;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int i = i0 + k * G;
          if (i < lm) win[so + (1 + i) * B.RS] = dsub_mul(a[k], m[k], u);
        }
      }
    }
    __syncthreads();
  }
  store_cols(stored, B.M);
  if (t == 0) info[s] = 0;
}

// rows [r0, r0 + nr) x columns [c0, c0 + w) of a band into ch[col][RS] (column-major in shared
// memory: the lanes of the substitution steps walk rows); eight global loads in flight
__device__ __forceinline__ void load_chunk(double* ch, int RS, const double* g, int r0, int nr, int c0, int w, int M,
                                           int lane) {
  const int tot = nr * w;
  for (int e0 = 0; e0 < tot; e0 += 32 * 8) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * 32 + lane;
      v[u] = (e < tot) ? g[(int64_t)(r0 + e / w) * M + c0 + e % w] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * 32 + lane;
      if (e < tot) ch[(e % w) * RS + e / w] = v[u];
    }
  }
}

// Solve with the factors streamed through shared memory in CHS-column chunks (row segments of
// a chunk are contiguous in the band layout: coalesced).  Forward: pivot swap + L column
// (reference order, a - (l * x) without contraction).  Backward in column order: x_i /= U_ii,
// then the column's U entries update the rows above (same operations as the reference's row
// sums, different summation order: within the fp64 bar, not bitwise).
__global__ void band_solve_kernel(BandDims B, int64_t nb, const double* __restrict__ data,
                                  const int32_t* __restrict__ ipiv, double* __restrict__ x) {
  extern __shared__ double xs_all[];
  const int wpb = blockDim.x / 32;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t s = (int64_t)blockIdx.x * wpb + warp;
  const int d = B.kl + B.ku;
  const int RW = d + 1;                          // chunk rows: U part 0..d (forward uses d+1..d+kl)
  const int RL = B.kl;
  const int CRS = RW | 1;                        // odd column stride of the chunk buffer
  double* xs = xs_all + (size_t)warp * (B.M + CRS * CHS);
  double* ch = xs + B.M;                         // [col][CRS]
  if (s >= nb) return;
  const double* g = data + s * (int64_t)B.R * B.M;
  double* xg = x + s * (int64_t)B.M;
  for (int i = lane; i < B.M; i += 32) xs[i] = xg[i];
  const int32_t* ip = ipiv + s * (int64_t)B.M;
  __syncwarp();
  // forward: L rows d+1 .. d+kl of each chunk
  for (int c0 = 0; c0 < B.M - 1; c0 += CHS) {
    const int w = min(CHS, B.M - 1 - c0);
    load_chunk(ch, CRS, g, d + 1, RL, c0, w, B.M, lane);
    const int pl = (lane < w) ? ip[c0 + lane] : 0;   // the chunk's pivots, one per lane
    __syncwarp();
    for (int jj = 0; jj < w; ++jj) {
      const int j = c0 + jj;
      const int p = __shfl_sync(0xffffffffu, pl, jj);
      if (p != j && lane == 0) {
        const double tmp = xs[j];
        xs[j] = xs[p];
        xs[p] = tmp;
      }
      __syncwarp();
      const int lm = min(B.kl, B.M - 1 - j);
      const double xj = xs[j];
      for (int i = lane; i < lm; i += 32) xs[j + 1 + i] = dsub_mul(xs[j + 1 + i], ch[jj * CRS + i], xj);
      __syncwarp();
    }
  }
  // backward, column by column from the last: rows 0 .. d of each chunk (d = diagonal)
  for (int c1 = B.M; c1 > 0; c1 -= CHS) {
    const int c0 = max(0, c1 - CHS), w = c1 - c0;
    load_chunk(ch, CRS, g, 0, RW, c0, w, B.M, lane);
    __syncwarp();
    for (int jj = w - 1; jj >= 0; --jj) {
      const int i = c0 + jj;
      if (lane == 0) xs[i] = xs[i] / ch[jj * CRS + d];
      __syncwarp();
      const double xi = xs[i];
      const int nr = min(d, i);                  // rows i-1 .. i-nr hold this column's U entries
      for (int r = lane; r < nr; r += 32) xs[i - 1 - r] = dsub_mul(xs[i - 1 - r], ch[jj * CRS + d - 1 - r], xi);
      __syncwarp();
    }
  }
  for (int i = lane; i < B.M; i += 32) xg[i] = xs[i];
}

BandDims band_dims(int kl, int ku, int M) {
  BandDims B;
  B.kl = kl;
  B.ku = ku;
  B.R = 2 * kl + ku + 1;
  B.M = M;
  B.WC = kl + ku + 1 + CH;
  // row stride = 3 (mod 4): odd, so the row-update lanes (one row each) hit distinct banks,
  // and RS - 1 = 2 (mod 4), so the column-walking swaps (stride 1 - RS) are at most 2-way
  B.RS = B.WC;
  while ((B.RS & 3) != 3) ++B.RS;
  return B;
}

}  // namespace

extern "C" int hv_column_jacobian(int N, const double* h_D, const double* h_w, int set_id, double P_A, double R,
                                  double gamma, double lam, int64_t ncol, int nlay, int n_z,
                                  const int32_t* d_col_gid, const double* d_qcol, const double* d_Jg,
                                  const double* d_gz, const double* d_mask_g, const double* d_Phi_g, double* d_band,
                                  void* stream) {
  if (N < 1 || N > 7 || !h_D || !h_w || set_id < 0 || set_id > 2 || ncol <= 0 || nlay <= 0 || n_z != nlay * N + 1 ||
      !d_col_gid || !d_qcol || !d_Jg || !d_gz || !d_mask_g || !d_Phi_g || !d_band)
    HV_FAIL(HV_ERR_INVALID, "hv_column_jacobian: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  ColConsts K{P_A, R, gamma, lam, set_id};
#define HV_JAC(NN_) \
  case NN_: return run_jacobian<NN_>(h_D, h_w, K, ncol, nlay, n_z, d_col_gid, d_qcol, d_Jg, d_gz, d_mask_g, d_Phi_g, d_band, st);
  switch (N + 1) {
    HV_JAC(2) HV_JAC(3) HV_JAC(4) HV_JAC(5) HV_JAC(6) HV_JAC(7) HV_JAC(8)
  }
#undef HV_JAC
  HV_FAIL(HV_ERR_UNSUPPORTED, "hv_column_jacobian: N=%d", N);
}

extern "C" int hv_band_lu_factor(double* d_data, int64_t nb, int kl, int ku, int M, int32_t* d_ipiv, int32_t* d_info,
                                 void* stream) {
  if (!d_data || !d_ipiv || !d_info || nb <= 0 || kl < 0 || ku < 0 || M <= 0)
    HV_FAIL(HV_ERR_INVALID, "hv_band_lu_factor: bad arguments");
  const char* lv = getenv("HV_BAND_LU");
  if (!(lv && atoi(lv) == 1)) {   // block per system (default); HV_BAND_LU=1: the warp-per-system kernel
    BandDims B = band_dims(kl, ku, M);
    B.RS = B.WC + (B.WC & 1);      // even: stride RS - 1 of the column walks is odd
    const int d = kl + ku, CB = d > 1 ? d - 1 : 1;
    const int G = CB >= 128 ? 1 : 128 / CB;
    const int NT = ((CB * G + 31) / 32) * 32;
    const size_t smem = sizeof(double) * ((size_t)B.R * B.RS + kl + 2);
    if (smem > 227 * 1024 || B.R * CH > NT * 8 || NT > 128 || NT < kl + 1)
      HV_FAIL(HV_ERR_UNSUPPORTED, "hv_band_lu_factor: band too wide (kl=%d ku=%d)", kl, ku);
    auto kern = (B.R * CH <= NT * 4) ? band_lu_block_kernel<4> : band_lu_block_kernel<8>;
    HV_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<(unsigned)nb, NT, smem, (cudaStream_t)stream>>>(B, nb, d_data, d_ipiv, d_info);
    HV_LAUNCH_CHECK();
    return HV_OK;
  }
  const BandDims B = band_dims(kl, ku, M);
  // one warp (system) per block: the SM packs as many ~35 KB windows as fit (6 at N = 4)
  const int wpb = 1;
  const size_t smem = sizeof(double) * (size_t)wpb * B.R * B.RS;
  if (smem > 227 * 1024 || B.R * CH > 32 * 16)
    HV_FAIL(HV_ERR_UNSUPPORTED, "hv_band_lu_factor: band too wide (kl=%d ku=%d)", kl, ku);
  HV_CUDA_CHECK(cudaFuncSetAttribute(band_lu_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  band_lu_kernel<<<(unsigned)((nb + wpb - 1) / wpb), 32 * wpb, smem, (cudaStream_t)stream>>>(B, nb, d_data, d_ipiv,
                                                                                              d_info);
  HV_LAUNCH_CHECK();
  return HV_OK;
}

extern "C" int hv_band_solve(const double* d_data, const int32_t* d_ipiv, int64_t nb, int kl, int ku, int M,
                             double* d_x, void* stream) {
  if (!d_data || !d_ipiv || !d_x || nb <= 0 || kl < 0 || ku < 0 || M <= 0)
    HV_FAIL(HV_ERR_INVALID, "hv_band_solve: bad arguments");
  const BandDims B = band_dims(kl, ku, M);
  const int wpb = 4;
  const size_t smem = sizeof(double) * (size_t)wpb * (M + ((kl + ku + 1) | 1) * CHS);
  if (smem > 200 * 1024) HV_FAIL(HV_ERR_UNSUPPORTED, "hv_band_solve: system too large (M=%d)", M);
  HV_CUDA_CHECK(cudaFuncSetAttribute(band_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  band_solve_kernel<<<(unsigned)((nb + wpb - 1) / wpb), 32 * wpb, smem, (cudaStream_t)stream>>>(B, nb, d_data, d_ipiv,
                                                                                                d_x);
  HV_LAUNCH_CHECK();
  return HV_OK;
}
