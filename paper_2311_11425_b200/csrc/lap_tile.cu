// Hot path v2: tile-sweep Laplacian with on-chip DSS (sm_100a, fp64).
//
// laplacian_apply (hyperdiff.py:84-94) for F fields at once.  One CTA owns a
// TX x TY patch of element columns (tiles.py) and sweeps it bottom to top:
//
//   G  gather the tile-layer nodes of q once into shared memory (shared
//      faces stored once), through the per-tile gid table;
//   S1 strong xi / eta derivatives: one thread per (element, line, field),
//      register-resident line, results transposed through shared memory;
//   P  per (element, k-line, field): zeta derivative in registers, flux
//      f_m = W_mn dq_n with the packed metric W = w3 Jg G_nu (6 components,
//      read once per node and broadcast to the F field lanes), zeta weak
//      derivative in registers;
//   W1 weak xi / eta derivatives in place (transposed lines);
//   A  element accumulator = sum of the three weak parts; the top face is
//      carried in a register into the next layer (vertical DSS, no memory);
//      the horizontal DSS inside the tile is a 4-colour in-place summation
//      in shared memory (elements of one colour share no node);
//   O  nodes owned by the tile alone are final: y = scale * Minv * acc is
//      written straight to the output; perimeter nodes shared with other
//      tiles go to their partial row, summed in fixed order by
//      lap_tile_fixup (deterministic, atomics-free).
//
// No atomics anywhere; every sum is in a fixed order, so results are
// bitwise reproducible run to run.
#include <cuda_runtime.h>

#include "hv_common.h"
#include "lap_common.cuh"
#include "lap_tile.cuh"

namespace {

using hv::TileArgs;

template <int n, int TX, int TY, int F>
struct TileCfg {
  static constexpr int N = n - 1;
  static constexpr int U = TX * N + 1, V = TY * N + 1;
  static constexpr int NE = TX * TY, NN = n * n;
  static constexpr int NT = NE * NN * F;
  static constexpr int NODES = U * V * n;
  static constexpr int SQ = NODES * F;
  static constexpr int SE = NE * n * n * n * F;
  static constexpr int WL = 6 * n * NE * NN;             // packed metric doubles per tile-layer
  static constexpr int PQ = (SQ + NT - 1) / NT;          // gather items per thread
  static constexpr int PM = (NODES + NT - 1) / NT;       // node items per thread
  // shared memory carve-up (doubles): q | W | a | b | Minv[2] ; ints: gid[2] ; mbarrier
  static constexpr int OFF_W = (SQ + 1) & ~1;             // 16-byte aligned TMA destination
  static constexpr int OFF_A = OFF_W + WL;
  static constexpr int OFF_B = OFF_A + SE;
  static constexpr int OFF_M = OFF_B + SE;
  static constexpr int OFF_G = OFF_M + 2 * NODES;         // in doubles; ints packed 2 per double
  static constexpr int OFF_BAR = OFF_G + NODES;           // 2*NODES ints == NODES doubles
  static constexpr size_t SMEM = sizeof(double) * (OFF_BAR + 2);
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// one elected thread: expect `bytes` on the barrier and start the bulk copy global -> shared
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}

template <int n, int TX, int TY, int F>
__global__ void __launch_bounds__(TileCfg<n, TX, TY, F>::NT, (TileCfg<n, TX, TY, F>::NT <= 512 ? 2 : 1))
    lap_tile_kernel(hv::DTab<n> Dt, TileArgs A) {
  using C = TileCfg<n, TX, TY, F>;
  constexpr int N = C::N, V = C::V, NE = C::NE, NN = C::NN, U = C::U;
  extern __shared__ __align__(16) double sm[];
  double* s_q = sm;                 // [U][V][n][F] gathered q of the current layer
  double* s_w = sm + C::OFF_W;      // [6][n][NE][NN] packed metric of the current layer (TMA)
  double* s_a = sm + C::OFF_A;      // [NE][n][n][n][F] xi scratch / element accumulator
  double* s_b = sm + C::OFF_B;      // [NE][n][n][n][F] eta scratch
  double* s_mi = sm + C::OFF_M;     // [2][NODES] Minv of the tile nodes
  int* s_g = reinterpret_cast<int*>(sm + C::OFF_G);   // [2][NODES] gids of the tile nodes
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + C::OFF_BAR);
  const int tid = threadIdx.x;
  const int f = tid % F;
  const int line = tid / F;
  const int e = line / NN;
  const int ij = line % NN;
  const int i = ij / n, j = ij % n;
  const int px = e / TY, py = e % TY;
  const int64_t t = blockIdx.x;
  const int tx = A.tmeta[2 * t], ty = A.tmeta[2 * t + 1];
  const bool act = (px < tx) && (py < ty);
  const int nlay = A.nlay;
  const int32_t* code_t = A.code + t * (U * V);
  const int32_t* gt_t = A.gt + t * (int64_t)nlay * C::NODES;
  const double* Wt_t = A.Wt + t * (int64_t)nlay * C::WL;
  auto eidx = [&](int ee, int a, int b, int c) { return (((ee * n + a) * n + b) * n + c) * F + f; };
  auto tidx = [&](int u, int v, int k) { return ((u * V + v) * n + k) * F + f; };

  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  // prologue: layer 0 gather (direct), its gids / Minv, W(0) by TMA; gids of layer 1 in registers
  for (int s = 0; s < C::PM; ++s) {
    const int node = tid + s * C::NT;
    if (node < C::NODES) {
      const int g = gt_t[node];
      s_g[node] = g;
      s_mi[node] = (g >= 0) ? A.Minv[g] : 0.0;
    }
  }
  for (int s = 0; s < C::PQ; ++s) {
    const int idx = tid + s * C::NT;
    if (idx < C::SQ) {
      const int g = gt_t[idx / F];
      s_q[idx] = (g >= 0) ? A.q[(int64_t)g * A.ldq + A.qf.f[idx % F]] : 0.0;
    }
  }
  __syncthreads();
  if (tid == 0) tma_load_1d(s_w, Wt_t, C::WL * sizeof(double), bar);
  int gq[C::PQ], gm[C::PM];   // gids of the next layer's gather items
  for (int s = 0; s < C::PQ; ++s) {
    const int idx = tid + s * C::NT;
    gq[s] = (nlay > 1 && idx < C::SQ) ? gt_t[C::NODES + idx / F] : -1;
  }
  for (int s = 0; s < C::PM; ++s) {
    const int node = tid + s * C::NT;
    gm[s] = (nlay > 1 && node < C::NODES) ? gt_t[C::NODES + node] : -1;
  }
  double carry = 0.0;

  for (int l = 0; l < nlay; ++l) {
    const int cur = l & 1, nxt = cur ^ 1;
    // ---- prefetch of layer l+1 into registers (overlaps this layer's compute)
    double qn[C::PQ], mn[C::PM];
#pragma unroll
    for (int s = 0; s < C::PQ; ++s) {
      const int idx = tid + s * C::NT;
      qn[s] = (gq[s] >= 0) ? A.q[(int64_t)gq[s] * A.ldq + A.qf.f[idx % F]] : 0.0;
    }
#pragma unroll
    for (int s = 0; s < C::PM; ++s) mn[s] = (gm[s] >= 0) ? A.Minv[gm[s]] : 0.0;
    // ---- S1: strong xi and eta derivatives (one line each per thread)
    if (act) {
      const int b = ij / n, c = ij % n;
      double v[n];
#pragma unroll
      for (int a = 0; a < n; ++a) v[a] = s_q[tidx(px * N + a, py * N + b, c)];
#pragma unroll
      for (int a2 = 0; a2 < n; ++a2) {
        double d = 0.0;
#pragma unroll
        for (int a = 0; a < n; ++a) d = fma(Dt.D[a2][a], v[a], d);
        s_a[eidx(e, a2, b, c)] = d;
      }
#pragma unroll
      for (int a = 0; a < n; ++a) v[a] = s_q[tidx(px * N + b, py * N + a, c)];
#pragma unroll
      for (int a2 = 0; a2 < n; ++a2) {
        double d = 0.0;
#pragma unroll
        for (int a = 0; a < n; ++a) d = fma(Dt.D[a2][a], v[a], d);
        s_b[eidx(e, b, a2, c)] = d;
      }
    }
    __syncthreads();
    // ---- P: zeta derivative, metric contraction, zeta weak derivative
    mbar_wait(bar, (uint32_t)(l & 1));
    double acc[n];
#pragma unroll
    for (int k = 0; k < n; ++k) acc[k] = 0.0;
    if (act) {
      double qk[n], f2[n];
#pragma unroll
      for (int k = 0; k < n; ++k) qk[k] = s_q[tidx(px * N + i, py * N + j, k)];
      const double* W = s_w + e * NN + ij;
#pragma unroll
      for (int k = 0; k < n; ++k) {
        double d2 = 0.0;
#pragma unroll
        for (int a = 0; a < n; ++a) d2 = fma(Dt.D[k][a], qk[a], d2);
        const int id = eidx(e, i, j, k);
        const double d0 = s_a[id], d1 = s_b[id];
        const double w00 = W[(0 * n + k) * NE * NN], w01 = W[(1 * n + k) * NE * NN];
        const double w02 = W[(2 * n + k) * NE * NN], w11 = W[(3 * n + k) * NE * NN];
        const double w12 = W[(4 * n + k) * NE * NN], w22 = W[(5 * n + k) * NE * NN];
        s_a[id] = w00 * d0 + w01 * d1 + w02 * d2;
        s_b[id] = w01 * d0 + w11 * d1 + w12 * d2;
        f2[k] = w02 * d0 + w12 * d1 + w22 * d2;
      }
#pragma unroll
      for (int k = 0; k < n; ++k) {
        double s = 0.0;
#pragma unroll
        for (int a = 0; a < n; ++a) s = fma(Dt.D[a][k], f2[a], s);
        acc[k] = -s;
      }
    }
    __syncthreads();
    // s_q and s_w of layer l are dead: start W(l+1), park the prefetched layer l+1
    if (l + 1 < nlay) {
      if (tid == 0) {
        fence_proxy_async();
        tma_load_1d(s_w, Wt_t + (int64_t)(l + 1) * C::WL, C::WL * sizeof(double), bar);
      }
#pragma unroll
      for (int s = 0; s < C::PQ; ++s) {
        const int idx = tid + s * C::NT;
        if (idx < C::SQ) s_q[idx] = qn[s];
      }
#pragma unroll
      for (int s = 0; s < C::PM; ++s) {
        const int node = tid + s * C::NT;
        if (node < C::NODES) {
          s_g[nxt * C::NODES + node] = gm[s];
          s_mi[nxt * C::NODES + node] = mn[s];
        }
      }
      // gids of layer l+2
#pragma unroll
      for (int s = 0; s < C::PQ; ++s) {
        const int idx = tid + s * C::NT;
        gq[s] = (l + 2 < nlay && idx < C::SQ) ? gt_t[(int64_t)(l + 2) * C::NODES + idx / F] : -1;
      }
#pragma unroll
      for (int s = 0; s < C::PM; ++s) {
        const int node = tid + s * C::NT;
        gm[s] = (l + 2 < nlay && node < C::NODES) ? gt_t[(int64_t)(l + 2) * C::NODES + node] : -1;
      }
    }
    // ---- W1: weak xi / eta derivatives in place
    if (act) {
      const int b = ij / n, c = ij % n;
      double v[n];
#pragma unroll
      for (int a = 0; a < n; ++a) v[a] = s_a[eidx(e, a, b, c)];
#pragma unroll
      for (int a2 = 0; a2 < n; ++a2) {
        double s = 0.0;
#pragma unroll
        for (int a = 0; a < n; ++a) s = fma(Dt.D[a][a2], v[a], s);
        s_a[eidx(e, a2, b, c)] = s;
      }
#pragma unroll
      for (int a = 0; a < n; ++a) v[a] = s_b[eidx(e, b, a, c)];
#pragma unroll
      for (int a2 = 0; a2 < n; ++a2) {
        double s = 0.0;
#pragma unroll
        for (int a = 0; a < n; ++a) s = fma(Dt.D[a][a2], v[a], s);
        s_b[eidx(e, b, a2, c)] = s;
      }
    }
    __syncthreads();
    // ---- A: element accumulator (+ vertical carry) into s_a
    const int kmax = (l == nlay - 1) ? n : N;
    if (act) {
#pragma unroll
      for (int k = 0; k < n; ++k) {
        const int id = eidx(e, i, j, k);
        acc[k] -= s_a[id] + s_b[id];
      }
      acc[0] += carry;
      carry = acc[N];
#pragma unroll
      for (int k = 0; k < n; ++k) s_a[eidx(e, i, j, k)] = acc[k];
    }
    __syncthreads();
    // ---- O: node owners sum the (1, 2 or 4) element copies in fixed order
    {
      const int* g_l = s_g + cur * C::NODES;
      const double* mi_l = s_mi + cur * C::NODES;
      const int nout = U * V * kmax * F;
      for (int idx = tid; idx < nout; idx += C::NT) {
        const int ff = idx % F;
        const int r = idx / F;
        const int uv = r / kmax, k = r % kmax;
        const int u = uv / V, v = uv % V;
        const int node = uv * n + k;
        const int g = g_l[node];
        if (g < 0) continue;
        const int pu1 = min(u / N, TX - 1), pv1 = min(v / N, TY - 1);
        const int pu0 = (u % N == 0 && u > 0) ? u / N - 1 : pu1;
        const int pv0 = (v % N == 0 && v > 0) ? v / N - 1 : pv1;
        double val = 0.0;
        for (int a = pu0; a <= pu1; ++a)
          for (int b = pv0; b <= pv1; ++b) {
            if (a >= tx || b >= ty) continue;
            const int ee = a * TY + b;
            val += s_a[(((ee * n + (u - a * N)) * n + (v - b * N)) * n + k) * F + ff];
          }
        const int cd = code_t[uv];
        if (cd < 0) {
          double* o = A.out + (int64_t)g * A.ldo;
          o[A.of.f[ff]] = A.scale * (mi_l[node] * val);
          if (ff == 0 && A.zero_mask)
            for (int zc = 0; zc < A.ldo; ++zc)
              if ((A.zero_mask >> zc) & 1u) o[zc] = 0.0;
        } else {
          A.part[((int64_t)cd * A.n_z + l * N + k) * 5 + ff] = val;
        }
      }
    }
    __syncthreads();
  }
}

// Perimeter nodes: sum the partial rows of all owning tiles in fixed order.
template <int F>
__global__ void lap_tile_fixup(TileArgs A, int64_t nslot) {
  const int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (id >= nslot * A.n_z) return;
  const int64_t s = id / A.n_z;
  const int z = (int)(id % A.n_z);
  const int c = A.slot_col[s];
  const int g = A.col_gid[(int64_t)c * A.n_z + z];
  const int r0 = A.slot_row0[s], nc = A.slot_nc[s];
  double acc[F];
#pragma unroll
  for (int ff = 0; ff < F; ++ff) acc[ff] = 0.0;
  for (int r = 0; r < nc; ++r) {
    const double* p = A.part + ((int64_t)(r0 + r) * A.n_z + z) * 5;
#pragma unroll
    for (int ff = 0; ff < F; ++ff) acc[ff] += p[ff];
  }
  double* o = A.out + (int64_t)g * A.ldo;
  const double mi = A.Minv[g];
#pragma unroll
  for (int ff = 0; ff < F; ++ff) o[A.of.f[ff]] = A.scale * (mi * acc[ff]);
  if (A.zero_mask)
    for (int zc = 0; zc < A.ldo; ++zc)
      if ((A.zero_mask >> zc) & 1u) o[zc] = 0.0;
}

// Tiled packed metric: Wt[t][l][c][k][e][ij] = W[c][elem(t,l,e)*n^3 + ij*n + k].
__global__ void tile_pack_metric(int n, int NE, int64_t ntiles, int nlay, const int32_t* __restrict__ elem,
                                 const double* __restrict__ W, int64_t nloc, double* __restrict__ Wt) {
  const int NN = n * n;
  const int64_t per = (int64_t)6 * n * NE * NN;
  const int64_t total = ntiles * nlay * per;
  for (int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; id < total; id += (int64_t)gridDim.x * blockDim.x) {
    const int64_t tl = id / per;
    int64_t r = id % per;
    const int ij = (int)(r % NN); r /= NN;
    const int e = (int)(r % NE); r /= NE;
    const int k = (int)(r % n); r /= n;
    const int c = (int)r;
    const int eg = elem[tl * NE + e];
    Wt[id] = (eg >= 0) ? W[c * nloc + (int64_t)eg * n * NN + ij * n + k] : 0.0;
  }
}

template <int n, int TX, int TY, int F>
int run_tile(const TileArgs& A, const double* Drow, cudaStream_t st) {
  using C = TileCfg<n, TX, TY, F>;
  hv::DTab<n> Dt;
  hv::fill_dtab(Dt, Drow);
  auto kern = lap_tile_kernel<n, TX, TY, F>;
  static bool attr = false;
  if (!attr) {
    HV_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
    attr = true;
  }
  kern<<<(unsigned)A.ntiles, C::NT, C::SMEM, st>>>(Dt, A);
  HV_LAUNCH_CHECK();
  if (A.nslot > 0) {
    const int64_t tot = A.nslot * A.n_z;
    lap_tile_fixup<F><<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(A, A.nslot);
    HV_LAUNCH_CHECK();
  }
  return HV_OK;
}

}  // namespace

namespace hv {

bool tile_supported(int N, int TX, int TY, int F) {
  if (F != 1 && F != 4 && F != 5) return false;
  if (N == 7) return TX == 2 && TY == 1;
  return N >= 1 && N <= 6 && TX == 2 && TY == 2;
}

int laplacian_tile(const TileArgs& A, int N, int F, const double* Drow, cudaStream_t st) {
#define HV_TILE_CASE(NN_, TX_, TY_)                                             \
  if (N == NN_ && A.TX == TX_ && A.TY == TY_) {                                \
    if (F == 1) return run_tile<NN_ + 1, TX_, TY_, 1>(A, Drow, st);            \
    if (F == 4) return run_tile<NN_ + 1, TX_, TY_, 4>(A, Drow, st);            \
    if (F == 5) return run_tile<NN_ + 1, TX_, TY_, 5>(A, Drow, st);            \
  }
  HV_TILE_CASE(1, 2, 2)
  HV_TILE_CASE(2, 2, 2)
  HV_TILE_CASE(3, 2, 2)
  HV_TILE_CASE(4, 2, 2)
  HV_TILE_CASE(5, 2, 2)
  HV_TILE_CASE(6, 2, 2)
  HV_TILE_CASE(7, 2, 1)
#undef HV_TILE_CASE
  HV_FAIL(HV_ERR_UNSUPPORTED, "tile kernel: no instantiation for N=%d TX=%d TY=%d F=%d", N, A.TX, A.TY, F);
}

int tile_pack(int N, int NE, int64_t ntiles, int nlay, const int32_t* elem, const double* W, int64_t nloc,
              double* Wt, cudaStream_t st) {
  tile_pack_metric<<<148 * 8, 256, 0, st>>>(N + 1, NE, ntiles, nlay, elem, W, nloc, Wt);
  HV_LAUNCH_CHECK();
  return HV_OK;
}

}  // namespace hv
