// Hot path v3: plane-owner tile sweep for the Laplacian (sm_100a, fp64).
//
// Same tile sweep and on-chip DSS as lap_tile.cu (tiles.py plan, perimeter
// partial rows + fixed-order fix-up), different work split inside a layer:
// thread (element e, eta index jp, field f) owns the (xi, zeta) PLANE of its
// element at eta = jp, so the xi and zeta line contractions (strong and weak)
// run entirely in registers and only the eta direction is transposed through
// shared memory.  Shared-memory traffic drops from ~21 to ~11 accesses per
// element-node-field; the packed metric is read straight from L2 (the next
// layer's block is prefetched into L2 by a bulk-prefetch one step ahead) and
// the next layer's q gather lands in a second shared buffer by cp.async.
//
// Per layer step (5 CTA barriers):
//   a  wait for q(l) (cp.async group), issue q(l+1) gather + metric L2 prefetch
//   b  plane load; dq_xi, dq_zeta in registers; eta lines (i = jp) strong -> scratch
//   c  dq_eta at the plane; flux f = W dq; f_eta -> scratch; weak xi / zeta in registers
//   d  eta lines weak (in place in scratch)
//   e  element accumulator (+ vertical carry in registers) -> scratch
//   f  node owners sum the element copies; final values / partial rows
#include <cuda_runtime.h>

#include <cstdlib>

#include "hv_common.h"
#include "lap_common.cuh"
#include "lap_tile.cuh"

namespace {

using hv::TileArgs;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tma_copy(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void l2_prefetch(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
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
struct PlaneCfg {
  static constexpr int N = n - 1;
  static constexpr int U = TX * N + 1, V = TY * N + 1, UV = U * V;
  static constexpr int NE = TX * TY;
  static constexpr int NT = NE * n * F;                  // threads: (element, eta plane, field)
  static constexpr int NODES = UV * n;
  static constexpr int GTS = (NODES + 3) & ~3;
  static constexpr int MTS = (NODES + 1) & ~1;
  // field-major (SoA) shared arrays; plane strides padded to 4 (mod 16 doubles) so the lanes
  // (element, eta plane, field) of a warp spread over the banks and node-granular lanes
  // (gather / output) are conflict-free
  static constexpr int pad16(int x) { return x + ((4 - (x % 16)) + 16) % 16; }
  static constexpr int QP = pad16(NODES);                // s_q field-plane stride
  static constexpr int SP = pad16(NE * n * n * n);       // scratch field-plane stride
  static constexpr int SQ = QP * F;
  static constexpr int SE = SP * F;
  static constexpr int WL = 6 * n * NE * n * n;          // packed metric doubles per tile-layer
  static constexpr int PN = (NODES + NT - 1) / NT;       // node items per thread
  // shared memory (doubles): q | W | scratch | Minv[2] | gid[3] (ints) | ctab (int4) | code | mbarrier[2]
  static constexpr int OFF_W = (SQ + 1) & ~1;
  static constexpr int OFF_S = OFF_W + WL;
  static constexpr int OFF_M = OFF_S + SE;
  static constexpr int OFF_G = OFF_M + 2 * MTS;
  static constexpr int OFF_T = OFF_G + 3 * GTS / 2;
  static constexpr int OFF_C = OFF_T + 2 * UV;
  static constexpr int OFF_BAR = OFF_C + (UV + 1) / 2 + 1;
  static constexpr size_t SMEM = sizeof(double) * (OFF_BAR + 2);
  static constexpr int BY_SMEM = (int)((227 * 1024) / (SMEM + 1024));
  static constexpr int MINB = BY_SMEM >= 3 ? 3 : (BY_SMEM >= 2 ? 2 : 1);
};

// Wp layout (per tile-layer): [cp 3][i n][k n][e NE][j n][2] (component pairs (w00,w01)
// (w02,w11) (w12,w22)); the F field lanes of a plane broadcast one LDS.128.
template <int n, int TX, int TY, int F, int MB>
__global__ void __launch_bounds__(PlaneCfg<n, TX, TY, F>::NT, MB) lap_plane_kernel(hv::DTab<n> Dt, TileArgs A) {
  using C = PlaneCfg<n, TX, TY, F>;
  constexpr int N = C::N, V = C::V, NE = C::NE, UV = C::UV;
  extern __shared__ __align__(16) double sm[];
  double* s_q = sm;                                    // [NODES][F]
  double* s_w = sm + C::OFF_W;                         // metric of the current layer (TMA)
  double* s_s = sm + C::OFF_S;                         // [NE][n i][n j][n k][F] eta scratch / element acc
  double* s_m0 = sm + C::OFF_M;                        // [2][MTS] Minv (TMA)
  int* s_g0 = reinterpret_cast<int*>(sm + C::OFF_G);   // [3][GTS] gids (TMA)
  int4* s_ct = reinterpret_cast<int4*>(sm + C::OFF_T); // [UV] element-copy offsets
  int* s_code = reinterpret_cast<int*>(sm + C::OFF_C); // [UV] partial row or -1
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + C::OFF_BAR);  // [0] Minv/gid stage, [1] metric
  const int tid = threadIdx.x;
  const int f = tid % F;
  const int jp = (tid / F) % n;
  const int e = tid / (F * n);
  const int px = e / TY, py = e % TY;
  const int64_t t = blockIdx.x;
  const int tx = A.tmeta[2 * t], ty = A.tmeta[2 * t + 1];
  const bool act = (px < tx) && (py < ty);
  const int nlay = A.nlay;
  const int32_t* gt_t = A.gt + t * (int64_t)nlay * C::GTS;
  const double* Wt_t = A.Wt + t * (int64_t)nlay * C::WL;
  const double* Mt_t = A.Mt + t * (int64_t)nlay * C::MTS;
  int qcol[F], ocol[F];
#pragma unroll
  for (int p = 0; p < F; ++p) {
    qcol[p] = A.qf.f[p];
    ocol[p] = A.of.f[p];
  }
  const bool row5 = (F == 4 && A.ldo == 5 && ocol[0] == 1 && ocol[1] == 2 && ocol[2] == 3 && ocol[3] == 4);
  // element-private scratch index (this thread's field); tile-node index (field-major planes)
  auto sidx = [&](int ee, int a, int b, int c) { return f * C::SP + ((ee * n + a) * n + b) * n + c; };
  auto tq = [&](int u, int v, int k) { return f * C::QP + (u * V + v) * n + k; };

  auto issue_stage = [&](int l) {       // Minv(l) -> M[l%2], gids(l+1) -> G[(l+1)%3] on bar[0]
    const int b = l & 1;
    const bool nextg = (l + 1 < nlay);
    const uint32_t bytes = C::MTS * 8 + (nextg ? C::GTS * 4 : 0);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
    tma_copy(s_m0 + b * C::MTS, Mt_t + (int64_t)l * C::MTS, C::MTS * 8, bar);
    if (nextg) tma_copy(s_g0 + ((l + 1) % 3) * C::GTS, gt_t + (int64_t)(l + 1) * C::GTS, C::GTS * 4, bar);
  };
  auto issue_metric = [&](int l) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar + 1)), "r"(C::WL * 8)
                 : "memory");
    tma_copy(s_w, Wt_t + (int64_t)l * C::WL, C::WL * 8, bar + 1);
  };
  // node-granular async gather of one layer of q (all F fields of a node per item)
  auto issue_gather = [&](const int* g_src) {
    for (int node = tid; node < C::NODES; node += C::NT) {
      const int g = g_src[node];
      if (g < 0) {
#pragma unroll
        for (int p = 0; p < F; ++p) s_q[p * C::QP + node] = 0.0;
      } else {
        const double* src = A.q + (int64_t)g * A.ldq;
#pragma unroll
        for (int p = 0; p < F; ++p) cp_async8(s_q + p * C::QP + node, src + qcol[p]);
      }
    }
    cp_async_commit();
  };

  if (tid == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    fence_mbar_init();
  }
  for (int uv = tid; uv < UV; uv += C::NT) {
    const int u = uv / V, v = uv % V;
    const int pu1 = min(u / N, TX - 1), pv1 = min(v / N, TY - 1);
    const int pu0 = (u % N == 0 && u > 0) ? u / N - 1 : pu1;
    const int pv0 = (v % N == 0 && v > 0) ? v / N - 1 : pv1;
    int o[4] = {-1, -1, -1, -1}, c = 0;
    for (int a = pu0; a <= pu1; ++a)
      for (int b = pv0; b <= pv1; ++b) o[c++] = (((a * TY + b) * n + (u - a * N)) * n + (v - b * N)) * n;
    s_ct[uv] = make_int4(o[0], o[1], o[2], o[3]);
    s_code[uv] = A.code[t * UV + uv];
  }
  for (int node = tid; node < C::NODES; node += C::NT) s_g0[node] = gt_t[node];
  __syncthreads();
  if (tid == 0) {
    issue_stage(0);
    issue_metric(0);
  }
  issue_gather(s_g0);
  double carry[n];
#pragma unroll
  for (int i = 0; i < n; ++i) carry[i] = 0.0;

  for (int l = 0; l < nlay; ++l) {
    const int b = l & 1;
    // ---- a: q(l) and stage l have landed; start Minv / gids of l+1
    cp_async_wait_all();
    mbar_wait(bar, (uint32_t)(l & 1));
    __syncthreads();
    if (tid == 0 && l + 1 < nlay) {
      fence_proxy_async();
      issue_stage(l + 1);
    }
    const double* s_mi = s_m0 + b * C::MTS;
    const int* s_g = s_g0 + (l % 3) * C::GTS;
    // ---- b: plane derivatives in registers, eta lines (i = jp) strong
    double p0[n][n], p2[n][n];   // [i][k]: dq_xi, dq_zeta -> f_xi, f_zeta -> accumulator
    if (act) {
#pragma unroll
      for (int i = 0; i < n; ++i) {
        double ql[n];
#pragma unroll
        for (int k = 0; k < n; ++k) ql[k] = s_q[tq(px * N + i, py * N + jp, k)];
#pragma unroll
        for (int k = 0; k < n; ++k) {
          double s = 0.0;
#pragma unroll
          for (int a = 0; a < n; ++a) s = fma(Dt.D[k][a], ql[a], s);
          p2[i][k] = s;
        }
#pragma unroll
        for (int k = 0; k < n; ++k) p0[i][k] = ql[k];   // q plane, xi-differentiated below
      }
#pragma unroll
      for (int k = 0; k < n; ++k) {
        double ql[n];
#pragma unroll
        for (int i = 0; i < n; ++i) ql[i] = p0[i][k];
#pragma unroll
        for (int i = 0; i < n; ++i) {
          double s = 0.0;
#pragma unroll
          for (int a = 0; a < n; ++a) s = fma(Dt.D[i][a], ql[a], s);
          p0[i][k] = s;
        }
      }
      // eta lines of element e with i = jp: dq_eta(e, jp, a', k)
#pragma unroll
      for (int k = 0; k < n; ++k) {
        double ql[n];
#pragma unroll
        for (int a = 0; a < n; ++a) ql[a] = s_q[tq(px * N + jp, py * N + a, k)];
#pragma unroll
        for (int a2 = 0; a2 < n; ++a2) {
          double s = 0.0;
#pragma unroll
          for (int a = 0; a < n; ++a) s = fma(Dt.D[a2][a], ql[a], s);
          s_s[sidx(e, jp, a2, k)] = s;
        }
      }
    }
    __syncthreads();
    // s_q of layer l is dead: gather q(l+1) (addresses arrived with stage l)
    if (l + 1 < nlay) issue_gather(s_g0 + ((l + 1) % 3) * C::GTS);
    // ---- c: flux at the plane nodes, weak xi / zeta in registers
    mbar_wait(bar + 1, (uint32_t)(l & 1));
    if (act) {
      const double* W = s_w + (e * n + jp) * 2;
#pragma unroll
      for (int i = 0; i < n; ++i)
#pragma unroll
        for (int k = 0; k < n; ++k) {
          const int wo = (i * n + k) * NE * n * 2;
          const double2 wa = *reinterpret_cast<const double2*>(W + 0 * n * n * NE * n * 2 + wo);   // w00 w01
          const double2 wb = *reinterpret_cast<const double2*>(W + 1 * n * n * NE * n * 2 + wo);   // w02 w11
          const double2 wc = *reinterpret_cast<const double2*>(W + 2 * n * n * NE * n * 2 + wo);   // w12 w22
          const int id = sidx(e, i, jp, k);
          const double d0 = p0[i][k], d1 = s_s[id], d2 = p2[i][k];
          p0[i][k] = wa.x * d0 + wa.y * d1 + wb.x * d2;
          s_s[id] = wa.y * d0 + wb.y * d1 + wc.x * d2;
          p2[i][k] = wb.x * d0 + wc.x * d1 + wc.y * d2;
        }
      // weak xi (columns of p0, in place): p0[i][k] <- -sum_a D[a][i] f_xi[a][k]
#pragma unroll
      for (int k = 0; k < n; ++k) {
        double c[n];
#pragma unroll
        for (int a = 0; a < n; ++a) c[a] = p0[a][k];
#pragma unroll
        for (int i = 0; i < n; ++i) {
          double s = 0.0;
#pragma unroll
          for (int a = 0; a < n; ++a) s = fma(Dt.D[a][i], c[a], s);
          p0[i][k] = -s;
        }
      }
      // weak zeta (rows of p2) accumulated into p0
#pragma unroll
      for (int i = 0; i < n; ++i)
#pragma unroll
        for (int k = 0; k < n; ++k) {
          double s = 0.0;
#pragma unroll
          for (int a = 0; a < n; ++a) s = fma(Dt.D[a][k], p2[i][a], s);
          p0[i][k] -= s;
        }
    }
    __syncthreads();
    if (tid == 0 && l + 1 < nlay) {      // metric buffer free: W(l+1) lands during d, e, f, a, b
      fence_proxy_async();
      issue_metric(l + 1);
    }
    // ---- d: eta lines weak, in place (line i = jp of element e)
    if (act) {
#pragma unroll
      for (int k = 0; k < n; ++k) {
        double ql[n];
#pragma unroll
        for (int a = 0; a < n; ++a) ql[a] = s_s[sidx(e, jp, a, k)];
#pragma unroll
        for (int a2 = 0; a2 < n; ++a2) {
          double s = 0.0;
#pragma unroll
          for (int a = 0; a < n; ++a) s = fma(Dt.D[a][a2], ql[a], s);
          s_s[sidx(e, jp, a2, k)] = s;
        }
      }
    }
    __syncthreads();
    // ---- e: element accumulator (+ vertical carry) -> scratch
    if (act) {
#pragma unroll
      for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int k = 0; k < n; ++k) p0[i][k] -= s_s[sidx(e, i, jp, k)];
        p0[i][0] += carry[i];
        carry[i] = p0[i][N];
#pragma unroll
        for (int k = 0; k < n; ++k) s_s[sidx(e, i, jp, k)] = p0[i][k];
      }
    } else {
#pragma unroll
      for (int i = 0; i < n; ++i)
#pragma unroll
        for (int k = 0; k < n; ++k) s_s[sidx(e, i, jp, k)] = 0.0;
    }
    __syncthreads();
    // ---- f: node owners sum the element copies (all F fields per item); whole-row stores
    {
      const int kmax = (l == nlay - 1) ? n : N;
#pragma unroll
      for (int it = 0; it < C::PN; ++it) {
        const int node = tid + it * C::NT;   // = uv * n + k
        if (node >= C::NODES) break;
        const int k = node % n, uv = node / n;
        if (k >= kmax) continue;
        const int g = s_g[node];
        if (g < 0) continue;
        const int4 ct = s_ct[uv];
        double val[F];
#pragma unroll
        for (int p = 0; p < F; ++p) {
          const double* sp = s_s + p * C::SP + k;
          double a = sp[ct.x];
          if (ct.y >= 0) a += sp[ct.y];
          if (ct.z >= 0) a += sp[ct.z] + sp[ct.w];
          val[p] = a;
        }
        const int cd = s_code[uv];
        if (cd < 0) {
          double* o = A.out + (int64_t)g * A.ldo;
          const double m = A.scale * s_mi[node];
          if (A.accumulate) {
#pragma unroll
            for (int p = 0; p < F; ++p) o[ocol[p]] += m * val[p];
          } else if (row5) {
            o[0] = 0.0;
#pragma unroll
            for (int p = 0; p < F; ++p) o[1 + p] = m * val[p];
          } else {
#pragma unroll
            for (int p = 0; p < F; ++p) o[ocol[p]] = m * val[p];
            if (A.zero_mask)
              for (int zc = 0; zc < A.ldo; ++zc)
                if ((A.zero_mask >> zc) & 1u) o[zc] = 0.0;
          }
        } else {
          double* o = A.part + ((int64_t)cd * A.n_z + l * N + k) * 5;
#pragma unroll
          for (int p = 0; p < F; ++p) o[p] = val[p];
        }
      }
    }
    // the next step's barrier (a) orders these reads before the scratch is rewritten
  }
}


// Plane-layout packed metric, component pairs:
// Wp[t][l][cp][i][k][e][j][h] = W[2cp+h][elem(t,l,e)*n^3 + (i*n + j)*n + k].
__global__ void plane_pack_metric(int n, int NE, int64_t ntiles, int nlay, const int32_t* __restrict__ elem,
                                  const double* __restrict__ W, int64_t nloc, double* __restrict__ Wp) {
  const int64_t per = (int64_t)6 * n * n * NE * n;
  const int64_t total = ntiles * nlay * per;
  for (int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; id < total; id += (int64_t)gridDim.x * blockDim.x) {
    const int64_t tl = id / per;
    int64_t r = id % per;
    const int h = (int)(r % 2); r /= 2;
    const int j = (int)(r % n); r /= n;
    const int e = (int)(r % NE); r /= NE;
    const int k = (int)(r % n); r /= n;
    const int i = (int)(r % n); r /= n;
    const int c = (int)r * 2 + h;
    const int eg = elem[tl * NE + e];
    Wp[id] = (eg >= 0) ? W[c * nloc + (int64_t)eg * n * n * n + (i * n + j) * n + k] : 0.0;
  }
}

template <int n, int TX, int TY, int F>
int run_plane(const TileArgs& A, const double* Drow, cudaStream_t st) {
  using C = PlaneCfg<n, TX, TY, F>;
  hv::DTab<n> Dt;
  hv::fill_dtab(Dt, Drow);
  auto kern = lap_plane_kernel<n, TX, TY, F, C::MINB>;
  HV_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
  kern<<<(unsigned)A.ntiles, C::NT, C::SMEM, st>>>(Dt, A);
  HV_LAUNCH_CHECK();
  return HV_OK;
}

}  // namespace

namespace hv {

bool plane_supported(int N, int TX, int TY, int F) {
  return (F == 1 || F == 4 || F == 5) && TX == 2 && TY == 2 && N >= 1 && N <= 4;
}

int laplacian_plane(const TileArgs& A, int N, int F, const double* Drow, cudaStream_t st) {
#define HV_PLANE_CASE(NN_)                                        \
  if (N == NN_) {                                                 \
    if (F == 1) return run_plane<NN_ + 1, 2, 2, 1>(A, Drow, st);  \
    if (F == 4) return run_plane<NN_ + 1, 2, 2, 4>(A, Drow, st);  \
    if (F == 5) return run_plane<NN_ + 1, 2, 2, 5>(A, Drow, st);  \
  }
  HV_PLANE_CASE(1)
  HV_PLANE_CASE(2)
  HV_PLANE_CASE(3)
  HV_PLANE_CASE(4)
#undef HV_PLANE_CASE
  HV_FAIL(HV_ERR_UNSUPPORTED, "plane kernel: no instantiation for N=%d F=%d", N, F);
}

int plane_pack(int N, int NE, int64_t ntiles, int nlay, const int32_t* elem, const double* W, int64_t nloc,
               double* Wp, cudaStream_t st) {
  plane_pack_metric<<<148 * 8, 256, 0, st>>>(N + 1, NE, ntiles, nlay, elem, W, nloc, Wp);
  HV_LAUNCH_CHECK();
  return HV_OK;
}

}  // namespace hv
