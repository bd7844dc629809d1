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
//      slot_fixup in dss_slots.cu (deterministic, atomics-free).
//
// No atomics anywhere; every sum is in a fixed order, so results are
// bitwise reproducible run to run.
#include <cuda_runtime.h>

#include <cstdlib>

#ifndef HV_FP2_MAXN
#define HV_FP2_MAXN 8   // two fields per thread below this n (N = 7 uses one: more warps per SM)
#endif
#ifndef HV_ABLATE
#define HV_ABLATE 0   // timing experiments only: bit 1 skip S1, 2 skip W1, 4 skip O, 8 skip P
#endif

#include "hv_common.h"
#include "lap_common.cuh"
#include "lap_tile.cuh"

namespace {

using hv::TileArgs;

// FP doubles held per thread (FP = 2: one LDS.128 / STS.128 per access)
template <int FP>
struct Vec {
  double x[FP];
  __device__ __forceinline__ static Vec ld(const double* p) {
    Vec r;
    if constexpr (FP == 2) {
      const double2 d = *reinterpret_cast<const double2*>(p);
      r.x[0] = d.x;
      r.x[1] = d.y;
    } else {
#pragma unroll
      for (int q = 0; q < FP; ++q) r.x[q] = p[q];
    }
    return r;
  }
  __device__ __forceinline__ void st_any(double* p) const {
#pragma unroll
    for (int q = 0; q < FP; ++q) p[q] = x[q];
  }
  __device__ __forceinline__ void st(double* p) const {
    if constexpr (FP == 2) {
      *reinterpret_cast<double2*>(p) = make_double2(x[0], x[1]);
    } else {
#pragma unroll
      for (int q = 0; q < FP; ++q) p[q] = x[q];
    }
  }
};

template <int n, int TX, int TY, int F, int FP>
struct TileCfg {
  static constexpr int N = n - 1;
  static constexpr int U = TX * N + 1, V = TY * N + 1;
  static constexpr int NE = TX * TY, NN = n * n;
  static constexpr int FL = F / FP;                       // field lanes per line
  static constexpr int NT = NE * NN * FL;                 // threads
  static constexpr int NODES = U * V * n;
  static constexpr int GTS = (NODES + 3) & ~3;            // padded gid-table stride (ints, 16 B multiple)
  static constexpr int MTS = (NODES + 1) & ~1;            // padded Minv-table stride (doubles)
  static constexpr int SQ = NODES * F;
  static constexpr int SE = NE * n * n * n * F;
  static constexpr int WL = 6 * n * NE * NN;             // packed metric doubles per tile-layer
  static constexpr int PN = (NODES + NT - 1) / NT;       // node items per thread (gather / output)
  static constexpr int UV = U * V;
  // shared memory (doubles): q | W[WB] | a | b | Minv[2] | gid[3] (ints) | ctab (ints) | mbarrier[2]
  static constexpr int OFF_W = (SQ + 1) & ~1;
  static constexpr size_t SMEM2 = sizeof(double) * (OFF_W + 2 * WL + 2 * SE + 2 * MTS + 3 * GTS / 2 + 3 * UV + 6);
  static constexpr int WB = (SMEM2 <= 220 * 1024) ? 2 : 1;   // metric ring depth
  static constexpr int OFF_A = OFF_W + WB * WL;
  static constexpr int OFF_B = OFF_A + SE;
  static constexpr int OFF_M = OFF_B + SE;
  static constexpr int OFF_G = OFF_M + 2 * MTS;
  static constexpr int OFF_T = OFF_G + 3 * GTS / 2;        // ctab: 4 ints per tile column node
  static constexpr int OFF_C = OFF_T + 2 * UV;              // code: 1 int per tile column node
  static constexpr int OFF_BAR = OFF_C + (UV + 1) / 2 + 1;
  static constexpr size_t SMEM = sizeof(double) * (OFF_BAR + 2);
  static constexpr int BY_SMEM = (int)((227 * 1024) / (SMEM + 1024));
  static constexpr int MINB = BY_SMEM >= 3 ? 3 : (BY_SMEM >= 2 ? 2 : 1);   // CTAs per SM we aim for
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
__device__ __forceinline__ void tma_copy(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
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

template <int n, int TX, int TY, int F, int FP, int MB>
__global__ void __launch_bounds__(TileCfg<n, TX, TY, F, FP>::NT, MB)
    lap_tile_kernel(hv::DTab<n> Dt, TileArgs A) {
  using C = TileCfg<n, TX, TY, F, FP>;
  using VT = Vec<FP>;
  constexpr int N = C::N, V = C::V, NE = C::NE, NN = C::NN, U = C::U, FL = C::FL;
  extern __shared__ __align__(16) double sm[];
  double* s_q = sm;                 // [U][V][n][F] gathered q of the current layer
  double* s_w0 = sm + C::OFF_W;     // [2][3 pairs][n][NE][NN][2] packed metric ring (TMA)
  double* s_a = sm + C::OFF_A;      // [NE][n][n][n][F] xi scratch / element accumulator
  double* s_b = sm + C::OFF_B;      // [NE][n][n][n][F] eta scratch
  double* s_m0 = sm + C::OFF_M;     // [2][MTS] Minv of the tile nodes (TMA)
  int* s_g0 = reinterpret_cast<int*>(sm + C::OFF_G);   // [3][GTS] gids of the tile nodes (TMA)
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + C::OFF_BAR);
  const int tid = threadIdx.x;
  const int fl = tid % FL;
  const int f0 = fl * FP;
  const int line = tid / FL;
  const int e = line / NN;
  const int ij = line % NN;
  const int i = ij / n, j = ij % n;
  const int px = e / TY, py = e % TY;
  const int64_t t = A.tile0 + blockIdx.x;
  const int tx = A.tmeta[2 * t], ty = A.tmeta[2 * t + 1];
  const bool act = (px < tx) && (py < ty);
  const int nlay = A.nlay;
  const int32_t* code_t = A.code + t * (U * V);
  const int32_t* gt_t = A.gt + t * (int64_t)nlay * C::GTS;
  const double* Wt_t = A.Wt + t * (int64_t)nlay * C::WL;
  const double* Mt_t = A.Mt + t * (int64_t)nlay * C::MTS;
  auto eidx = [&](int ee, int a, int b, int c) { return (((ee * n + a) * n + b) * n + c) * F + f0; };
  auto tidx = [&](int u, int v, int k) { return ((u * V + v) * n + k) * F + f0; };
  // column indices of the F fields in q and out (node-granular gather / output)
  int qcol[F], ocol[F];
#pragma unroll
  for (int p = 0; p < F; ++p) {
    qcol[p] = A.qf.f[p];
    ocol[p] = A.of.f[p];
  }
  // the common state-row case: out is (ng, 5) with fields 1..4 written and column 0 zeroed
  const bool row5 = (F == 4 && A.ldo == 5 && ocol[0] == 1 && ocol[1] == 2 && ocol[2] == 3 && ocol[3] == 4);
  auto gather = [&](int g, double* dst) {   // all F fields of one node
    const double* src = A.q + (int64_t)g * A.ldq;
#pragma unroll
    for (int p = 0; p < F; ++p) dst[p] = (g >= 0) ? src[qcol[p]] : 0.0;
  };
  auto park = [&](int node, const double* v) {
    if constexpr (F % 2 == 0) {
#pragma unroll
      for (int p = 0; p < F; p += 2) *reinterpret_cast<double2*>(s_q + node * F + p) = make_double2(v[p], v[p + 1]);
    } else {
#pragma unroll
      for (int p = 0; p < F; ++p) s_q[node * F + p] = v[p];
    }
  };
  int* s_ct = reinterpret_cast<int*>(sm + C::OFF_T);  // [UV][4] scratch offsets of the element copies
  int* s_code = reinterpret_cast<int*>(sm + C::OFF_C);  // [UV] partial row of a shared column node, -1 owned
  // stage l: W(l) -> W[l%2], Minv(l) -> M[l%2], gids(l+1) -> G[(l+1)%3], all on bar[l%2]
  auto issue_stage = [&](int l) {
    const int b = l & 1;
    const bool nextg = (l + 1 < nlay);
    const uint32_t bytes = C::WL * 8 + C::MTS * 8 + (nextg ? C::GTS * 4 : 0);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar + b)), "r"(bytes)
                 : "memory");
    tma_copy(s_w0 + (C::WB == 2 ? b : 0) * C::WL, Wt_t + (int64_t)l * C::WL, C::WL * 8, bar + b);
    tma_copy(s_m0 + b * C::MTS, Mt_t + (int64_t)l * C::MTS, C::MTS * 8, bar + b);
    if (nextg) tma_copy(s_g0 + ((l + 1) % 3) * C::GTS, gt_t + (int64_t)(l + 1) * C::GTS, C::GTS * 4, bar + b);
  };

  if (tid == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    fence_mbar_init();
  }
  // ctab: for tile column node (u, v) the scratch offsets (k = 0, field 0) of its 1, 2 or 4
  // element copies, -1 padded (absent elements of ragged tiles hold zeros, see phase A)
  for (int uv = tid; uv < C::UV; uv += C::NT) {
    const int u = uv / V, v = uv % V;
    const int pu1 = min(u / N, TX - 1), pv1 = min(v / N, TY - 1);
    const int pu0 = (u % N == 0 && u > 0) ? u / N - 1 : pu1;
    const int pv0 = (v % N == 0 && v > 0) ? v / N - 1 : pv1;
    int c = 0;
    for (int a = pu0; a <= pu1; ++a)
      for (int b = pv0; b <= pv1; ++b) s_ct[uv * 4 + c++] = (((a * TY + b) * n + (u - a * N)) * n + (v - b * N)) * n * F;
    for (; c < 4; ++c) s_ct[uv * 4 + c] = -1;
    s_code[uv] = code_t[uv];
  }
  // prologue: gids and gather of layer 0 directly; stage 0 by TMA
  for (int node = tid; node < C::NODES; node += C::NT) s_g0[node] = gt_t[node];
  __syncthreads();
  if (tid == 0) issue_stage(0);
  for (int node = tid; node < C::NODES; node += C::NT) {
    double v[F];
    gather(s_g0[node], v);
    park(node, v);
  }
  double carry[FP];
#pragma unroll
  for (int p = 0; p < FP; ++p) carry[p] = 0.0;
  __syncthreads();

  for (int l = 0; l < nlay; ++l) {
    const int b = l & 1;
    mbar_wait(bar + b, (uint32_t)((l >> 1) & 1));     // W(l), Minv(l), gids(l+1) have landed
    if (C::WB == 2 && tid == 0 && l + 1 < nlay) {
      fence_proxy_async();
      issue_stage(l + 1);                               // one full step ahead
    }
    const double* s_w = s_w0 + (C::WB == 2 ? b : 0) * C::WL;
    const double* s_mi = s_m0 + b * C::MTS;
    const int* s_g = s_g0 + (l % 3) * C::GTS;
    const int* s_gn = s_g0 + ((l + 1) % 3) * C::GTS;
    // ---- prefetch q(l+1) into registers (addresses from shared memory)
    double qn[C::PN][F];
    if (l + 1 < nlay) {
#pragma unroll
      for (int s = 0; s < C::PN; ++s) {
        const int node = tid + s * C::NT;
        if (node < C::NODES) gather(s_gn[node], qn[s]);
      }
    }
    // ---- S1: strong xi and eta derivatives (one line each per thread)
    if (act && !(HV_ABLATE & 1)) {
      const int b2 = ij / n, c = ij % n;
      VT v[n];
#pragma unroll
      for (int a = 0; a < n; ++a) v[a] = VT::ld(s_q + tidx(px * N + a, py * N + b2, c));
#pragma unroll
      for (int a2 = 0; a2 < n; ++a2) {
        VT d;
#pragma unroll
        for (int p = 0; p < FP; ++p) {
          double s = 0.0;
#pragma unroll
          for (int a = 0; a < n; ++a) s = fma(Dt.D[a2][a], v[a].x[p], s);
          d.x[p] = s;
        }
        d.st(s_a + eidx(e, a2, b2, c));
      }
#pragma unroll
      for (int a = 0; a < n; ++a) v[a] = VT::ld(s_q + tidx(px * N + b2, py * N + a, c));
#pragma unroll
      for (int a2 = 0; a2 < n; ++a2) {
        VT d;
#pragma unroll
        for (int p = 0; p < FP; ++p) {
          double s = 0.0;
#pragma unroll
          for (int a = 0; a < n; ++a) s = fma(Dt.D[a2][a], v[a].x[p], s);
          d.x[p] = s;
        }
        d.st(s_b + eidx(e, b2, a2, c));
      }
    }
    __syncthreads();
    // ---- P: zeta derivative, metric contraction, zeta weak derivative
    double acc[n][FP];
#pragma unroll
    for (int k = 0; k < n; ++k)
#pragma unroll
      for (int p = 0; p < FP; ++p) acc[k][p] = 0.0;
    if (act && !(HV_ABLATE & 8)) {
      VT qk[n];
      double f2[n][FP];
#pragma unroll
      for (int k = 0; k < n; ++k) qk[k] = VT::ld(s_q + tidx(px * N + i, py * N + j, k));
      const double* W = s_w + (e * NN + ij) * 2;
#pragma unroll
      for (int k = 0; k < n; ++k) {
        const double2 wa = *reinterpret_cast<const double2*>(W + (0 * n + k) * NE * NN * 2);   // w00 w01
        const double2 wb = *reinterpret_cast<const double2*>(W + (1 * n + k) * NE * NN * 2);   // w02 w11
        const double2 wc = *reinterpret_cast<const double2*>(W + (2 * n + k) * NE * NN * 2);   // w12 w22
        const int id = eidx(e, i, j, k);
        const VT d0 = VT::ld(s_a + id), d1 = VT::ld(s_b + id);
        VT o0, o1;
#pragma unroll
        for (int p = 0; p < FP; ++p) {
          double d2 = 0.0;
#pragma unroll
          for (int a = 0; a < n; ++a) d2 = fma(Dt.D[k][a], qk[a].x[p], d2);
          o0.x[p] = wa.x * d0.x[p] + wa.y * d1.x[p] + wb.x * d2;
          o1.x[p] = wa.y * d0.x[p] + wb.y * d1.x[p] + wc.x * d2;
          f2[k][p] = wb.x * d0.x[p] + wc.x * d1.x[p] + wc.y * d2;
        }
        o0.st(s_a + id);
        o1.st(s_b + id);
      }
#pragma unroll
      for (int k = 0; k < n; ++k)
#pragma unroll
        for (int p = 0; p < FP; ++p) {
          double s = 0.0;
#pragma unroll
          for (int a = 0; a < n; ++a) s = fma(Dt.D[a][k], f2[a][p], s);
          acc[k][p] = -s;
        }
    }
    __syncthreads();
    if (C::WB == 1 && tid == 0 && l + 1 < nlay) {
      fence_proxy_async();
      issue_stage(l + 1);                               // metric buffer free after phase P
    }
    // s_q of layer l is dead: park the prefetched q(l+1)
    if (l + 1 < nlay) {
#pragma unroll
      for (int s = 0; s < C::PN; ++s) {
        const int node = tid + s * C::NT;
        if (node < C::NODES) park(node, qn[s]);
      }
    }
    // ---- W1: weak xi / eta derivatives in place
    if (act && !(HV_ABLATE & 2)) {
      const int b2 = ij / n, c = ij % n;
      VT v[n];
#pragma unroll
      for (int a = 0; a < n; ++a) v[a] = VT::ld(s_a + eidx(e, a, b2, c));
#pragma unroll
      for (int a2 = 0; a2 < n; ++a2) {
        VT d;
#pragma unroll
        for (int p = 0; p < FP; ++p) {
          double s = 0.0;
#pragma unroll
          for (int a = 0; a < n; ++a) s = fma(Dt.D[a][a2], v[a].x[p], s);
          d.x[p] = s;
        }
        d.st(s_a + eidx(e, a2, b2, c));
      }
#pragma unroll
      for (int a = 0; a < n; ++a) v[a] = VT::ld(s_b + eidx(e, b2, a, c));
#pragma unroll
      for (int a2 = 0; a2 < n; ++a2) {
        VT d;
#pragma unroll
        for (int p = 0; p < FP; ++p) {
          double s = 0.0;
#pragma unroll
          for (int a = 0; a < n; ++a) s = fma(Dt.D[a][a2], v[a].x[p], s);
          d.x[p] = s;
        }
        d.st(s_b + eidx(e, b2, a2, c));
      }
    }
    __syncthreads();
    // ---- A: element accumulator (+ vertical carry) into s_a
    const int kmax = (l == nlay - 1) ? n : N;
    if (!act) {
      VT z;
#pragma unroll
      for (int p = 0; p < FP; ++p) z.x[p] = 0.0;
#pragma unroll
      for (int k = 0; k < n; ++k) z.st(s_a + eidx(e, i, j, k));
    } else {
#pragma unroll
      for (int k = 0; k < n; ++k) {
        const int id = eidx(e, i, j, k);
        const VT a = VT::ld(s_a + id), bb = VT::ld(s_b + id);
#pragma unroll
        for (int p = 0; p < FP; ++p) acc[k][p] -= a.x[p] + bb.x[p];
      }
#pragma unroll
      for (int p = 0; p < FP; ++p) {
        acc[0][p] += carry[p];
        carry[p] = acc[N][p];
      }
#pragma unroll
      for (int k = 0; k < n; ++k) {
        VT o;
#pragma unroll
        for (int p = 0; p < FP; ++p) o.x[p] = acc[k][p];
        o.st(s_a + eidx(e, i, j, k));
      }
    }
    __syncthreads();
    // ---- O: node owners sum the (1, 2 or 4) element copies in fixed order and write
    //      whole rows (all fields of a node from one thread: full sectors, no partial writes)
#pragma unroll
    for (int sidx = 0; sidx < ((HV_ABLATE & 4) ? 0 : C::PN); ++sidx) {
      const int node = tid + sidx * C::NT;    // = uv * n + k
      if (node >= C::NODES) break;
      const int k = node % n, uv = node / n;
      if (k >= kmax) continue;
      const int g = s_g[node];
      if (g < 0) continue;
      const int4 ct = *reinterpret_cast<const int4*>(s_ct + uv * 4);
      const int kof = k * F;
      double val[F];
#pragma unroll
      for (int p = 0; p < F; p += (F % 2 == 0 ? 2 : 1)) {
        if constexpr (F % 2 == 0) {
          double2 a = *reinterpret_cast<const double2*>(s_a + ct.x + kof + p);
          if (ct.y >= 0) {
            const double2 b = *reinterpret_cast<const double2*>(s_a + ct.y + kof + p);
            a.x += b.x;
            a.y += b.y;
          }
          if (ct.z >= 0) {
            const double2 c = *reinterpret_cast<const double2*>(s_a + ct.z + kof + p);
            const double2 d = *reinterpret_cast<const double2*>(s_a + ct.w + kof + p);
            a.x += c.x + d.x;
            a.y += c.y + d.y;
          }
          val[p] = a.x;
          val[p + 1] = a.y;
        } else {
          double a = s_a[ct.x + kof + p];
          if (ct.y >= 0) a += s_a[ct.y + kof + p];
          if (ct.z >= 0) a += s_a[ct.z + kof + p] + s_a[ct.w + kof + p];
          val[p] = a;
        }
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
        double* o = A.part + ((int64_t)cd * A.n_z + l * N + k) * F;
#pragma unroll
        for (int p = 0; p < F; ++p) o[p] = val[p];
      }
    }
    __syncthreads();
  }
}


// Tiled packed metric, component pairs (w00,w01) (w02,w11) (w12,w22):
// Wt[t][l][cp][k][e][ij][2] = W[2cp + h][elem(t,l,e)*n^3 + ij*n + k].
__global__ void tile_pack_metric(int n, int NE, int64_t ntiles, int nlay, const int32_t* __restrict__ elem,
                                 const double* __restrict__ W, int64_t nloc, double* __restrict__ Wt) {
  const int NN = n * n;
  const int64_t per = (int64_t)6 * n * NE * NN;
  const int64_t total = ntiles * nlay * per;
  for (int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; id < total; id += (int64_t)gridDim.x * blockDim.x) {
    const int64_t tl = id / per;
    int64_t r = id % per;
    const int h = (int)(r % 2); r /= 2;
    const int ij = (int)(r % NN); r /= NN;
    const int e = (int)(r % NE); r /= NE;
    const int k = (int)(r % n); r /= n;
    const int c = (int)r * 2 + h;
    const int eg = elem[tl * NE + e];
    Wt[id] = (eg >= 0) ? W[c * nloc + (int64_t)eg * n * NN + ij * n + k] : 0.0;
  }
}

// Minv in tile order: Mt[t][l][node] = Minv[gt[t][l][node]] (0 for absent nodes / padding).
__global__ void tile_pack_minv_kernel(int64_t rows, int gts, int mts, const int32_t* __restrict__ gt,
                                      const double* __restrict__ Minv, double* __restrict__ Mt) {
  const int64_t total = rows * mts;
  for (int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; id < total; id += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = id / mts;
    const int c = (int)(id % mts);
    const int g = (c < gts) ? gt[r * gts + c] : -1;
    Mt[id] = (g >= 0) ? Minv[g] : 0.0;
  }
}

template <int n, int TX, int TY, int F>
int run_tile(const TileArgs& A, const double* Drow, cudaStream_t st) {
  constexpr int FP = (F % 2 == 0 && n < HV_FP2_MAXN) ? 2 : 1;
  using C = TileCfg<n, TX, TY, F, FP>;
  hv::DTab<n> Dt;
  hv::fill_dtab(Dt, Drow);
  auto kern = lap_tile_kernel<n, TX, TY, F, FP, C::MINB>;
  HV_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
  if (A.tile1 <= A.tile0) return HV_OK;
  kern<<<(unsigned)(A.tile1 - A.tile0), C::NT, C::SMEM, st>>>(Dt, A);
  HV_LAUNCH_CHECK();
  return HV_OK;
}

}  // namespace

namespace hv {

namespace {
template <int n, int TX, int TY, int F>
constexpr bool fits() {
  return TileCfg<n, TX, TY, F, (F % 2 == 0 && n < HV_FP2_MAXN) ? 2 : 1>::SMEM <= 227 * 1024;
}
template <int n, int TX, int TY>
bool fits_f(int F) {
  return (F == 1) ? fits<n, TX, TY, 1>() : (F == 4) ? fits<n, TX, TY, 4>() : fits<n, TX, TY, 5>();
}
}  // namespace

bool tile_supported(int N, int TX, int TY, int F) {
  if (F != 1 && F != 4 && F != 5) return false;
  if (N == 7) return TX == 1 && TY == 1 && fits_f<8, 1, 1>(F);
  if (!(N >= 1 && N <= 6 && TX == 2 && TY == 2)) return false;
  switch (N) {   // shared memory of the instantiation must fit one SM (227 KB)
    case 1: return fits_f<2, 2, 2>(F);
    case 2: return fits_f<3, 2, 2>(F);
    case 3: return fits_f<4, 2, 2>(F);
    case 4: return fits_f<5, 2, 2>(F);
    case 5: return fits_f<6, 2, 2>(F);
    default: return fits_f<7, 2, 2>(F);
  }
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
  HV_TILE_CASE(7, 1, 1)
#undef HV_TILE_CASE
  HV_FAIL(HV_ERR_UNSUPPORTED, "tile kernel: no instantiation for N=%d TX=%d TY=%d F=%d", N, A.TX, A.TY, F);
}

int tile_pack(int N, int NE, int64_t ntiles, int nlay, const int32_t* elem, const double* W, int64_t nloc,
              double* Wt, cudaStream_t st) {
  tile_pack_metric<<<148 * 8, 256, 0, st>>>(N + 1, NE, ntiles, nlay, elem, W, nloc, Wt);
  HV_LAUNCH_CHECK();
  return HV_OK;
}

int tile_pack_minv(int64_t rows, int gts, int mts, const int32_t* gt, const double* Minv, double* Mt, cudaStream_t st) {
  tile_pack_minv_kernel<<<148 * 8, 256, 0, st>>>(rows, gts, mts, gt, Minv, Mt);
  HV_LAUNCH_CHECK();
  return HV_OK;
}

}  // namespace hv
