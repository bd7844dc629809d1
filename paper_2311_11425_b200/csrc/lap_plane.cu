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

__device__ __forceinline__ void st_v2(double* p, double a, double b) {
  *reinterpret_cast<double2*>(p) = make_double2(a, b);
}
__device__ __forceinline__ double2 ldg_stream2(const double* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}

// WV: where the packed metric comes from in step c.
//   0  TMA bulk copy of the tile-layer block into shared memory (mbarrier)
//   1  straight from global memory (L2-prefetched one layer ahead), no shared staging
// H: plane split.  H = 1: a thread owns the whole (xi, zeta) plane of its (element, eta
// index, field).  H = 2 (N = 7: a 64-node plane does not fit in registers): the plane's xi
// rows are split over two lanes (ih = 0, 1) that exchange the other half of every xi line
// with warp shuffles; the eta lines of the line-owner role are split by zeta halves.
// WF: form of the packed metric.  0: the 6 components of W as 3 pairs; 1: axis form (scaled
// mode with c_1 == c_2): u = sqrt(w3 Jg) e_3 (3 doubles per node), W d = kh |u|^2 d + kd u (u . d);
// 2: isotropic form (c_1 == c_2 == c_3): s = kh w3 Jg (1 double per node), W d = s d.
template <int n, int TX, int TY, int F, int WV, int H = 1, int WF = 0, int IO = 0>
struct PlaneCfg {
  static constexpr int N = n - 1;
  static constexpr int U = TX * N + 1, V = TY * N + 1, UV = U * V;
  static constexpr int NE = TX * TY;
  static constexpr int NR = n / H, NK = n / H;           // xi rows / eta-line zeta levels per thread
  static constexpr int NP = NE * n * F * H;              // plane threads: (eta plane, element, half, field)
  static constexpr int NT = (NP + 31) & ~31;             // + helper lanes filling the last warp (gather / output)
  static constexpr int NODES = UV * n;
  static constexpr int GTS = (NODES + 3) & ~3;
  static constexpr int MTS = (NODES + 1) & ~1;
  // field-major (SoA) shared arrays with padded strides.  For the production shape (n = 5,
  // 2x2 tiles, thread order (jp, e, f)) the strides come from an exhaustive bank-conflict
  // search (tools/bank_search.py): every plane / eta-line access of a half-warp then hits
  // 16 distinct 8-byte banks.  Other shapes use the plain padded layout.
  static constexpr bool TUNED = (n == 5 && TX == 2 && TY == 2 && H == 1);
  // N = 7 single-column tiles, H = 4 (tools/bank_search_n7.py, half-warp model: ~2x fewer wavefronts than plain)
  static constexpr bool TUNED7 = (n == 8 && TX == 1 && TY == 1 && H == 4 && F == 4);
  static constexpr int pad16(int x) { return x + ((4 - (x % 16)) + 16) % 16; }
  static constexpr int KS = n;                                   // node column (k) stride
  static constexpr int US = TUNED ? 46 : TUNED7 ? 66 : V * n;    // u stride of s_q
  static constexpr int QP = TUNED ? 415 : TUNED7 ? 529 : pad16(NODES);   // s_q field-plane stride
  static constexpr int BS = n;                                   // scratch: [f][e][a][b][c]
  static constexpr int AS = TUNED ? 28 : TUNED7 ? 66 : n * n;
  static constexpr int ES = TUNED ? 147 : TUNED7 ? 529 : n * n * n;
  static constexpr int SP = TUNED ? 588 : TUNED7 ? 529 : pad16(NE * n * n * n);
  // isotropic metric (WF 2): [i][k][e][j] with an i-row stride padded where tuned
  // (the packing must agree for every kernel variant of the shape: keyed on n and the tile only)
  static constexpr int MIS = NE * n * n + ((n == 8 && TX == 1 && TY == 1) ? 1 : 0);
  static constexpr int SQ = QP * F;
  static constexpr int SE = SP * F;
  static constexpr int WL = WF == 2 ? n * MIS : (WF == 1 ? 3 : 6) * n * NE * n * n;   // packed metric doubles per tile-layer
  // the bulk copy of a tile-layer's metric moves a multiple of 16 bytes (else its mbarrier never completes)
  static_assert(WV != 0 || WL % 2 == 0, "packed metric per tile-layer must be a multiple of 16 bytes");
  static constexpr int PN = (NODES + NT - 1) / NT;       // gather node items per thread
  static constexpr int FI = UV * N;                      // output items per layer (k < N)
  static constexpr int PF = (FI + NT - 1) / NT;          // output items per thread
  // tile-ordered intermediate (IO 1 writes it, IO 2 reads it): one block per tile-layer, level-major
  // [k < N][f][u][v] (block nlay: the top level of the columns, k = 0).  A half-warp's lanes vary
  // (f, e) in the plane and eta-line reads: field stride = 1 (mod 4) and u stride = 2 (mod 4) put
  // them on 16 distinct 8-byte banks (f*YFS + px*N*YUS + py*N spans 0..15 mod 16 at N = 4).  A
  // level of all fields is whole 16-byte units, so levels 1..N-1 and a level 0 are single bulk copies.
  static constexpr int YUS = V + ((2 - V % 4) + 4) % 4;
  static constexpr int YFS = U * YUS + ((1 - (U * YUS) % 4) + 4) % 4;
  static constexpr int YLS = F * YFS + (F * YFS) % 2;
  static constexpr int YBLK = N * YLS;
  static constexpr int FIY = N * UV;                     // block items per layer, (k, u, v) order
  static constexpr int PFY = (FIY + NT - 1) / NT;
  // perimeter column nodes of a tile (shared with other tiles): their final values come from the
  // slot fix-up's compact (slot, z, F) rows, staged per layer (levels 1..N of the layer; the
  // prologue stages levels 0..N) and patched into the level buffers
  static constexpr int NPER = 2 * V + 2 * (U - 2);
  // shared memory (doubles): q (IO 2: levels 1..N-1 | level 0 ring [2] | perimeter stage) | W (WV 0) |
  // scratch | ctab (int4) | code | mbarriers (metric, IO 2 loads)
  static constexpr int QB_L0 = (N - 1) * YLS;            // IO 2: the two level-0 planes
  static constexpr int QB_S = QB_L0 + 2 * YLS;           // IO 2: perimeter stage [NPER][N][F]
  // IO 3 (pass 1 with bulk-copied input, tiles.build_chunk_table): the state's (nglobal, 5) rows of
  // levels 1..N in a row buffer (whole rows, runs of consecutive gids), level 0 in two planes laid
  // out like a Yt level [f][u][v]
  static constexpr int CRR = 392;                        // row-buffer rows (the table places <= 390)
  static constexpr int QB_P = CRR * 5;                   // IO 3: the two level-0 planes
  static constexpr int TCW = UV + 1 + 4 * 32;            // IO 3: ints per tile of TileArgs::tchunk
  static constexpr int SQB = IO == 2 ? QB_S + NPER * N * F : (IO == 3 ? QB_P + 2 * YLS : SQ);
  static constexpr int TPW = NPER + 3 * 32;              // IO 2: ints per tile of TileArgs::tper
  static constexpr int OFF_W = (SQB + 1) & ~1;
  static constexpr int OFF_S = OFF_W + (WV == 0 ? WL : 0);
  static constexpr int OFF_T = (OFF_S + SE + 1) & ~1;
  static constexpr int OFF_C = OFF_T + 2 * UV;
  static constexpr int OFF_P = OFF_C + (UV + 1) / 2;
  static constexpr int OFF_PD = OFF_P + (UV + 1) / 2;  // IO 2: [NPER] level offset of the stage's slot columns
  static constexpr int OFF_BAR = (OFF_PD + (IO == 2 ? (NPER + 1) / 2 : (IO == 3 ? (UV + 1) / 2 : 0)) + 1) & ~1;
  // split planes (H > 1): D in shared memory for the xi exchange, whose row / column offsets vary
  // across the lanes of a warp (constant-bank loads would serialise)
  static constexpr int OFF_D = OFF_BAR + 4;
  // split planes writing the tile-ordered intermediate (N = 7: shared memory is not what bounds the CTAs per
  // SM): the block's padding positions as a table, so that the per-layer zeroing is a load and a store per item
  static constexpr int PADN = N * F * (U * (YUS - V) + YFS - U * YUS);
  static constexpr bool PADTAB = H > 1 && (IO == 1 || IO == 3);
  static constexpr int OFF_PT = OFF_D + (H > 1 ? n * n : 0);
  static constexpr size_t SMEM = sizeof(double) * (OFF_PT + (PADTAB ? (PADN + 1) / 2 : 0));
};

// Wp layout (per tile-layer): [cp 3][i n][k n][e NE][j n][2] (component pairs (w00,w01)
// (w02,w11) (w12,w22)); the F field lanes of a plane read one 16-byte pair together.
//
// Node items: thread tid handles the tile nodes tid + it*NT (it < PN) in the gather of the
// next layer and in the final node-owner step; their gids live in registers (loaded one
// layer ahead, coalesced from the tile-ordered map), Minv is read coalesced at step e.
// AB: ablation bit mask for development timing only (0 in production): 1 = no node-owner
// step (f), 2 = no q gather, 4 = no metric TMA, 8 = no plane arithmetic (steps b-e)
// OM: output rows, fixed at compile time for the hot passes (smaller code): 0 = any (runtime
// checks below), 1 = (ng, 4) rows of fields 0..3 written, 2 = (ng, 5) rows of fields 1..4 written
// with column 0 zeroed (H_nu's second pass)
// IO: 0 = q gathered by gid and results written to (nglobal, ld) rows; 1 = results written to the
// tile-ordered intermediate at A.out (final values for tile-owned nodes, raw partial sums for the
// perimeter nodes other tiles share: slot_fixup_yt completes them in place); 2 = q read from the
// tile-ordered intermediate at A.q, one bulk copy per tile-layer block into a two-slot ring
template <int n, int TX, int TY, int F, int WV, int MB, int AB = 0, int H = 1, int WF = 0, int OM = 0, int IO = 0>
__global__ void __launch_bounds__(PlaneCfg<n, TX, TY, F, WV, H, WF, IO>::NT, MB) lap_plane_kernel(hv::DTabEO<n> Dt, TileArgs A) {
  using C = PlaneCfg<n, TX, TY, F, WV, H, WF, IO>;
  static_assert(IO == 0 || (F == 4 && (H == 1 || IO != 3) && (AB == 0 || (IO == 1 && AB == 2))),
                "tile-ordered intermediate: 4 fields (split planes: no bulk-copied pass-1 input)");
  constexpr bool OUT_YT = (IO == 1 || IO == 3);   // results into the tile-ordered intermediate
  constexpr bool GATHER = (IO == 0 || IO == 1);   // q gathered by gid every layer (IO 3: layer 0 only)
  // line contractions held whole in a thread's registers (zeta, eta; xi too for whole planes, H = 1)
  // in the even-odd form (DTabEO); step d then stores -D^T sums and step e adds them
  constexpr bool EO = true;
  constexpr int N = C::N, U = C::U, V = C::V, NE = C::NE, UV = C::UV, PN = C::PN, PF = C::PF, NR = C::NR, NK = C::NK;
  extern __shared__ __align__(16) double sm[];
  double* s_q = sm;                                    // [F][QP] gathered q of the current layer
  double* s_w = sm + C::OFF_W;                         // metric of the current layer (WV 0, TMA)
  double* s_s = sm + C::OFF_S;                         // [F][NE][n i][n j][n k] eta scratch / element acc
  int4* s_ct = reinterpret_cast<int4*>(sm + C::OFF_T); // [UV] element-copy offsets
  int* s_code = reinterpret_cast<int*>(sm + C::OFF_C); // [UV] partial row or -1
  int* s_perm = reinterpret_cast<int*>(sm + C::OFF_P); // [UV] output column order: tile-owned first
  int* s_pdst = reinterpret_cast<int*>(sm + C::OFF_PD);  // IO 2: [stage position] u * YUS + v of the slot column
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + C::OFF_BAR);  // [0] metric stage (WV 0), [1] IO 2 loads
  double* sD = sm + C::OFF_D;                          // [n][n] (H > 1)
  const int tid = threadIdx.x;
  const int f = tid % F;
  const int ih = (tid / F) % H;       // thread order (jp, e, ih, f): f fastest (metric pairs broadcast),
  const int e = (tid / (F * H)) % NE; // the two halves of a plane in lanes 4 apart (shuffle partner)
  const int jp = min(tid / (F * H * NE), n - 1);
  const int I0 = ih * NR, K0 = ih * NK;
  const int px = e / TY, py = e % TY;
  const int nlay = A.nlay;
  // vertical segments (IO 0): CTA = (tile, segment of A.seg layers) sweeping layers [l0, l1)
  const int nseg = (IO == 0 && A.seg > 0) ? (nlay + A.seg - 1) / A.seg : 1;
  const int64_t t = A.tile0 + blockIdx.x / nseg;
  const int sg = blockIdx.x % nseg;
  const int l0 = (nseg > 1) ? sg * A.seg : 0, l1 = (nseg > 1) ? min(nlay, l0 + A.seg) : nlay;
  const int tx = A.tmeta[2 * t], ty = A.tmeta[2 * t + 1];
  const bool pth = tid < C::NP;       // plane thread (the rest: helper lanes for the node-granular steps)
  const bool act = pth && (px < tx) && (py < ty);
  const int32_t* gt_t = A.gt + t * (int64_t)nlay * C::GTS;
  const double* Wt_t = A.Wt + t * (int64_t)nlay * C::WL;
  const double* Mt_t = A.Mt + t * (int64_t)nlay * C::MTS;
  int qcol[F], ocol[F];
#pragma unroll
  for (int p = 0; p < F; ++p) {
    qcol[p] = A.qf.f[p];
    ocol[p] = A.of.f[p];
  }
  int myqc = qcol[0];   // the thread's field column in a q row
#pragma unroll
  for (int p = 1; p < F; ++p)
    if (p == f) myqc = qcol[p];
  const bool row5 = (F == 4 && A.ldo == 5 && A.zero_mask == 1u && ocol[0] == 1 && ocol[1] == 2 && ocol[2] == 3 && ocol[3] == 4);
  auto sidx = [&](int ee, int a, int b, int c) { return f * C::SP + ee * C::ES + a * C::AS + b * C::BS + c; };
  auto tq = [&](int u, int v, int k) { return f * C::QP + u * C::US + v * C::KS + k; };
  // tile node (uv * n + k) -> s_q offset within a field plane
  auto qnode = [&](int node) { const int uv = node / n; return (uv / V) * C::US + (uv % V) * C::KS + node % n; };

  auto load_gids = [&](int l, int (&g)[PN]) {
#pragma unroll
    for (int it = 0; it < PN; ++it) {
      const int node = tid + it * C::NT;
      g[it] = (node < C::NODES) ? __ldg(gt_t + (int64_t)l * C::GTS + node) : -1;
    }
  };
  // node-granular async gather of one layer of q (all F fields of a node per item)
  auto issue_gather = [&](const int (&g)[PN]) {
    if (AB & 2) return;
#pragma unroll
    for (int it = 0; it < PN; ++it) {
      const int node = tid + it * C::NT;
      if (node < C::NODES) {
        if constexpr (IO == 3) {   // layer 0: level 0 -> plane 0, levels >= 1 -> their rows of the buffer
          const int uv = node / n, k = node % n;
          const double* src = A.q + (int64_t)g[it] * A.ldq;
#pragma unroll
          for (int p = 0; p < F; ++p)
            cp_async8(k == 0 ? s_q + C::QB_P + p * C::YFS + (uv / V) * C::YUS + uv % V
                             : s_q + (s_pdst[uv] + k - 1) * 5 + qcol[p], src + qcol[p]);
        } else if (g[it] < 0) {
#pragma unroll
          for (int p = 0; p < F; ++p) s_q[p * C::QP + qnode(node)] = 0.0;
        } else {
          const double* src = A.q + (int64_t)g[it] * A.ldq;
          const int qo = qnode(node);
#pragma unroll
          for (int p = 0; p < F; ++p) cp_async8(s_q + p * C::QP + qo, src + qcol[p]);
        }
      }
    }
    cp_async_commit();
  };
  const int64_t chain = (int64_t)(nlay + 1) * C::YBLK;
  // IO 2: the tile's slot columns (perimeter columns other tiles share), staged in slot order: run r of
  // consecutive slots (lane r of warp 0: first slot, count, first stage position); nper = their number
  const int32_t* tper = A.tper + t * C::TPW;
  int r_start = 0, r_cnt = 0, r_pos = 0, nper = 0;
  if constexpr (IO == 2) {
    if (tid < 32) {
      r_start = tper[C::NPER + 3 * tid];
      r_cnt = tper[C::NPER + 3 * tid + 1];
      r_pos = tper[C::NPER + 3 * tid + 2];
    }
    for (int j = 0; j < C::NPER; ++j) nper += (tper[j] >= 0) ? 1 : 0;
  }
  // IO 2 loads of layer l: levels 1..N-1 of block l -> s_q, level 0 of block l+1 -> level-0 plane
  // (l+1)&1, the slot rows of levels z = l*N+1 .. l*N+N (slot-row block l: [slot][N][F]) -> the stage;
  // l = -1 (prologue): level 0 of block 0 -> plane 0, slot rows of z = 0 -> the stage.  One mbarrier
  // phase, issued by warp 0 (lane r: run r of consecutive slots).
  auto issue_loads = [&](int l, int nper) {
    const int lane = tid & 31;
    const int nlev = (l < 0) ? 1 : N;
    if (lane == 0) {
      const uint32_t bytes = (uint32_t)((l < 0 ? 1 : N) * C::YLS * 8 + nper * nlev * F * 8);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar + 1)), "r"(bytes)
                   : "memory");
      const double* base = A.q + t * chain;
      if (l < 0) {
        tma_copy(s_q + C::QB_L0, base, C::YLS * 8, bar + 1);                              // block 0, level 0
      } else {
        tma_copy(s_q, base + (int64_t)l * C::YBLK + C::YLS, (N - 1) * C::YLS * 8, bar + 1);
        tma_copy(s_q + C::QB_L0 + ((l + 1) & 1) * C::YLS, base + (int64_t)(l + 1) * C::YBLK, C::YLS * 8, bar + 1);
      }
    }
    if (r_cnt > 0) {
      const double* src = (l < 0) ? A.sv + (int64_t)r_start * F
                                  : A.sv + A.nslot * F + ((int64_t)l * A.nslot + r_start) * N * F;
      tma_copy(s_q + C::QB_S + r_pos * nlev * F, src, (uint32_t)(r_cnt * nlev * F * 8), bar + 1);
    }
  };
  // IO 3: lane r of warp 0 holds run r of the tile's chunk table (gid at layer 1, gid stride per
  // layer, rows, row-buffer position); a layer l >= 1 is one bulk copy per run (16-byte aligned ends:
  // a run starting at an odd gid moves 8 bytes before its first row too; the table keeps one spare
  // row between runs)
  int c_g1 = 0, c_st = 0, c_rows = 0, c_dst = 0;
  if constexpr (IO == 3) {
    const int32_t* tc = A.tchunk + t * C::TCW;
    if (tid < 32 && tid < tc[UV]) {
      c_g1 = tc[UV + 1 + 4 * tid];
      c_st = tc[UV + 2 + 4 * tid];
      c_rows = tc[UV + 3 + 4 * tid];
      c_dst = tc[UV + 4 + 4 * tid];
    }
  }
  int64_t c_tail = -1;   // IO 3: gid of a run's last row that a bulk copy would overrun (the end of q)
  auto issue_chunks = [&](int l) {
    const int64_t g = (int64_t)c_g1 + (int64_t)c_st * (l - 1);
    const uint32_t shift = (uint32_t)(g & 1) * 8u;
    uint32_t bytes = c_rows ? ((c_rows * 40u + shift + 15u) & ~15u) : 0u;
    if (c_rows && g * 40 - shift + bytes > A.ng * 40) {                  // the last rows of q: the
      bytes = ((c_rows - 1) * 40u + shift + 15u) & ~15u;                  // final row loaded at step a
      c_tail = g + c_rows - 1;
    }
    const uint32_t tot = __reduce_add_sync(0xffffffffu, bytes);
    if (tid == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar + 1)), "r"(tot)
                   : "memory");
    if (bytes)
      tma_copy(reinterpret_cast<char*>(s_q) + c_dst * 40 - shift,
               reinterpret_cast<const char*>(A.q) + g * 40 - shift, bytes, bar + 1);
  };
  // IO 2: stage -> level buffers (layer l: levels 1..N; prologue: level 0 -> plane 0); an item =
  // (stage position j, level kk): its F fields in two 16-byte loads, stored at the column's offset
  auto patch = [&](int l, int nper) {
    const int nit = (l < 0) ? nper : nper * N;
    for (int x = tid; x < nit; x += C::NT) {
      const int j = (l < 0) ? x : x / N, kk = (l < 0) ? 0 : 1 + x % N;
      const int o = s_pdst[j];
      const double* src = s_q + C::QB_S + ((l < 0) ? j : j * N + kk - 1) * F;
      const double2 a = *reinterpret_cast<const double2*>(src);
      const double2 b = *reinterpret_cast<const double2*>(src + 2);
      double* dst = (kk == 0) ? s_q + C::QB_L0
                              : (kk == N ? s_q + C::QB_L0 + ((l + 1) & 1) * C::YLS : s_q + (kk - 1) * C::YLS);
      dst[o] = a.x;
      dst[o + C::YFS] = a.y;
      dst[o + 2 * C::YFS] = b.x;
      dst[o + 3 * C::YFS] = b.y;
    }
  };
  // q at tile node (u, v, k) of the current layer (IO 2: level 0 from plane l&1, levels 1..N-1 from
  // the level buffer, the top level k = N from plane (l+1)&1)
  auto qrd = [&](const double* lo, const double* hi, int u, int v, int k) -> double {
    if constexpr (IO == 2) {
      const int o = f * C::YFS + u * C::YUS + v;
      return (k == 0) ? lo[o] : (k == N ? hi[o] : s_q[(k - 1) * C::YLS + o]);
    } else if constexpr (IO == 3) {
      return (k == 0) ? lo[f * C::YFS + u * C::YUS + v] : s_q[(s_pdst[u * V + v] + k - 1) * 5 + myqc];
    } else {
      return s_q[tq(u, v, k)];
    }
  };
  // sum of the (up to four) element copies of a tile node, fixed order (c0 + c1) + (c2 + c3)
  auto csum = [&](const int4 ct, const double* sp) -> double {
    const double c0 = sp[ct.x];
    const double c1 = (ct.y >= 0) ? sp[ct.y] : 0.0;
    const double c2 = (ct.z >= 0) ? sp[ct.z] : 0.0;
    const double c3 = (ct.z >= 0) ? sp[ct.w] : 0.0;
    return (c0 + c1) + (c2 + c3);
  };
  auto issue_metric = [&](int l) {
    if (AB & 4) return;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(C::WL * 8)
                 : "memory");
    tma_copy(s_w, Wt_t + (int64_t)l * C::WL, C::WL * 8, bar);
  };

  // one output item: final value scale * Minv * sum (row store, 16-byte stores where the row
  // alignment allows) or the raw sum into the item's partial row (perimeter slot)
  const bool vec4 = (F == 4 && A.ldo == 4 && !A.accumulate && !A.zero_mask && ocol[0] == 0 && ocol[1] == 1 &&
                     ocol[2] == 2 && ocol[3] == 3);
  auto emit = [&](int g, double mi, hv::Vec<F> val, int cd, int z) {
    if (cd < 0) {
      double* o = A.out + (int64_t)g * A.ldo;
      const double m = A.scale * mi;
      if constexpr (F == 4 && OM == 1) {
        st_v2(o, m * val.v[0], m * val.v[1]);
        st_v2(o + 2, m * val.v[2], m * val.v[3]);
        return;
      } else if constexpr (F == 4 && OM == 2) {   // parity-selected offsets (see the row5 path below)
        const bool odd = (g & 1) != 0;
        const double v0 = m * val.v[0], v1 = m * val.v[1], v2 = m * val.v[2], v3 = m * val.v[3];
        o[odd ? 0 : 4] = odd ? 0.0 : v3;
        st_v2(o + (odd ? 1 : 0), odd ? v0 : 0.0, odd ? v1 : v0);
        st_v2(o + (odd ? 3 : 2), odd ? v2 : v1, odd ? v3 : v2);
        return;
      }
      if constexpr (F == 4) {
        if (vec4) {
          st_v2(o, m * val.v[0], m * val.v[1]);
          st_v2(o + 2, m * val.v[2], m * val.v[3]);
          return;
        }
        if (row5 && !A.accumulate) {
          // row (0, v0, v1, v2, v3) of 40 bytes: 16-byte aligned when g is even, 8 bytes past that when odd --
          // one 8-byte and two 16-byte stores with parity-selected offsets (no divergent branch)
          const bool odd = (g & 1) != 0;
          const double v0 = m * val.v[0], v1 = m * val.v[1], v2 = m * val.v[2], v3 = m * val.v[3];
          o[odd ? 0 : 4] = odd ? 0.0 : v3;
          st_v2(o + (odd ? 1 : 0), odd ? v0 : 0.0, odd ? v1 : v0);
          st_v2(o + (odd ? 3 : 2), odd ? v2 : v1, odd ? v3 : v2);
          return;
        }
      }
      if (A.accumulate) {
#pragma unroll
        for (int p = 0; p < F; ++p) o[ocol[p]] += m * val.v[p];
      } else {
#pragma unroll
        for (int p = 0; p < F; ++p) o[ocol[p]] = m * val.v[p];
        if (A.zero_mask)
          for (int zc = 0; zc < A.ldo; ++zc)
            if ((A.zero_mask >> zc) & 1u) o[zc] = 0.0;
      }
    } else {
      const int64_t r = (int64_t)cd * A.n_z + z;
      double* o = A.part + r * F;                       // partial rows: F doubles
      if constexpr (F == 4) {
        st_v2(o, val.v[0], val.v[1]);
        st_v2(o + 2, val.v[2], val.v[3]);
      } else {
#pragma unroll
        for (int p = 0; p < F; ++p) o[p] = val.v[p];
      }
    }
  };

  int gcur[PN], gnext[PN];
  if constexpr (IO != 2) load_gids(l0, gcur);   // IO 3: layer 0 is gathered
  if (WV == 0 && tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  if ((IO == 2 || IO == 3) && tid == 0) {
    mbar_init(bar + 1, 1);
    fence_mbar_init();
  }
  if constexpr (IO == 2)
    for (int j = tid; j < C::NPER; j += C::NT) s_pdst[j] = tper[j];
  if constexpr (IO == 3)   // s_pdst: the row of level 1 of each tile column in the row buffer
    for (int j = tid; j < UV; j += C::NT) s_pdst[j] = A.tchunk[t * C::TCW + j];
  if (WV == 1 && tid == 0) l2_prefetch(Wt_t, C::WL * 8);
  for (int uv = tid; uv < UV; uv += C::NT) {
    const int u = uv / V, v = uv % V;
    const int pu1 = min(u / N, TX - 1), pv1 = min(v / N, TY - 1);
    const int pu0 = (u % N == 0 && u > 0) ? u / N - 1 : pu1;
    const int pv0 = (v % N == 0 && v > 0) ? v / N - 1 : pv1;
    int o[4] = {-1, -1, -1, -1}, c = 0;
    for (int a = pu0; a <= pu1; ++a)
      for (int b = pv0; b <= pv1; ++b) o[c++] = (a * TY + b) * C::ES + (u - a * N) * C::AS + (v - b * N) * C::BS;
    s_ct[uv] = make_int4(o[0], o[1], o[2], o[3]);
    s_code[uv] = A.code[t * UV + uv];
  }
  if constexpr (IO == 3) __syncthreads();   // s_pdst before the layer-0 gather uses it
  if constexpr (IO != 2) {
    issue_gather(gcur);
    if (GATHER && l0 + 1 < l1) load_gids(l0 + 1, gnext);
  }
  if constexpr (H > 1)
    for (int x = tid; x < n * n; x += C::NT) sD[x] = Dt.D[x / n][x % n];
  int* s_pad = reinterpret_cast<int*>(sm + C::OFF_PT);   // PADTAB: offsets of the block's padding doubles
  if constexpr (C::PADTAB) {
    constexpr int PV = C::YUS - V, PT = C::YFS - U * C::YUS, PP = U * PV + PT;
    for (int x = tid; x < C::PADN; x += C::NT) {
      const int kf = x / PP, j = x - kf * PP;
      s_pad[x] = (kf / F) * C::YLS + (kf % F) * C::YFS + ((j < U * PV) ? (j / PV) * C::YUS + V + j % PV : U * C::YUS + j - U * PV);
    }
  }
  __syncthreads();
  if (tid == 0) {   // output items walk the tile-owned columns first (uniform warps in step f)
    int c = 0;
    for (int pass = 0; pass < 2; ++pass)
      for (int uv = 0; uv < UV; ++uv)
        if ((s_code[uv] < 0) == (pass == 0)) s_perm[c++] = uv;
  }
  __syncthreads();
  if (WV == 0 && tid == 0) issue_metric(l0);
  if constexpr (IO == 2) {   // prologue: level 0 of block 0 (+ its perimeter rows); then layer 0's loads
    if (tid < 32) issue_loads(-1, nper);
    mbar_wait(bar + 1, 0);
    patch(-1, nper);
    __syncthreads();
    if (tid < 32) {
      fence_proxy_async();
      issue_loads(0, nper);
    }
  }
  // IO 3: the row-buffer address of level 0 of the thread's plane rows (u = px*N + r) and eta lines
  // (v = py*N + a) minus one row: level k >= 1 of them is at + 5 k (layer-invariant)
  int prow[IO == 3 ? n : 1], erow[IO == 3 ? n : 1];
  if constexpr (IO == 3) {
#pragma unroll
    for (int r = 0; r < n; ++r) {
      prow[r] = (s_pdst[(px * N + r) * V + py * N + jp] - 1) * 5 + myqc;
      erow[r] = (s_pdst[(px * N + jp) * V + py * N + r] - 1) * 5 + myqc;
    }
  }
  double carry[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) carry[r] = 0.0;
  // H = 2: inactive elements of ragged tiles run the plane steps on zeros so that shuffle
  // partners stay converged (their scratch is zeroed in step e)
  const bool run = (H == 1) ? act : pth;

  for (int l = l0; l < l1; ++l) {
    // ---- a: q(l) has landed
    if constexpr (IO == 2) {   // layer l's loads (levels 1..N-1, level 0 of block l+1, perimeter rows)
      mbar_wait(bar + 1, (uint32_t)((l + 1) & 1));
      patch(l, nper);
    } else if constexpr (IO == 3) {   // layer 0 gathered, then one bulk-copy phase per layer
      if (l == 0) {
        cp_async_wait_all();
      } else {
        mbar_wait(bar + 1, (uint32_t)((l - 1) & 1));
        if (c_tail >= 0) {   // the row at the end of q (after the bulk copy, which ends before it)
#pragma unroll
          for (int ff = 0; ff < 5; ++ff) s_q[(c_dst + c_rows - 1) * 5 + ff] = A.q[c_tail * 5 + ff];
          c_tail = -1;
        }
      }
    } else {
      cp_async_wait_all();
    }
    __syncthreads();
    const double* sq_lo = s_q + (IO == 3 ? C::QB_P : C::QB_L0) + (l & 1) * C::YLS;
    const double* sq_hi = s_q + (IO == 3 ? C::QB_P : C::QB_L0) + ((l + 1) & 1) * C::YLS;
    if (WV == 1 && tid == 0 && l + 1 < l1) l2_prefetch(Wt_t + (int64_t)(l + 1) * C::WL, C::WL * 8);
    if (tid == C::NT - 1 && l + 1 < l1) {   // output-item gid / Minv of the next layer -> L2
      l2_prefetch(Mt_t + (int64_t)(l + 1) * C::MTS, C::MTS * 8);
      if (!OUT_YT) l2_prefetch(gt_t + (int64_t)(l + 1) * C::GTS, C::GTS * 4);
    }
    // ---- b: plane derivatives in registers, eta lines (i = jp) strong
    double p0[NR][n], p2[NR][n];   // [row][k]: dq_xi, dq_zeta -> f_xi, f_zeta -> accumulator
    if (run && !(AB & 8)) {
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        double ql[n];
#pragma unroll
        for (int k = 0; k < n; ++k)
          ql[k] = (IO == 3 && k > 0) ? s_q[prow[IO == 3 ? r : 0] + 5 * k] : qrd(sq_lo, sq_hi, px * N + I0 + r, py * N + jp, k);
        if constexpr (EO) {
          hv::eo_mv<n, 0>(Dt, ql, p2[r]);
        } else {
#pragma unroll
          for (int k = 0; k < n; ++k) {
            double s = 0.0;
#pragma unroll
            for (int a = 0; a < n; ++a) s = fma(Dt.D[k][a], ql[a], s);
            p2[r][k] = s;
          }
        }
#pragma unroll
        for (int k = 0; k < n; ++k) p0[r][k] = ql[k];   // q plane, xi-differentiated below
        if constexpr (IO == 3) {
          // level N of layer l is level 0 of layer l + 1: the plane owners hold it, so they fill plane
          // (l+1)&1 (unused during layer l) before the row buffer is refilled -- the tile's 81 columns
          // are the union of the elements' plane rows (shared edges written twice, same value)
          if (l + 1 < nlay)
            s_q[C::QB_P + ((l + 1) & 1) * C::YLS + f * C::YFS + (px * N + I0 + r) * C::YUS + py * N + jp] = ql[N];
        }
      }
#pragma unroll
      for (int k = 0; k < n; ++k) {
        if constexpr (H == 1) {
          double ql[n], yl[n];
#pragma unroll
          for (int i = 0; i < n; ++i) ql[i] = p0[i][k];
          hv::eo_mv<n, 0>(Dt, ql, yl);
#pragma unroll
          for (int i = 0; i < n; ++i) p0[i][k] = yl[i];
        } else {
          // own rows, then the other H - 1 blocks of the xi line from the shuffle partners
          double co[NR], cp[H - 1][NR];
#pragma unroll
          for (int r = 0; r < NR; ++r) co[r] = p0[r][k];
#pragma unroll
          for (int m = 1; m < H; ++m)
#pragma unroll
            for (int r = 0; r < NR; ++r) cp[m - 1][r] = __shfl_xor_sync(0xffffffffu, co[r], F * m);
#pragma unroll
          for (int r = 0; r < NR; ++r) {
            double s = 0.0;
#pragma unroll
            for (int a = 0; a < NR; ++a) s = fma(sD[(I0 + r) * n + I0 + a], co[a], s);
#pragma unroll
            for (int m = 1; m < H; ++m) {
              const int pb = (ih ^ m) * NR;
#pragma unroll
              for (int a = 0; a < NR; ++a) s = fma(sD[(I0 + r) * n + pb + a], cp[m - 1][a], s);
            }
            p0[r][k] = s;
          }
        }
      }
      // eta lines of element e: H = 1: lines i = jp, all zeta levels; split planes: lines
      // i = I0 .. I0 + NK at level k = jp (the lanes of a half-warp then vary i, as in the plane
      // accesses, whose layout is bank-conflict-free): dq_eta(e, i, a', k)
#pragma unroll
      for (int kk = 0; kk < NK; ++kk) {
        const int li = (H == 1) ? jp : I0 + kk, k = (H == 1) ? K0 + kk : jp;
        double ql[n];
#pragma unroll
        for (int a = 0; a < n; ++a)
          ql[a] = (IO == 3 && k > 0) ? s_q[erow[IO == 3 ? a : 0] + 5 * k] : qrd(sq_lo, sq_hi, px * N + li, py * N + a, k);
        if constexpr (EO) {
          double yl[n];
          hv::eo_mv<n, 0>(Dt, ql, yl);
#pragma unroll
          for (int a2 = 0; a2 < n; ++a2) s_s[sidx(e, li, a2, k)] = yl[a2];
        } else {
#pragma unroll
          for (int a2 = 0; a2 < n; ++a2) {
            double s = 0.0;
#pragma unroll
            for (int a = 0; a < n; ++a) s = fma(Dt.D[a2][a], ql[a], s);
            s_s[sidx(e, li, a2, k)] = s;
          }
        }
      }
    }
    __syncthreads();
    // s_q of layer l is dead: gather q(l+1) (IO 2: the loads of layer l + 1; plane l&1 takes level 0 of
    // block l + 2, the level buffer and the stage the rest; IO 3: the row buffer takes layer l + 1)
    if constexpr (IO == 2) {
      if (tid < 32 && l + 1 < nlay) {
        fence_proxy_async();
        issue_loads(l + 1, nper);
      }
    } else if constexpr (IO == 3) {
      if (tid < 32 && l + 1 < nlay) {
        fence_proxy_async();
        issue_chunks(l + 1);
      }
    } else {
      if (l + 1 < l1) issue_gather(gnext);
    }
    if (AB & 8) {
#pragma unroll
      for (int r = 0; r < NR; ++r)
#pragma unroll
        for (int k = 0; k < n; ++k) p0[r][k] = p2[r][k] = s_q[tq(r, jp, k)];
    }
    // ---- c: flux at the plane nodes, weak xi / zeta in registers
    if (WV == 0 && !(AB & 4)) mbar_wait(bar, (uint32_t)((l - l0) & 1));
    if (run && WF == 2) {
      // isotropic form: [i][k][e][j]; the F field lanes of a plane read the same s (broadcast)
      const double* Sw = s_w + e * n + jp;
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        const int i = I0 + r;
        double d1[n], sv[n];
#pragma unroll
        for (int k = 0; k < n; ++k) {
          sv[k] = Sw[i * C::MIS + k * NE * n];
          d1[k] = s_s[sidx(e, i, jp, k)];
        }
#pragma unroll
        for (int k = 0; k < n; ++k) {
          p0[r][k] *= sv[k];
          s_s[sidx(e, i, jp, k)] = sv[k] * d1[k];
          p2[r][k] *= sv[k];
        }
      }
    }
    if (run && WF == 1) {
      // axis form: [c][i][k][e][j]; the F field lanes of a plane read the same u (broadcast)
      const double* Uw = s_w + e * n + jp;
      const double kh = A.kh;   // kh / kd: u is scaled by sqrt(|kd|), the sign of kd is in A.scale (capi_lap.cu)
      constexpr int CS = n * n * NE * n;
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        const int i = I0 + r;
        constexpr int KB = (n > 5) ? 1 : n;
#pragma unroll
        for (int k0 = 0; k0 < n; k0 += KB) {
          double d1[KB], u0[KB], u1[KB], u2[KB];
#pragma unroll
          for (int kk = 0; kk < KB; ++kk) {
            const int wo = (i * n + k0 + kk) * NE * n;
            u0[kk] = Uw[wo];
            u1[kk] = Uw[CS + wo];
            u2[kk] = Uw[2 * CS + wo];
            d1[kk] = s_s[sidx(e, i, jp, k0 + kk)];
          }
#pragma unroll
          for (int kk = 0; kk < KB; ++kk) {
            const int k = k0 + kk;
            const double d0 = p0[r][k], d2 = p2[r][k];
            const double hs = kh * (u0[kk] * u0[kk] + u1[kk] * u1[kk] + u2[kk] * u2[kk]);
            const double tv = u0[kk] * d0 + u1[kk] * d1[kk] + u2[kk] * d2;
            p0[r][k] = hs * d0 + tv * u0[kk];
            s_s[sidx(e, i, jp, k)] = hs * d1[kk] + tv * u1[kk];
            p2[r][k] = hs * d2 + tv * u2[kk];
          }
        }
      }
    }
    if (run) {
      const double* W = (WV == 0) ? s_w + (e * n + jp) * 2 : Wt_t + (int64_t)l * C::WL + (e * n + jp) * 2;
#pragma unroll
      for (int r = 0; r < NR && WF == 0; ++r) {
        const int i = I0 + r;
        // all loads of a row chunk first: one shared-memory round trip per chunk, not per node
        constexpr int KB = (n > 5) ? n / 2 : n;
#pragma unroll
        for (int k0 = 0; k0 < n; k0 += KB) {
          double d1[KB];
          double2 wa[KB], wb[KB], wc[KB];   // (w00 w01) (w02 w11) (w12 w22)
#pragma unroll
          for (int kk = 0; kk < KB; ++kk) {
            const int wo = (i * n + k0 + kk) * NE * n * 2;
            if (WV == 0) {
              wa[kk] = *reinterpret_cast<const double2*>(W + 0 * n * n * NE * n * 2 + wo);
              wb[kk] = *reinterpret_cast<const double2*>(W + 1 * n * n * NE * n * 2 + wo);
              wc[kk] = *reinterpret_cast<const double2*>(W + 2 * n * n * NE * n * 2 + wo);
            } else {
              wa[kk] = ldg_stream2(W + 0 * n * n * NE * n * 2 + wo);
              wb[kk] = ldg_stream2(W + 1 * n * n * NE * n * 2 + wo);
              wc[kk] = ldg_stream2(W + 2 * n * n * NE * n * 2 + wo);
            }
            d1[kk] = s_s[sidx(e, i, jp, k0 + kk)];
          }
#pragma unroll
          for (int kk = 0; kk < KB; ++kk) {
            const int k = k0 + kk;
            const double d0 = p0[r][k], d2 = p2[r][k];
            p0[r][k] = wa[kk].x * d0 + wa[kk].y * d1[kk] + wb[kk].x * d2;
            s_s[sidx(e, i, jp, k)] = wa[kk].y * d0 + wb[kk].y * d1[kk] + wc[kk].x * d2;
            p2[r][k] = wb[kk].x * d0 + wc[kk].x * d1[kk] + wc[kk].y * d2;
          }
        }
      }
      // weak xi (columns of p0, in place): p0[i][k] <- -sum_a D[a][i] f_xi[a][k]
#pragma unroll
      for (int k = 0; k < n; ++k) {
        if constexpr (H == 1) {
          double c[n], yl[n];
#pragma unroll
          for (int a = 0; a < n; ++a) c[a] = p0[a][k];
          hv::eo_mv<n, 1>(Dt, c, yl);
#pragma unroll
          for (int i = 0; i < n; ++i) p0[i][k] = yl[i];
        } else {
          double co[NR], cp[H - 1][NR];
#pragma unroll
          for (int r = 0; r < NR; ++r) co[r] = p0[r][k];
#pragma unroll
          for (int m = 1; m < H; ++m)
#pragma unroll
            for (int r = 0; r < NR; ++r) cp[m - 1][r] = __shfl_xor_sync(0xffffffffu, co[r], F * m);
#pragma unroll
          for (int r = 0; r < NR; ++r) {
            double s = 0.0;
#pragma unroll
            for (int a = 0; a < NR; ++a) s = fma(sD[(I0 + a) * n + I0 + r], co[a], s);
#pragma unroll
            for (int m = 1; m < H; ++m) {
              const int pb = (ih ^ m) * NR;
#pragma unroll
              for (int a = 0; a < NR; ++a) s = fma(sD[(pb + a) * n + I0 + r], cp[m - 1][a], s);
            }
            p0[r][k] = -s;
          }
        }
      }
      // weak zeta (rows of p2) accumulated into p0
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        if constexpr (EO) {
          double yl[n];
          hv::eo_mv<n, 1>(Dt, p2[r], yl);
#pragma unroll
          for (int k = 0; k < n; ++k) p0[r][k] += yl[k];
        } else {
#pragma unroll
          for (int k = 0; k < n; ++k) {
            double s = 0.0;
#pragma unroll
            for (int a = 0; a < n; ++a) s = fma(Dt.D[a][k], p2[r][a], s);
            p0[r][k] -= s;
          }
        }
      }
    }
    __syncthreads();
    if (WV == 0 && tid == 0 && l + 1 < l1) {      // metric buffer free: W(l+1) lands during d, e, f, a, b
      fence_proxy_async();
      issue_metric(l + 1);
    }
    // ---- d: eta lines weak, in place (line i = jp of element e, zeta levels K0 .. K0 + NK)
    if (run) {
#pragma unroll
      for (int kk = 0; kk < NK; ++kk) {
        const int li = (H == 1) ? jp : I0 + kk, k = (H == 1) ? K0 + kk : jp;   // the lines of step b
        double ql[n];
#pragma unroll
        for (int a = 0; a < n; ++a) ql[a] = s_s[sidx(e, li, a, k)];
        if constexpr (EO) {   // -D^T: step e adds
          double yl[n];
          hv::eo_mv<n, 1>(Dt, ql, yl);
#pragma unroll
          for (int a2 = 0; a2 < n; ++a2) s_s[sidx(e, li, a2, k)] = yl[a2];
        } else {
#pragma unroll
          for (int a2 = 0; a2 < n; ++a2) {
            double s = 0.0;
#pragma unroll
            for (int a = 0; a < n; ++a) s = fma(Dt.D[a][a2], ql[a], s);
            s_s[sidx(e, li, a2, k)] = s;
          }
        }
      }
    }
    __syncthreads();
    // ---- e: element accumulator (+ vertical carry) -> scratch; gid / Minv of the output items
    int gf[PF];
    double mf[PF];
    double my[C::PFY];   // IO 1: scale * Minv of tile-owned block items, 1 for perimeter (raw partial sums)
    // IO 1 / 3: the items' columns (7 bits each, bit 7 = tile-owned) stay packed in one register from here
    // to step f, which then starts at the element-copy offsets instead of the chain s_perm -> s_ct
    static_assert(!OUT_YT || (UV < 128 && C::PFY <= 4), "packed item columns");
    unsigned uvp = 0;
    if constexpr (OUT_YT) {
#pragma unroll
      for (int it = 0; it < C::PFY; ++it) {
        const int qi = tid + it * C::NT;
        my[it] = 1.0;
        if (qi < C::FIY) {
          const int uv = s_perm[qi / N], k = qi % N;
          const bool own = s_code[uv] < 0;
          uvp |= (unsigned)(uv | (own ? 0x80 : 0)) << (8 * it);
          if (own) my[it] = __ldg(Mt_t + (int64_t)l * C::MTS + uv * n + k);   // scaled at its use in step f
        }
      }
    } else {
#pragma unroll
      for (int it = 0; it < PF; ++it) {
        const int qi = tid + it * C::NT;
        const int node = (qi < C::FI) ? s_perm[qi / N] * n + qi % N : 0;
        gf[it] = (qi < C::FI) ? __ldg(gt_t + (int64_t)l * C::GTS + node) : -1;
        mf[it] = (qi < C::FI) ? __ldg(Mt_t + (int64_t)l * C::MTS + node) : 0.0;
      }
    }
    if (act) {
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        const int i = I0 + r;
#pragma unroll
        for (int k = 0; k < n; ++k) p0[r][k] = EO ? p0[r][k] + s_s[sidx(e, i, jp, k)] : p0[r][k] - s_s[sidx(e, i, jp, k)];
        p0[r][0] += carry[r];
        carry[r] = p0[r][N];
#pragma unroll
        for (int k = 0; k < n; ++k) s_s[sidx(e, i, jp, k)] = p0[r][k];
      }
    } else if (pth) {
#pragma unroll
      for (int r = 0; r < NR; ++r)
#pragma unroll
        for (int k = 0; k < n; ++k) s_s[sidx(e, I0 + r, jp, k)] = 0.0;
    }
    __syncthreads();
    // ---- f: node owners (items (column, k < N); k = N only on the top layer) sum the
    // element copies of all F fields (predicated loads, fixed order (c0 + c1) + (c2 + c3)),
    // then one row store per item
    if constexpr (OUT_YT) {
      // block items in s_perm order (tile-owned columns first, the N levels of a column in consecutive
      // lanes: the element-copy reads then have fewer bank conflicts than in (k, u, v) order, and a warp
      // still stores runs of a level).  Perimeter (slot) items: raw partial sums (my = 1) also into their
      // partial rows, 4 lanes one 128-byte run (the fix-up sums them into the compact slot rows that pass
      // 2 stages); their block entries are never read, the raw sums keep the block's sectors whole
      double* yb = A.out + t * chain + (int64_t)l * C::YBLK;
#pragma unroll
      for (int it = 0; it < C::PFY; ++it) {
        const int qi = tid + it * C::NT;
        if (qi >= C::FIY) continue;
        const unsigned ub = (uvp >> (8 * it)) & 0xffu;
        const int uv = (int)(ub & 0x7fu), k = qi % N, u = uv / V, v = uv - u * V;
        const int4 ct = s_ct[uv];
        const bool own = (ub & 0x80u) != 0;
        const double ms = own ? A.scale * my[it] : 1.0;
        hv::Vec<F> val;
#pragma unroll
        for (int p = 0; p < F; ++p) {
          val.v[p] = ms * csum(ct, s_s + p * C::SP + k);
          yb[k * C::YLS + p * C::YFS + u * C::YUS + v] = val.v[p];
        }
        if (!own) {
          double* o = A.part + ((int64_t)s_code[uv] * A.n_z + l * N + k) * F;
          st_v2(o, val.v[0], val.v[1]);
          st_v2(o + 2, val.v[2], val.v[3]);
        }
      }
      // the layout's padding (v = V..YUS-1 of every u row, u*YUS >= U*YUS up to YFS): zeros, so that
      // every sector of the block is written whole (no partial-sector read-modify-write in L2)
      if constexpr (C::PADTAB) {
        for (int x = tid; x < C::PADN; x += C::NT) yb[s_pad[x]] = 0.0;
      } else {
        constexpr int PV = C::YUS - V, PT = C::YFS - U * C::YUS, PP = U * PV + PT;
        for (int x = tid; x < N * F * PP; x += C::NT) {
          const int kf = x / PP, j = x - kf * PP;
          yb[(kf / F) * C::YLS + (kf % F) * C::YFS + ((j < U * PV) ? (j / PV) * C::YUS + V + j % PV : U * C::YUS + j - U * PV)] = 0.0;
        }
      }
      if (l == nlay - 1) {        // top level of the columns -> level 0 of block nlay
        double* yt = yb + C::YBLK;
        for (int uv = tid; uv < UV; uv += C::NT) {
          const int u = uv / V, v = uv % V;
          const int4 ct = s_ct[uv];
          const int cd = s_code[uv];
          const double m = (cd < 0) ? A.scale * __ldg(Mt_t + (int64_t)l * C::MTS + uv * n + N) : 1.0;
          hv::Vec<F> val;
#pragma unroll
          for (int p = 0; p < F; ++p) {
            val.v[p] = m * csum(ct, s_s + p * C::SP + N);
            yt[p * C::YFS + u * C::YUS + v] = val.v[p];
          }
          if (cd >= 0) {
            double* o = A.part + ((int64_t)cd * A.n_z + l * N + N) * F;
            st_v2(o, val.v[0], val.v[1]);
            st_v2(o + 2, val.v[2], val.v[3]);
          }
        }
        // the top block holds level 0 only: its padding, and levels 1..N-1 left unwritten (never read)
        constexpr int PV = C::YUS - V, PT = C::YFS - U * C::YUS, PP = U * PV + PT;
        for (int x = tid; x < F * PP; x += C::NT) {
          const int ff = x / PP, j = x - ff * PP;
          yt[ff * C::YFS + ((j < U * PV) ? (j / PV) * C::YUS + V + j % PV : U * C::YUS + j - U * PV)] = 0.0;
        }
      }
    } else if (!(AB & 1)) {
#pragma unroll
      for (int it = 0; it < PF; ++it) {
        const int qi = tid + it * C::NT;
        if (gf[it] < 0) continue;
        const int uv = s_perm[qi / N], k = qi % N;
        const int4 ct = s_ct[uv];
        hv::Vec<F> val;
#pragma unroll
        for (int p = 0; p < F; ++p) {
          const double* sp = s_s + p * C::SP + k;
          const double c0 = sp[ct.x];
          const double c1 = (ct.y >= 0) ? sp[ct.y] : 0.0;
          const double c2 = (ct.z >= 0) ? sp[ct.z] : 0.0;
          const double c3 = (ct.z >= 0) ? sp[ct.w] : 0.0;
          val.v[p] = (c0 + c1) + (c2 + c3);
        }
        if (IO == 0 && k == 0 && l == l0 && l0 > 0) {   // segment bottom: raw sum, from above
          double* o = A.bnd + (((t * (nseg - 1) + sg - 1) * 2 + 1) * UV + uv) * F;
#pragma unroll
          for (int p = 0; p < F; ++p) o[p] = val.v[p];
        } else {
          emit(gf[it], mf[it], val, s_code[uv], l * N + k);
        }
      }
      if (IO == 0 && l == l1 - 1 && l1 < nlay) {   // segment top: raw sums, from below
        for (int uv = tid; uv < UV; uv += C::NT) {
          const int4 ct = s_ct[uv];
          double* o = A.bnd + (((t * (nseg - 1) + sg) * 2 + 0) * UV + uv) * F;
#pragma unroll
          for (int p = 0; p < F; ++p) o[p] = csum(ct, s_s + p * C::SP + N);
        }
      }
      if (l == nlay - 1) {        // top nodes of the columns
        for (int uv = tid; uv < UV; uv += C::NT) {
          const int node = uv * n + N;
          const int g = __ldg(gt_t + (int64_t)l * C::GTS + node);
          if (g < 0) continue;
          const int4 ct = s_ct[uv];
          hv::Vec<F> v;
#pragma unroll
          for (int p = 0; p < F; ++p) {
            const double* sp = s_s + p * C::SP + N;
            const double c0 = sp[ct.x];
            const double c1 = (ct.y >= 0) ? sp[ct.y] : 0.0;
            const double c2 = (ct.z >= 0) ? sp[ct.z] : 0.0;
            const double c3 = (ct.z >= 0) ? sp[ct.w] : 0.0;
            v.v[p] = (c0 + c1) + (c2 + c3);
          }
          emit(g, __ldg(Mt_t + (int64_t)l * C::MTS + node), v, s_code[uv], l * N + N);
        }
      }
    }
    if (GATHER && l + 2 < l1) load_gids(l + 2, gnext);   // consumed by the gather issued in step b of l + 1
    // the next step's barrier (a) orders these reads before the scratch is rewritten
  }
}


// Plane-layout packed metric, component pairs:
// Wp[t][l][cp][i][k][e][j][h] = W[2cp+h][elem(t,l,e)*n^3 + (i*n + j)*n + k];
// axis form (axis == 1, W = U (3, nloc)): Wp[t][l][c][i][k][e][j] = U[c][...];
// isotropic form (axis == 2, W = s (1, nloc)): Wp[t][l][i][k][e][j] = s[...].
__global__ void plane_pack_metric(int n, int NE, int64_t ntiles, int nlay, const int32_t* __restrict__ elem,
                                  const double* __restrict__ W, int64_t nloc, int axis, int mis,
                                  double* __restrict__ Wp) {
  const int64_t per = axis == 2 ? (int64_t)n * mis : (int64_t)(axis ? 3 : 6) * n * n * NE * n;
  const int64_t total = ntiles * nlay * per;
  for (int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; id < total; id += (int64_t)gridDim.x * blockDim.x) {
    const int64_t tl = id / per;
    int64_t r = id % per;
    if (axis == 2) {   // [i][mis]: k, e, j in the first n * NE * n of a row, zero padding after
      const int i = (int)(r / mis), rr = (int)(r % mis);
      if (rr >= n * NE * n) { Wp[id] = 0.0; continue; }
      r = (int64_t)(i * n + rr / (NE * n)) * NE * n + rr % (NE * n);
    }
    int h = 0;
    if (!axis) { h = (int)(r % 2); r /= 2; }
    const int j = (int)(r % n); r /= n;
    const int e = (int)(r % NE); r /= NE;
    const int k = (int)(r % n); r /= n;
    const int i = (int)(r % n); r /= n;
    const int c = axis ? (int)r : (int)r * 2 + h;
    const int eg = elem[tl * NE + e];
    Wp[id] = (eg >= 0) ? W[c * nloc + (int64_t)eg * n * n * n + (i * n + j) * n + k] : 0.0;
  }
}

// compile-time output mode of this pass (OM of lap_plane_kernel)
inline int output_mode(const TileArgs& A, int F) {
  if (F != 4 || A.accumulate) return 0;
  const bool f0 = A.of.f[0] == 0 && A.of.f[1] == 1 && A.of.f[2] == 2 && A.of.f[3] == 3;
  const bool f1 = A.of.f[0] == 1 && A.of.f[1] == 2 && A.of.f[2] == 3 && A.of.f[3] == 4;
  if (A.ldo == 4 && !A.zero_mask && f0) return 1;
  if (A.ldo == 5 && A.zero_mask == 1u && f1) return 2;   // the OM 2 rows zero column 0
  return 0;
}

template <int n, int TX, int TY, int F, int WV, int MB, int AB = 0, int H = 1, int WF = 0, int OM = 0, int IO = 0>
int run_plane_om(const TileArgs& A, const hv::DTabEO<n>& Dt, cudaStream_t st) {
  using C = PlaneCfg<n, TX, TY, F, WV, H, WF, IO>;
  auto kern = lap_plane_kernel<n, TX, TY, F, WV, MB, AB, H, WF, OM, IO>;
  HV_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
  if (A.tile1 <= A.tile0) return HV_OK;
  const int nseg = (IO == 0 && A.seg > 0) ? (A.nlay + A.seg - 1) / A.seg : 1;
  if (IO != 0 && A.seg > 0) HV_FAIL(HV_ERR_UNSUPPORTED, "plane kernel: vertical segments need io 0");
  kern<<<(unsigned)((A.tile1 - A.tile0) * nseg), C::NT, C::SMEM, st>>>(Dt, A);
  HV_LAUNCH_CHECK();
  return HV_OK;
}

template <int n, int TX, int TY, int F, int WV, int MB, int AB = 0, int H = 1, int WF = 0>
int run_plane_v(const TileArgs& A, const hv::DTabEO<n>& Dt, cudaStream_t st) {
  // N = 7 hot passes (c4: 6.17 -> 6.02 ms); at N = 4 the specialised code measured slower
  // (c5 sweep 1.76 -> 1.90 ms, scheduling), so N <= 4 keeps the runtime checks
  if constexpr (F == 4 && n == 8 && AB == 0) {
    const int om = output_mode(A, F);
    if (om == 1) return run_plane_om<n, TX, TY, F, WV, MB, AB, H, WF, 1>(A, Dt, st);
    if (om == 2) return run_plane_om<n, TX, TY, F, WV, MB, AB, H, WF, 2>(A, Dt, st);
  }
  return run_plane_om<n, TX, TY, F, WV, MB, AB, H, WF, 0>(A, Dt, st);
}

// Production: W by TMA into shared memory, 3 CTAs/SM (N <= 4); split planes H = 4 at N = 7
// (HV_N7_SPLIT=2 for H = 2).  Building with -DHV_PLANE_ABLATE adds the development variants
// selected by HV_PLANE_VARIANT (metric from global memory, other occupancy targets, ablations
// of single steps; tools_time_plane.py).
template <int n, int TX, int TY, int F>
int run_plane(const TileArgs& A, const double* Drow, cudaStream_t st) {
  hv::DTabEO<n> Dt;
  hv::fill_dtab_eo(Dt, Drow);
  if constexpr (n == 8) {
    const char* hs = getenv("HV_N7_SPLIT");
    if constexpr (TX == 1 && TY == 1 && F == 4) {   // tile-ordered intermediate passes (split planes, H = 4)
      if (A.io == 1 || A.io == 2) {
        if (hs && atoi(hs) == 2) HV_FAIL(HV_ERR_UNSUPPORTED, "plane kernel: tile-ordered passes need H = 4 at N = 7");
        const bool w = A.io == 1;
        if (A.wform == 1) return w ? run_plane_om<n, TX, TY, F, 0, 1, 0, 4, 1, 0, 1>(A, Dt, st)
                                   : run_plane_om<n, TX, TY, F, 0, 1, 0, 4, 1, 0, 2>(A, Dt, st);
        // isotropic form (config 4): 168 registers without spills, so three CTAs per SM instead of two
        // (c4 5.06 -> 4.76 ms per op; four CTAs at 128 registers spill: 4.94 ms; the rows-path variants
        // spill at 168: no gain)
        if (A.wform == 2) return w ? run_plane_om<n, TX, TY, F, 0, 3, 0, 4, 2, 0, 1>(A, Dt, st)
                                   : (output_mode(A, F) == 2 ? run_plane_om<n, TX, TY, F, 0, 3, 0, 4, 2, 2, 2>(A, Dt, st)
                                                             : run_plane_om<n, TX, TY, F, 0, 3, 0, 4, 2, 0, 2>(A, Dt, st));
        return w ? run_plane_om<n, TX, TY, F, 0, 1, 0, 4, 0, 0, 1>(A, Dt, st)
                 : run_plane_om<n, TX, TY, F, 0, 1, 0, 4, 0, 0, 2>(A, Dt, st);
      }
    }
    if (A.io) HV_FAIL(HV_ERR_UNSUPPORTED, "plane kernel: no tile-ordered mode for this shape");
    if (A.wform == 1) {
      if (hs && atoi(hs) == 2) return run_plane_v<n, TX, TY, F, 0, 1, 0, 2, 1>(A, Dt, st);
      return run_plane_v<n, TX, TY, F, 0, 1, 0, 4, 1>(A, Dt, st);
    }
    if (A.wform == 2) {
      if (hs && atoi(hs) == 2) return run_plane_v<n, TX, TY, F, 0, 1, 0, 2, 2>(A, Dt, st);
      return run_plane_v<n, TX, TY, F, 0, 1, 0, 4, 2>(A, Dt, st);
    }
    if (hs && atoi(hs) == 2) return run_plane_v<n, TX, TY, F, 0, 1, 0, 2>(A, Dt, st);
    return run_plane_v<n, TX, TY, F, 0, 1, 0, 4>(A, Dt, st);
  } else {
#ifdef HV_PLANE_ABLATE
    if constexpr (n == 5 && F == 4) {
      const char* v = getenv("HV_PLANE_VARIANT");
      switch (v ? atoi(v) : 0) {
        case 1: return run_plane_v<n, TX, TY, F, 0, 4>(A, Dt, st);
        case 2: return run_plane_v<n, TX, TY, F, 1, 4>(A, Dt, st);
        case 3: return run_plane_v<n, TX, TY, F, 1, 5>(A, Dt, st);
        case 4: return run_plane_v<n, TX, TY, F, 1, 6>(A, Dt, st);
        case 11: return run_plane_v<n, TX, TY, F, 0, 3, 1>(A, Dt, st);
        case 12: return run_plane_v<n, TX, TY, F, 0, 3, 2>(A, Dt, st);
        case 14: return run_plane_v<n, TX, TY, F, 0, 3, 4>(A, Dt, st);
        case 18: return run_plane_v<n, TX, TY, F, 0, 3, 8>(A, Dt, st);
        case 13: return run_plane_v<n, TX, TY, F, 0, 3, 3>(A, Dt, st);
        case 17: return run_plane_v<n, TX, TY, F, 0, 3, 7>(A, Dt, st);
        case 25: return run_plane_v<n, TX, TY, F, 0, 3, 15>(A, Dt, st);
        default: break;
      }
    }
#endif
    if constexpr (n == 5 && TX == 2 && TY == 2 && F == 4) {   // tile-ordered intermediate passes
      if (A.io == 3) {
        if (A.wform == 1) return run_plane_om<n, TX, TY, F, 0, 3, 0, 1, 1, 0, 3>(A, Dt, st);
        if (A.wform == 2) return run_plane_om<n, TX, TY, F, 0, 3, 0, 1, 2, 0, 3>(A, Dt, st);
        return run_plane_om<n, TX, TY, F, 0, 3, 0, 1, 0, 0, 3>(A, Dt, st);
      }
      if (A.io == 1 || A.io == 2) {
        const bool w = A.io == 1;
#ifdef HV_PLANE_ABLATE
        {
          const char* v = getenv("HV_PLANE_VARIANT");   // 42: pass 1 without the q gather (timing only)
          if (w && A.wform == 1 && v && atoi(v) == 42) return run_plane_om<n, TX, TY, F, 0, 3, 2, 1, 1, 0, 1>(A, Dt, st);
        }
#endif
        if (A.wform == 1) {
          if (w) return run_plane_om<n, TX, TY, F, 0, 3, 0, 1, 1, 0, 1>(A, Dt, st);
          if (output_mode(A, F) == 2) return run_plane_om<n, TX, TY, F, 0, 3, 0, 1, 1, 2, 2>(A, Dt, st);
          return run_plane_om<n, TX, TY, F, 0, 3, 0, 1, 1, 0, 2>(A, Dt, st);
        }
        const bool o2 = !w && output_mode(A, F) == 2;   // H_nu's (ng, 5) result rows: compile-time row stores
        if (A.wform == 2) return w ? run_plane_om<n, TX, TY, F, 0, 3, 0, 1, 2, 0, 1>(A, Dt, st)
                                   : (o2 ? run_plane_om<n, TX, TY, F, 0, 3, 0, 1, 2, 2, 2>(A, Dt, st)
                                         : run_plane_om<n, TX, TY, F, 0, 3, 0, 1, 2, 0, 2>(A, Dt, st));
        return w ? run_plane_om<n, TX, TY, F, 0, 3, 0, 1, 0, 0, 1>(A, Dt, st)
                 : (o2 ? run_plane_om<n, TX, TY, F, 0, 3, 0, 1, 0, 2, 2>(A, Dt, st)
                       : run_plane_om<n, TX, TY, F, 0, 3, 0, 1, 0, 0, 2>(A, Dt, st));
      }
    }
    if (A.io) HV_FAIL(HV_ERR_UNSUPPORTED, "plane kernel: no tile-ordered mode for this shape");
    if (A.wform == 1) {
#ifdef HV_PLANE_ABLATE
      const char* v = getenv("HV_PLANE_VARIANT");
      switch (v ? atoi(v) : 0) {
        case 41: return run_plane_v<n, TX, TY, F, 0, 3, 1, 1, 1>(A, Dt, st);
        case 42: return run_plane_v<n, TX, TY, F, 0, 3, 2, 1, 1>(A, Dt, st);
        case 44: return run_plane_v<n, TX, TY, F, 0, 3, 4, 1, 1>(A, Dt, st);
        case 48: return run_plane_v<n, TX, TY, F, 0, 3, 8, 1, 1>(A, Dt, st);
        case 43: return run_plane_v<n, TX, TY, F, 0, 3, 3, 1, 1>(A, Dt, st);
        case 47: return run_plane_v<n, TX, TY, F, 0, 3, 7, 1, 1>(A, Dt, st);
        case 55: return run_plane_v<n, TX, TY, F, 0, 3, 15, 1, 1>(A, Dt, st);
        default: break;
      }
#endif
      return run_plane_v<n, TX, TY, F, 0, 3, 0, 1, 1>(A, Dt, st);
    }
    if (A.wform == 2) return run_plane_v<n, TX, TY, F, 0, 3, 0, 1, 2>(A, Dt, st);
    return run_plane_v<n, TX, TY, F, 0, 3>(A, Dt, st);
  }
}

}  // namespace

namespace hv {

bool plane_supported(int N, int TX, int TY, int F) {
  if (N == 7) return F == 4 && ((TX == 2 && TY == 2) || (TX == 1 && TY == 1));   // split planes
  return (F == 1 || F == 4 || F == 5) && TX == 2 && TY == 2 && N >= 1 && N <= 4;
}

int laplacian_plane(const TileArgs& A, int N, int F, const double* Drow, cudaStream_t st) {
#define HV_PLANE_CASE(NN_)                                        \
  if (N == NN_) {                                                 \
    if (F == 1) return run_plane<NN_ + 1, 2, 2, 1>(A, Drow, st);  \
    if (F == 4) return run_plane<NN_ + 1, 2, 2, 4>(A, Drow, st);  \
    if (F == 5) return run_plane<NN_ + 1, 2, 2, 5>(A, Drow, st);  \
  }
  if (N == 7 && F == 4 && A.TX == 2) return run_plane<8, 2, 2, 4>(A, Drow, st);
  if (N == 7 && F == 4 && A.TX == 1) return run_plane<8, 1, 1, 4>(A, Drow, st);
  HV_PLANE_CASE(1)
  HV_PLANE_CASE(2)
  HV_PLANE_CASE(3)
  HV_PLANE_CASE(4)
#undef HV_PLANE_CASE
  HV_FAIL(HV_ERR_UNSUPPORTED, "plane kernel: no instantiation for N=%d F=%d", N, F);
}

int plane_chunk_rows(int N, int TX, int TY) {
  if (N != 4 || TX != 2 || TY != 2) return -1;
  return PlaneCfg<5, 2, 2, 4, 0, 1, 1, 3>::CRR - 2;
}

bool plane_yt_layout(int N, int TX, int TY, int F, int64_t* lay) {
  if (F != 4) return false;
  if (N == 7 && TX == 1 && TY == 1) {   // split-plane kernel: lanes (f, ih) hit f + 4 ih (mod 16) as well
    using C = PlaneCfg<8, 1, 1, 4, 0, 4, 2, 1>;
    lay[0] = C::YLS;
    lay[1] = C::YUS;
    lay[2] = C::YFS;
    lay[3] = C::YBLK;
    lay[4] = C::NPER;
    return true;
  }
  if (N != 4 || TX != 2 || TY != 2) return false;
  using C = PlaneCfg<5, 2, 2, 4, 0, 1, 1, 1>;
  lay[0] = C::YLS;
  lay[1] = C::YUS;
  lay[2] = C::YFS;
  lay[3] = C::YBLK;
  lay[4] = C::NPER;
  return true;
}

int plane_metric_row(int N, int TX, int TY) {
  if (N == 7 && TX == 1 && TY == 1) return PlaneCfg<8, 1, 1, 4, 0, 4, 2>::MIS;
  return (N + 1) * TX * TY * (N + 1);
}

int64_t plane_metric_doubles(int N, int TX, int TY, int wform) {
  const int n = N + 1;
  if (wform == 2) return (int64_t)n * plane_metric_row(N, TX, TY);
  return (int64_t)(wform == 1 ? 3 : 6) * n * TX * TY * n * n;
}

int plane_pack(int N, int TX, int TY, int64_t ntiles, int nlay, const int32_t* elem, const double* W, int64_t nloc,
               int axis, double* Wp, cudaStream_t st) {
  plane_pack_metric<<<148 * 8, 256, 0, st>>>(N + 1, TX * TY, ntiles, nlay, elem, W, nloc, axis,
                                             plane_metric_row(N, TX, TY), Wp);
  HV_LAUNCH_CHECK();
  return HV_OK;
}

}  // namespace hv
