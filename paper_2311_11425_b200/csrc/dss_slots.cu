// Off-chip part of the DSS for the tile-sweep kernels: column nodes shared by
// several tiles ("slots", tiles.py) and, with several GPUs, slab-interface
// column nodes shared with a neighbouring rank (parallel.py).
//
// slot_pack   per interface slot and level: the fixed-order sum of the local
//             partial rows -> the send buffer of that side (ncclSend payload).
// slot_fixup  per slot and level: the fixed-order sum of the local partial rows,
//             plus the neighbour's sum (received) in global rank order
//             (lower rank first) so both ranks produce bitwise identical values;
//             times scale * Minv, written to the output row (reference DSS
//             semantics, assembly.py:17-26 and hyperdiff.py:94).
#include <cuda_runtime.h>

#include "hv_common.h"
#include "lap_common.cuh"
#include "lap_tile.cuh"

namespace {

using hv::TileArgs;

// partial row of F doubles (rows are F-strided, so F = 4 rows are 32-byte aligned: two 16-byte loads)
template <int F>
__device__ __forceinline__ void load_row(const double* p, double (&v)[F]) {
  if constexpr (F == 4) {
    const double2 a = __ldg(reinterpret_cast<const double2*>(p));
    const double2 b = __ldg(reinterpret_cast<const double2*>(p) + 1);
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
  } else {
#pragma unroll
    for (int ff = 0; ff < F; ++ff) v[ff] = __ldg(p + ff);
  }
}

// fixed-order (r ascending) sum of a slot's partial rows; the first four rows (all of them
// except at cube corners of fine meshes) are loaded before any is added, so their loads overlap
template <int F>
__device__ __forceinline__ void local_sum(const TileArgs& A, int64_t s, int z, double (&acc)[F]) {
  constexpr int U = 4;
  const int r0 = A.slot_row0[s], nc = A.slot_nc[s];
  double v[U][F];
#pragma unroll
  for (int r = 0; r < U; ++r)
    if (r < nc) load_row<F>(A.part + ((int64_t)(r0 + r) * A.n_z + z) * F, v[r]);   // partial rows: F doubles
#pragma unroll
  for (int ff = 0; ff < F; ++ff) acc[ff] = 0.0;
#pragma unroll
  for (int r = 0; r < U; ++r)
    if (r < nc) {
#pragma unroll
      for (int ff = 0; ff < F; ++ff) acc[ff] += v[r][ff];
    }
  for (int r = U; r < nc; ++r) {
    double w[F];
    load_row<F>(A.part + ((int64_t)(r0 + r) * A.n_z + z) * F, w);
#pragma unroll
    for (int ff = 0; ff < F; ++ff) acc[ff] += w[ff];
  }
}

__device__ __forceinline__ void st2(double* p, double a, double b) {
  *reinterpret_cast<double2*>(p) = make_double2(a, b);
}

template <int F>
__global__ void slot_pack_kernel(TileArgs A) {
  const int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (id >= A.next * A.n_z) return;
  const int64_t s = A.ext_slots[id / A.n_z];
  const int z = (int)(id % A.n_z);
  double acc[F];
  local_sum<F>(A, s, z, acc);
  double* o = A.send + ((int64_t)A.slot_ext[s] * A.n_z + z) * F;   // halo rows: F doubles
#pragma unroll
  for (int ff = 0; ff < F; ++ff) o[ff] = acc[ff];
}

// vertical segments (lap_plane.cu, TileArgs::seg): the partial of a slot column node on a segment
// boundary is the sum of the two segments' raw sums (from below, then from above) of its owning tile
template <int F>
__device__ __forceinline__ void bnd_partial(const TileArgs& A, int64_t r, int b, int nseg, int UV, double (&v)[F]) {
  const int64_t tu = A.prow[r], t = tu / UV, uv = tu - t * UV;
  const double* lo = A.bnd + (((t * (nseg - 1) + b) * 2 + 0) * UV + uv) * F;
  const double* hi = lo + (int64_t)UV * F;
#pragma unroll
  for (int ff = 0; ff < F; ++ff) v[ff] = lo[ff] + hi[ff];
}

template <int F>
__global__ void slot_fixup_kernel(TileArgs A, int row_mode) {
  const int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nsi = A.nslot * A.n_z;
  const int N = (A.n_z - 1) / A.nlay, n = N + 1;
  const int nseg = A.seg > 0 ? (A.nlay + A.seg - 1) / A.seg : 1;
  const int UV = (A.TX * N + 1) * (A.TY * N + 1);
  const unsigned nz = (unsigned)A.n_z;
  int64_t s = -1;  // slot (-1: a tile-owned node on a segment boundary)
  int z;           // level
  int g;           // output row
  double acc[F];
  double mi;
  double* o;
  if (id < nsi) {
    s = (unsigned)id / nz;       // nslot * n_z < 2^31 (checked by the launcher)
    z = (int)((unsigned)id - (unsigned)s * nz);
    g = A.col_gid[(int64_t)A.slot_col[s] * A.n_z + z];
    mi = A.Ms ? __ldg(A.Ms + s * A.n_z + z) : __ldg(A.Minv + g);
    const int zb = (nseg > 1) ? A.seg * N : 0;
    if (zb && z % zb == 0 && z > 0 && z < A.n_z - 1) {   // segment boundary: the owners' two halves
      const int b = z / zb - 1, r0 = A.slot_row0[s], nc = A.slot_nc[s];
#pragma unroll
      for (int ff = 0; ff < F; ++ff) acc[ff] = 0.0;
      for (int r = 0; r < nc; ++r) {
        double v[F];
        bnd_partial<F>(A, r0 + r, b, nseg, UV, v);
#pragma unroll
        for (int ff = 0; ff < F; ++ff) acc[ff] += v[ff];
      }
    } else {
      local_sum<F>(A, s, z, acc);
    }
  } else {
    // tile-owned column nodes on segment boundaries: (tile, boundary, column)
    if (nseg == 1) return;
    const int64_t x = id - nsi, per = (int64_t)(nseg - 1) * UV;
    const int64_t t = x / per;
    if (t >= A.ntiles) return;
    const int b = (int)((x - t * per) / UV), uv = (int)(x % UV);
    if (A.code[t * UV + uv] >= 0) return;                 // slot columns: the slot items above
    const int lb = (b + 1) * A.seg, gts = (UV * n + 3) & ~3;
    g = A.gt[(t * A.nlay + lb) * gts + uv * n];
    if (g < 0) return;
    z = lb * N;
    mi = __ldg(A.Minv + g);
    const double* lo = A.bnd + (((t * (nseg - 1) + b) * 2 + 0) * UV + uv) * F;
    const double* hi = lo + (int64_t)UV * F;
#pragma unroll
    for (int ff = 0; ff < F; ++ff) acc[ff] = lo[ff] + hi[ff];
  }
  if (row_mode == 3) {
    // the slot rows of the tile-ordered intermediate (lap_tile.cuh: [nslot][F] for z = 0, then per layer
    // block [nslot][N][F]); threads walk a column's levels (its partial rows are read as contiguous runs,
    // the slot rows written as 128-byte pieces)
    const int64_t row = (z == 0) ? s : A.nslot + (((int64_t)((z - 1) / N) * A.nslot + s) * N + (z - 1) % N);
    o = A.sv + row * F;
  } else {
    o = A.out + (int64_t)g * A.ldo;
  }
  double prev[F];
  if (A.accumulate) {
#pragma unroll
    for (int ff = 0; ff < F; ++ff) prev[ff] = o[A.of.f[ff]];
  }
  if (s >= 0 && A.slot_ext && A.slot_ext[s] >= 0) {
    const int ext = A.slot_ext[s];
    const double* rm = A.recv + ((int64_t)ext * A.n_z + z) * F;
    const bool lower_side = ext < A.face;   // side 0: the neighbour has the lower rank
#pragma unroll
    for (int ff = 0; ff < F; ++ff) acc[ff] = lower_side ? rm[ff] + acc[ff] : acc[ff] + rm[ff];
  }
  double r[F];
#pragma unroll
  for (int ff = 0; ff < F; ++ff) r[ff] = A.scale * (mi * acc[ff]);
  if constexpr (F == 4) {
    if (row_mode == 1 || row_mode == 3) {   // (ng, 4) rows, fields 0..3 / slot rows
      st2(o, r[0], r[1]);
      st2(o + 2, r[2], r[3]);
      return;
    }
    if (row_mode == 2) {             // (ng, 5) rows, fields 1..4, column 0 zeroed
      if ((g & 1) == 0) {
        st2(o, 0.0, r[0]);
        st2(o + 2, r[1], r[2]);
        o[4] = r[3];
      } else {
        o[0] = 0.0;
        st2(o + 1, r[0], r[1]);
        st2(o + 3, r[2], r[3]);
      }
      return;
    }
  }
#pragma unroll
  for (int ff = 0; ff < F; ++ff) o[A.of.f[ff]] = A.accumulate ? prev[ff] + r[ff] : r[ff];
  if (A.zero_mask && !A.accumulate)
    for (int zc = 0; zc < A.ldo; ++zc)
      if ((A.zero_mask >> zc) & 1u) o[zc] = 0.0;
}

// The two hot modes of slot_fixup_kernel<4> (H_nu's alpha = 2 on one GPU: slot rows of the tile-ordered
// intermediate, MODE 3; the (ng, 5) result rows of fields 1..4 with column 0 zeroed, MODE 2) without the
// generic kernel's segment / interface / accumulate paths: ~40 registers instead of 64, so 48 instead of 32
// warps per SM keep loads in flight.  Same sums in the same order (rows r ascending from 0.0).
template <int MODE>
__global__ void __launch_bounds__(256, MODE == 3 ? 6 : 5) slot_fixup_lean_kernel(TileArgs A) {
  constexpr int F = 4;
  const int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (id >= A.nslot * A.n_z) return;
  const unsigned nz = (unsigned)A.n_z;
  const int64_t s = (unsigned)id / nz;
  const int z = (int)((unsigned)id - (unsigned)s * nz);
  const int r0 = A.slot_row0[s], nc = A.slot_nc[s];
  int g = 0;
  if (MODE == 2) g = A.col_gid[(int64_t)A.slot_col[s] * A.n_z + z];
  const double mi = __ldg(A.Ms + id);
  const double* p0 = A.part + ((int64_t)r0 * A.n_z + z) * F;
  const int64_t rs = (int64_t)A.n_z * F;                  // doubles between a slot's consecutive partial rows
  double v0[F], v1[F], acc[F];
  load_row<F>(p0, v0);
  if (nc > 1) load_row<F>(p0 + rs, v1);
#pragma unroll
  for (int ff = 0; ff < F; ++ff) {
    acc[ff] = 0.0 + v0[ff];
    if (nc > 1) acc[ff] += v1[ff];
  }
  for (int r = 2; r < nc; ++r) {
    double w[F];
    load_row<F>(p0 + r * rs, w);
#pragma unroll
    for (int ff = 0; ff < F; ++ff) acc[ff] += w[ff];
  }
  double r[F];
#pragma unroll
  for (int ff = 0; ff < F; ++ff) r[ff] = A.scale * (mi * acc[ff]);
  if (MODE == 3) {
    const int N = (A.n_z - 1) / A.nlay;
    const int64_t row = (z == 0) ? s : A.nslot + (((int64_t)((z - 1) / N) * A.nslot + s) * N + (z - 1) % N);
    double* o = A.sv + row * F;
    st2(o, r[0], r[1]);
    st2(o + 2, r[2], r[3]);
  } else {   // row (0, r0, r1, r2, r3): parity-selected offsets, no divergent branch
    double* o = A.out + (int64_t)g * 5;
    const bool odd = (g & 1) != 0;
    o[odd ? 0 : 4] = odd ? 0.0 : r[3];
    st2(o + (odd ? 1 : 0), odd ? r[0] : 0.0, odd ? r[1] : r[0]);
    st2(o + (odd ? 3 : 2), odd ? r[2] : r[1], odd ? r[3] : r[2]);
  }
}

// 40-byte rows (5 doubles at element offset 5 r of a 16-byte aligned array) as one 8-byte and two 16-byte
// accesses with parity-selected offsets; Row5 keeps the raw pieces so that the selects, which wait for the
// data, happen where the values are used
struct Row5 {
  double a;
  double2 b, c;
};
__device__ __forceinline__ Row5 ld_row5_raw(const double* row, bool odd) {
  Row5 x;
  x.a = row[odd ? 0 : 4];
  x.b = *reinterpret_cast<const double2*>(row + (odd ? 1 : 0));
  x.c = *reinterpret_cast<const double2*>(row + (odd ? 3 : 2));
  return x;
}
__device__ __forceinline__ void row5_add(const Row5& x, bool odd, double (&v)[5]) {
  v[0] += odd ? x.a : x.b.x;
  v[1] += odd ? x.b.x : x.b.y;
  v[2] += odd ? x.b.y : x.c.x;
  v[3] += odd ? x.c.x : x.c.y;
  v[4] += odd ? x.c.y : x.a;
}

// The Euler column sweep's fix-up (5 fields into (ng, 5) rows, optionally accumulating; one GPU, no
// segments) without the generic kernel's other paths, rows moved in 16-byte pieces.  Same sums in the
// same order as slot_fixup_kernel<5>.
template <int ACC>
__global__ void __launch_bounds__(256, 5) slot_fixup_lean5_kernel(TileArgs A) {
  const int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (id >= A.nslot * A.n_z) return;
  const unsigned nz = (unsigned)A.n_z;
  const int64_t s = (unsigned)id / nz;
  const int z = (int)((unsigned)id - (unsigned)s * nz);
  const int r0 = A.slot_row0[s], nc = A.slot_nc[s];
  const int g = A.col_gid[(int64_t)A.slot_col[s] * A.n_z + z];
  const double mi = __ldg(A.Ms + id);
  const int64_t pr = (int64_t)r0 * A.n_z + z;             // first partial row; the next ones n_z rows apart
  const bool nzodd = A.n_z & 1;
  const bool odd0 = pr & 1, odd1 = odd0 != nzodd;
  double* o = A.out + (int64_t)g * 5;
  const bool oodd = g & 1;
  const Row5 x0 = ld_row5_raw(A.part + pr * 5, odd0);
  Row5 x1 = x0, xo = x0;
  if (nc > 1) x1 = ld_row5_raw(A.part + (pr + A.n_z) * 5, odd1);
  if (ACC) xo = ld_row5_raw(o, oodd);
  double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  row5_add(x0, odd0, acc);
  if (nc > 1) row5_add(x1, odd1, acc);
  for (int r = 2; r < nc; ++r) {
    const int64_t q = pr + (int64_t)r * A.n_z;
    const Row5 x = ld_row5_raw(A.part + q * 5, q & 1);
    row5_add(x, q & 1, acc);
  }
  double v[5];
#pragma unroll
  for (int ff = 0; ff < 5; ++ff) v[ff] = A.scale * (mi * acc[ff]);
  if (ACC) {
    double pv[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    row5_add(xo, oodd, pv);
#pragma unroll
    for (int ff = 0; ff < 5; ++ff) v[ff] = pv[ff] + v[ff];
  }
  o[oodd ? 0 : 4] = oodd ? v[0] : v[4];
  st2(o + (oodd ? 1 : 0), oodd ? v[1] : v[0], oodd ? v[2] : v[1]);
  st2(o + (oodd ? 3 : 2), oodd ? v[3] : v[2], oodd ? v[4] : v[3]);
}

template <int F>
int pack_f(const TileArgs& A, cudaStream_t st) {
  if (A.next <= 0) return HV_OK;
  const int64_t tot = A.next * A.n_z;
  slot_pack_kernel<F><<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(A);
  HV_LAUNCH_CHECK();
  return HV_OK;
}

template <int F>
int fixup_f(const TileArgs& A, cudaStream_t st) {
  const int nseg = A.seg > 0 ? (A.nlay + A.seg - 1) / A.seg : 1;
  const int N = (A.n_z - 1) / A.nlay;
  const int64_t nbi = (nseg > 1) ? A.ntiles * (nseg - 1) * (int64_t)((A.TX * N + 1) * (A.TY * N + 1)) : 0;
  if (nseg > 1 && (!A.bnd || !A.prow || A.io != 0 || A.slot_ext)) HV_FAIL(HV_ERR_INVALID, "slot_fixup: bad segment plan");
  if (A.nslot <= 0 && nbi == 0) return HV_OK;
  const int64_t tot = A.nslot * A.n_z + nbi;
  if (tot >= (int64_t)1 << 31) HV_FAIL(HV_ERR_UNSUPPORTED, "slot_fixup: %lld slot rows", (long long)tot);
  int row_mode = 0;
  if (A.io == 1 || A.io == 3) {   // pass 1 into the tile-ordered intermediate
    if (F != 4 || A.accumulate || !A.sv || A.slot_ext) HV_FAIL(HV_ERR_UNSUPPORTED, "slot_fixup: slot rows need F = 4");
    row_mode = 3;
  } else if (F == 4 && !A.accumulate && A.out && ((uintptr_t)A.out & 15) == 0) {
    if (A.ldo == 4 && !A.zero_mask && A.of.f[0] == 0 && A.of.f[1] == 1 && A.of.f[2] == 2 && A.of.f[3] == 3)
      row_mode = 1;
    else if (A.ldo == 5 && A.zero_mask == 1u && A.of.f[0] == 1 && A.of.f[1] == 2 && A.of.f[2] == 3 &&
             A.of.f[3] == 4)
      row_mode = 2;
  }
  if constexpr (F == 4) {
    if (nseg == 1 && !A.slot_ext && A.Ms && (row_mode == 2 || row_mode == 3)) {
      if (row_mode == 3) slot_fixup_lean_kernel<3><<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(A);
      else slot_fixup_lean_kernel<2><<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(A);
      HV_LAUNCH_CHECK();
      return HV_OK;
    }
  }
  if constexpr (F == 5) {
    const bool ident = A.of.f[0] == 0 && A.of.f[1] == 1 && A.of.f[2] == 2 && A.of.f[3] == 3 && A.of.f[4] == 4;
    if (nseg == 1 && !A.slot_ext && A.Ms && A.ldo == 5 && ident && !A.zero_mask && A.io == 0 && A.out &&
        ((uintptr_t)A.out & 15) == 0 && ((uintptr_t)A.part & 15) == 0) {
      if (A.accumulate) slot_fixup_lean5_kernel<1><<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(A);
      else slot_fixup_lean5_kernel<0><<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(A);
      HV_LAUNCH_CHECK();
      return HV_OK;
    }
  }
  slot_fixup_kernel<F><<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(A, row_mode);
  HV_LAUNCH_CHECK();
  return HV_OK;
}

}  // namespace

namespace hv {

int slot_pack(const TileArgs& A, int F, cudaStream_t st) {
  switch (F) {
    case 1: return pack_f<1>(A, st);
    case 4: return pack_f<4>(A, st);
    case 5: return pack_f<5>(A, st);
    default: HV_FAIL(HV_ERR_UNSUPPORTED, "slot_pack: F=%d", F);
  }
}

int slot_fixup(const TileArgs& A, int F, cudaStream_t st) {
  switch (F) {
    case 1: return fixup_f<1>(A, st);
    case 4: return fixup_f<4>(A, st);
    case 5: return fixup_f<5>(A, st);
    default: HV_FAIL(HV_ERR_UNSUPPORTED, "slot_fixup: F=%d", F);
  }
}

}  // namespace hv
