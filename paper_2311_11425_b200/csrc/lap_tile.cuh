// Tile-sweep kernel arguments (see lap_tile.cu and tiles.py).
#pragma once
#include <cuda_runtime.h>

#include "lap_common.cuh"

namespace hv {

struct TileArgs {
  int TX, TY, nlay, n_z;
  int64_t ntiles, nslot;
  int64_t tile0, tile1;     // tile range of this launch: [tile0, tile1)
  const int32_t* gt;        // (ntiles, nlay, GTS) tile node gids (U*V*n used, padded to 4), -1 = absent
  const int32_t* code;      // (ntiles, U, V) -1 = tile-owned column node, else partial row
  const int32_t* tmeta;     // (ntiles, 2) active tx, ty of ragged tiles
  const int32_t* slot_col;  // (nslot) column id of each shared column node
  const int32_t* slot_row0; // (nslot) first partial row
  const int32_t* slot_nc;   // (nslot) number of owning tiles
  const int32_t* col_gid;   // (ncol, n_z) int32
  const double* Wt;         // tiled packed metric (ntiles, nlay, 3 pairs, n, NE, n*n, 2)
  const double* Mt;         // Minv in tile order (ntiles, nlay, MTS)
  const double* Minv;
  const double* q;
  int64_t ldq, ldo;
  FieldMap qf, of;
  unsigned zero_mask;
  int accumulate;            // out += result (no zeroing of other columns)
  double scale;
  double* out;
  double* part;             // (rows, n_z, 5)
  // slab-interface slots (multi-GPU, parallel.py); slot_ext == nullptr on one GPU
  const int32_t* slot_ext;  // (nslot) -1, or side * face + jf  (side 0: lower rank, 1: upper rank)
  const int32_t* ext_slots; // (next) slots with slot_ext >= 0
  int64_t next;
  int face;                 // column nodes per slab face
  double* send;             // (2 * face, n_z, F) local sums for the neighbours (F = fields of the pass)
  const double* recv;       // (2 * face, n_z, F) neighbours' sums
  int wform;                // Wt form (plane kernel): 0 = 6 components, 1 = axis form u (W = kh|u|^2 I + kd u u^T)
  double kh, kd;
  const double* Ms;         // (nslot, n_z) Minv in slot order (coalesced in slot_fixup), or nullptr
  // tile-ordered intermediate (plane kernel, hv_lap_plan::d_yt): io 1 = the pass writes its result
  // into the block chain at out (tile-owned nodes) and the perimeter nodes' raw partial sums into
  // their partial rows, whose fix-up writes the compact slot rows sv; io 2 = the pass reads its
  // input from the block chain at q and the slot rows sv by bulk copies; 0 = (nglobal, ld) rows
  int io;
  const int32_t* tper;      // (ntiles, NPER + 96) per tile: [stage position] u*YUS + v of its slot columns
                            // (in slot order), then 32 runs of consecutive slots (first slot, count, position)
  const int32_t* tchunk;    // (ntiles, U*V + 1 + 128) bulk-copy runs of a tile's q input (io 3, tiles.py)
  int64_t ng;               // rows of q (io 3: no bulk copy reads past row ng - 1)
  // vertical segments (plane kernel, io 0): seg > 0 sweeps each tile's columns as segments of seg layers
  // (one CTA each); the levels between segments leave raw partial sums in bnd, [tile][boundary][side
  // 0: from below, 1: from above][U*V][F], which slot_fixup completes (prow: partial row -> tile*U*V + uv)
  int seg;
  double* bnd;
  const int32_t* prow;
  double* sv;               // final values of the slot column nodes: [nslot][F] (z = 0), then per layer
                            // block lb: [nslot][N][F] (z = lb*N + 1 + kk)
};

bool tile_supported(int N, int TX, int TY, int F);
int slot_pack(const TileArgs& A, int F, cudaStream_t st);
int slot_fixup(const TileArgs& A, int F, cudaStream_t st);
bool plane_yt_layout(int N, int TX, int TY, int F, int64_t* lay);
int plane_chunk_rows(int N, int TX, int TY);
bool plane_supported(int N, int TX, int TY, int F);
int laplacian_plane(const TileArgs& A, int N, int F, const double* Drow, cudaStream_t st);
int plane_pack(int N, int TX, int TY, int64_t ntiles, int nlay, const int32_t* elem, const double* W, int64_t nloc,
               int axis, double* Wp, cudaStream_t st);
int64_t plane_metric_doubles(int N, int TX, int TY, int wform);
int laplacian_tile(const TileArgs& A, int N, int F, const double* Drow, cudaStream_t st);
int tile_pack_minv(int64_t rows, int gts, int mts, const int32_t* gt, const double* Minv, double* Mt, cudaStream_t st);
int tile_pack(int N, int NE, int64_t ntiles, int nlay, const int32_t* elem, const double* W, int64_t nloc,
              double* Wt, cudaStream_t st);

}  // namespace hv
