// Host-side connectivity builder (C++/OpenMP): conforming global numbering,
// last-writer gridpoint coordinates, vertical columns and the DSS CSR map.
//
// Replaces reference mesh.py:86-145 (Mesh._number_gridpoints / _build_columns)
// and the index bookkeeping behind assembly.py:17-26 (dss via np.add.at).
// Results are bit-exact with the reference:
//  * gid: the reference unions every KD-tree pair within `tol` with
//    union-by-min-root and ranks the roots with np.unique, i.e. gid is the
//    first-appearance rank (flat point order) of each connected component of
//    the "distance <= tol" graph.  We find exactly the same pairs with a
//    sorted uniform cell grid (cell = 1024*tol): pairs inside a cell are
//    tested directly, and a point closer than tol to a cell face also tests
//    the neighbouring cells, so no pair within tol is missed.
//  * xg: last writer in flat order (mesh.py:107).
//  * columns: first-seen bottom gid, hcol ascending then i, j (mesh.py:114-131).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstring>
#include <numeric>
#include <vector>

#include "hv_common.h"

#include <omp.h>
#include <parallel/algorithm>

template <class It, class Cmp>
static void hv_parallel_sort(It a, It b, Cmp cmp) {
  __gnu_parallel::sort(a, b, cmp);
}
static int hv_max_threads() { return omp_get_max_threads(); }
static int hv_thread_num() { return omp_get_thread_num(); }

namespace hv {
static thread_local char g_err[1024] = "";
void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
}  // namespace hv

namespace hv {
static std::atomic<int64_t> g_launches{0};
void count_launch(int64_t k) { g_launches.fetch_add(k, std::memory_order_relaxed); }
}  // namespace hv

extern "C" const char* hv_last_error(void) { return hv::g_err; }
extern "C" int64_t hv_launch_count(void) { return hv::g_launches.load(); }
extern "C" int hv_abi_version(void) { return HV_ABI_VERSION; }

namespace {

// point p of the flat (e, i, j, k) order, coordinate c, from coords (nelem,3,n1,n2,n3)
inline double coord(const double* coords, int64_t p, int c, int64_t nn) {
  int64_t e = p / nn, r = p % nn;
  return coords[(e * 3 + c) * nn + r];
}

}  // namespace

extern "C" int hv_number_gridpoints(const double* coords, int64_t nelem, int n1, int n2, int n3,
                                    double tol, int64_t* gid, int64_t* nglobal) {
  if (!coords || !gid || !nglobal || nelem <= 0 || n1 < 2 || n2 < 2 || n3 < 2 || !(tol > 0))
    HV_FAIL(HV_ERR_INVALID, "hv_number_gridpoints: invalid arguments");
  const int64_t nn = (int64_t)n1 * n2 * n3;
  const int64_t np_ = nelem * nn;
  const double tol2 = tol * tol;
  // bounding box -> cell size (>= 1024 tol, and <= 2^20 cells per axis so a key packs in 63 bits)
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  bool bad = false;
#pragma omp parallel
  {
    double l[3] = {INFINITY, INFINITY, INFINITY}, h[3] = {-INFINITY, -INFINITY, -INFINITY};
    bool b = false;
#pragma omp for schedule(static) nowait
    for (int64_t e = 0; e < nelem; ++e)
      for (int c = 0; c < 3; ++c)
        for (int64_t r = 0; r < nn; ++r) {
          const double v = coords[(e * 3 + c) * nn + r];
          if (!std::isfinite(v)) b = true;
          l[c] = std::min(l[c], v);
          h[c] = std::max(h[c], v);
        }
#pragma omp critical
    {
      bad |= b;
      for (int c = 0; c < 3; ++c) { lo[c] = std::min(lo[c], l[c]); hi[c] = std::max(hi[c], h[c]); }
    }
  }
  if (bad) HV_FAIL(HV_ERR_INVALID, "hv_number_gridpoints: non-finite coordinates");
  double span = std::max(hi[0] - lo[0], std::max(hi[1] - lo[1], hi[2] - lo[2]));
  const double h = std::max(1024.0 * tol, span / (double)(1 << 20));
  for (int c = 0; c < 3; ++c) lo[c] -= 2.0 * h;  // cell indices >= 1 (neighbours stay >= 0)
  auto cell_of = [&](double v, int c) -> uint64_t { return (uint64_t)std::floor((v - lo[c]) / h); };
  auto pack = [](uint64_t x, uint64_t y, uint64_t z) -> uint64_t { return (x << 42) | (y << 21) | z; };
  struct Rec {
    uint64_t key;
    int64_t p;
  };
  std::vector<Rec> rec(np_);
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < nelem; ++e)
    for (int64_t r = 0; r < nn; ++r) {
      const int64_t p = e * nn + r;
      rec[p] = Rec{pack(cell_of(coords[(e * 3 + 0) * nn + r], 0), cell_of(coords[(e * 3 + 1) * nn + r], 1),
                        cell_of(coords[(e * 3 + 2) * nn + r], 2)),
                   p};
    }
  auto rless = [](const Rec& a, const Rec& b) { return a.key != b.key ? a.key < b.key : a.p < b.p; };
  hv_parallel_sort(rec.data(), rec.data() + np_, rless);
  // cell starts
  std::vector<int64_t> starts;
  starts.reserve(np_ / 2 + 2);
  for (int64_t s = 0; s < np_; ++s)
    if (s == 0 || rec[s].key != rec[s - 1].key) starts.push_back(s);
  const int64_t ncell = (int64_t)starts.size();
  starts.push_back(np_);
  auto close = [&](int64_t a, int64_t b) {
    const int64_t ea = a / nn, ra = a % nn, eb = b / nn, rb = b % nn;
    double d2 = 0.0;
    for (int c = 0; c < 3; ++c) {
      const double d = coords[(ea * 3 + c) * nn + ra] - coords[(eb * 3 + c) * nn + rb];
      d2 += d * d;
    }
    return d2 <= tol2;
  };
  auto near_face = [&](int64_t p) {
    const int64_t e = p / nn, r = p % nn;
    for (int c = 0; c < 3; ++c) {
      const double v = coords[(e * 3 + c) * nn + r];
      const double f0 = lo[c] + (double)cell_of(v, c) * h;
      if (v - f0 <= tol || (f0 + h) - v <= tol) return true;
    }
    return false;
  };
  // parent forest: simple cells (a clique within tol, no point near a face) point at their
  // minimum index directly; the rest is resolved by union-find over exact pair tests.
  std::vector<int64_t> parent(np_);
  std::vector<int64_t> complex_cells;
#pragma omp parallel
  {
    std::vector<int64_t> mine;
#pragma omp for schedule(dynamic, 4096)
    for (int64_t c = 0; c < ncell; ++c) {
      const int64_t s0 = starts[c], s1 = starts[c + 1];
      bool simple = true;
      for (int64_t s = s0; s < s1 && simple; ++s) {
        if (near_face(rec[s].p)) simple = false;
        for (int64_t t = s + 1; t < s1 && simple; ++t)
          if (!close(rec[s].p, rec[t].p)) simple = false;
      }
      const int64_t root = rec[s0].p;  // smallest index of the cell (ties sorted by p)
      for (int64_t s = s0; s < s1; ++s) parent[rec[s].p] = simple ? root : rec[s].p;
      if (!simple) mine.push_back(c);
    }
#pragma omp critical
    complex_cells.insert(complex_cells.end(), mine.begin(), mine.end());
  }
  std::sort(complex_cells.begin(), complex_cells.end());
  auto find = [&](int64_t i) {
    while (parent[i] != i) {
      parent[i] = parent[parent[i]];
      i = parent[i];
    }
    return i;
  };
  auto unite = [&](int64_t a, int64_t b) {
    int64_t ra = find(a), rb = find(b);
    if (ra != rb) parent[std::max(ra, rb)] = std::min(ra, rb);
  };
  auto find_cell = [&](uint64_t k) -> int64_t {
    int64_t a = 0, b = ncell;
    while (a < b) {
      const int64_t mid = (a + b) / 2;
      if (rec[starts[mid]].key < k) a = mid + 1; else b = mid;
    }
    return (a < ncell && rec[starts[a]].key == k) ? a : -1;
  };
  for (int64_t c : complex_cells) {
    const int64_t s0 = starts[c], s1 = starts[c + 1];
    for (int64_t s = s0; s < s1; ++s)
      for (int64_t t = s + 1; t < s1; ++t)
        if (close(rec[s].p, rec[t].p)) unite(rec[s].p, rec[t].p);
    for (int64_t s = s0; s < s1; ++s) {
      const int64_t p = rec[s].p;
      if (!near_face(p)) continue;
      const int64_t e = p / nn, r = p % nn;
      int64_t kc[3];
      int dlo[3], dhi[3];
      for (int c3 = 0; c3 < 3; ++c3) {
        const double v = coords[(e * 3 + c3) * nn + r];
        kc[c3] = (int64_t)cell_of(v, c3);
        const double f0 = lo[c3] + (double)kc[c3] * h;
        dlo[c3] = (v - f0 <= tol) ? -1 : 0;
        dhi[c3] = ((f0 + h) - v <= tol) ? 1 : 0;
      }
      for (int dx = dlo[0]; dx <= dhi[0]; ++dx)
        for (int dy = dlo[1]; dy <= dhi[1]; ++dy)
          for (int dz = dlo[2]; dz <= dhi[2]; ++dz) {
            if (!dx && !dy && !dz) continue;
            const int64_t nc = find_cell(pack(kc[0] + dx, kc[1] + dy, kc[2] + dz));
            if (nc < 0) continue;
            for (int64_t t = starts[nc]; t < starts[nc + 1]; ++t)
              if (close(p, rec[t].p)) unite(p, rec[t].p);
          }
    }
  }
  // full compression (read-only walk), then first-appearance ranks of the min-index roots
  std::vector<int64_t> root(np_);
#pragma omp parallel for schedule(static)
  for (int64_t p = 0; p < np_; ++p) {
    int64_t i = p;
    while (parent[i] != i) i = parent[i];
    root[p] = i;
  }
  std::vector<int64_t>().swap(parent);
  std::vector<Rec>().swap(rec);
  // rank = exclusive prefix count of roots (== np.unique(roots) order)
  const int nt = hv_max_threads();
  std::vector<int64_t> part(nt + 1, 0);
#pragma omp parallel num_threads(nt)
  {
    const int t = hv_thread_num();
    const int64_t b0 = np_ * t / nt, b1 = np_ * (t + 1) / nt;
    int64_t cnt = 0;
    for (int64_t p = b0; p < b1; ++p) cnt += (root[p] == p);
    part[t + 1] = cnt;
#pragma omp barrier
#pragma omp single
    for (int k = 0; k < nt; ++k) part[k + 1] += part[k];
    int64_t r = part[t];
    for (int64_t p = b0; p < b1; ++p)
      if (root[p] == p) gid[p] = r++;
  }
#pragma omp parallel for schedule(static)
  for (int64_t p = 0; p < np_; ++p)
    if (root[p] != p) gid[p] = gid[root[p]];
  *nglobal = part[nt];
  return HV_OK;
}

extern "C" int hv_last_writer_coords(const double* coords, const int64_t* gid, int64_t nelem, int n1,
                                     int n2, int n3, int64_t nglobal, double* xg) {
  if (!coords || !gid || !xg || nelem <= 0) HV_FAIL(HV_ERR_INVALID, "hv_last_writer_coords: invalid arguments");
  const int64_t nn = (int64_t)n1 * n2 * n3, np_ = nelem * nn;
  for (int64_t p = 0; p < np_; ++p) {
    int64_t g = gid[p];
    if (g < 0 || g >= nglobal) HV_FAIL(HV_ERR_INVALID, "hv_last_writer_coords: gid out of range");
    for (int c = 0; c < 3; ++c) xg[g * 3 + c] = coord(coords, p, c, nn);
  }
  return HV_OK;
}

extern "C" int hv_build_columns(const int64_t* gid, int64_t nelem, int n1, int n2, int n3,
                                const int64_t* elem_layer, const int64_t* elem_hcol, int64_t nglobal,
                                int64_t nlay, int64_t* col_gid, int64_t* col_of, int64_t* level_of,
                                double* flux_mask, int64_t* ncol_out) {
  if (!gid || !elem_layer || !elem_hcol || !col_gid || !col_of || !level_of || !flux_mask || !ncol_out || nlay < 1)
    HV_FAIL(HV_ERR_INVALID, "hv_build_columns: invalid arguments");
  const int64_t nn = (int64_t)n1 * n2 * n3;
  const int64_t nz = nlay * (n3 - 1) + 1;
  if (nglobal % nz != 0) HV_FAIL(HV_ERR_NONCONFORMING, "column extraction missed gridpoints");
  const int64_t ncol_max = nglobal / nz;
  // hcol -> elements sorted by layer (stable for equal layers as np.argsort is not;
  // the reference requires distinct layers per column, checked below)
  std::vector<int64_t> idx(nelem);
  std::iota(idx.begin(), idx.end(), 0);
  std::stable_sort(idx.begin(), idx.end(), [&](int64_t a, int64_t b) {
    if (elem_hcol[a] != elem_hcol[b]) return elem_hcol[a] < elem_hcol[b];
    return elem_layer[a] < elem_layer[b];
  });
  std::vector<int64_t> col_of_bottom(nglobal, -1);
  std::vector<int64_t> g(nz);
  int64_t ncol = 0;
  for (int64_t s = 0; s < nelem;) {
    int64_t t = s;
    while (t < nelem && elem_hcol[idx[t]] == elem_hcol[idx[s]]) ++t;
    if (t - s != nlay) HV_FAIL(HV_ERR_NONCONFORMING, "non-conforming column detected");
    for (int i = 0; i < n1; ++i)
      for (int j = 0; j < n2; ++j) {
        for (int64_t l = 0; l < nlay; ++l) {
          const int64_t e = idx[s + l];
          for (int k = 0; k < n3; ++k) g[l * (n3 - 1) + k] = gid[e * nn + ((int64_t)i * n2 + j) * n3 + k];
        }
        const int64_t key = g[0];
        if (key < 0 || key >= nglobal) HV_FAIL(HV_ERR_INVALID, "gid out of range");
        if (col_of_bottom[key] >= 0) {
          const int64_t* prev = col_gid + col_of_bottom[key] * nz;
          for (int64_t z = 0; z < nz; ++z)
            if (prev[z] != g[z]) HV_FAIL(HV_ERR_NONCONFORMING, "non-conforming column detected");
        } else {
          if (ncol >= ncol_max) HV_FAIL(HV_ERR_NONCONFORMING, "non-conforming column detected");
          col_of_bottom[key] = ncol;
          std::memcpy(col_gid + ncol * nz, g.data(), nz * sizeof(int64_t));
          ++ncol;
        }
      }
    s = t;
  }
  for (int64_t p = 0; p < nglobal; ++p) { col_of[p] = -1; level_of[p] = -1; flux_mask[p] = 1.0; }
  for (int64_t c = 0; c < ncol; ++c)
    for (int64_t z = 0; z < nz; ++z) {
      col_of[col_gid[c * nz + z]] = c;
      level_of[col_gid[c * nz + z]] = z;
    }
  for (int64_t p = 0; p < nglobal; ++p)
    if (col_of[p] < 0) HV_FAIL(HV_ERR_NONCONFORMING, "column extraction missed gridpoints");
  for (int64_t c = 0; c < ncol; ++c) {
    flux_mask[col_gid[c * nz]] = 0.0;
    flux_mask[col_gid[c * nz + nz - 1]] = 0.0;
  }
  *ncol_out = ncol;
  return HV_OK;
}

extern "C" int hv_build_dss_csr(const int64_t* gid, int64_t nloc, int64_t nglobal, int64_t* offsets,
                                int32_t* idx) {
  if (!gid || !offsets || !idx || nloc <= 0 || nglobal <= 0 || nloc > INT32_MAX)
    HV_FAIL(HV_ERR_INVALID, "hv_build_dss_csr: invalid arguments");
  std::vector<int64_t> cnt(nglobal + 1, 0);
  for (int64_t p = 0; p < nloc; ++p) {
    if (gid[p] < 0 || gid[p] >= nglobal) HV_FAIL(HV_ERR_INVALID, "hv_build_dss_csr: gid out of range");
    ++cnt[gid[p] + 1];
  }
  for (int64_t g = 0; g < nglobal; ++g) cnt[g + 1] += cnt[g];
  std::memcpy(offsets, cnt.data(), (nglobal + 1) * sizeof(int64_t));
  for (int64_t p = 0; p < nloc; ++p) idx[cnt[gid[p]]++] = (int32_t)p;  // flat order within a node
  return HV_OK;
}
