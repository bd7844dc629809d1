// C-ABI entry points of the hot path: hv_laplacian / hv_hyperdiffusion.
// hyperdiff.py:84-106 semantics; kernel selection (v1 element+CSR, or the tile
// sweep when the plan carries a tile map) happens here.
#include <cuda_runtime.h>

#include "hv_common.h"
#include "lap_common.cuh"
#include "lap_tile.cuh"

namespace {

__global__ void zero_cols_kernel(double* out, int64_t ng, int64_t ldo, unsigned keep_mask) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= ng * ldo) return;
  const int c = (int)(t % ldo);
  if (!((keep_mask >> c) & 1u)) out[t] = 0.0;
}

int check_plan(const hv_lap_plan* P) {
  if (!P) HV_FAIL(HV_ERR_INVALID, "null plan");
  if (P->N < 1 || P->N > 7) HV_FAIL(HV_ERR_UNSUPPORTED, "laplacian: degree %d not supported on the device (1..7)", P->N);
  if (P->nelem <= 0 || P->nglobal <= 0 || !P->d_gid || !P->d_off || !P->d_idx || !P->d_W || !P->d_Minv ||
      !P->d_work || !P->d_y)
    HV_FAIL(HV_ERR_INVALID, "incomplete laplacian plan");
  if (P->wform == 1 && !(P->kd != 0.0)) HV_FAIL(HV_ERR_INVALID, "axis-form plan with kd == 0 (use the isotropic form)");
  return HV_OK;
}

hv::TileArgs tile_args(const hv_lap_plan* P, const double* q, int64_t ldq, const hv::FieldMap& qf, double* out,
                       int64_t ldo, const hv::FieldMap& of, double scale, unsigned zero_mask, int accumulate) {
  hv::TileArgs A{};
  A.TX = P->TX; A.TY = P->TY; A.nlay = P->nlay; A.n_z = P->n_z;
  A.ntiles = P->ntiles; A.nslot = P->nslot; A.tile0 = 0; A.tile1 = P->ntiles;
  A.gt = P->d_gt; A.code = P->d_code; A.tmeta = P->d_tmeta;
  A.slot_col = P->d_slot_col; A.slot_row0 = P->d_slot_row0; A.slot_nc = P->d_slot_nc; A.col_gid = P->d_col_gid;
  A.Wt = P->d_Wt; A.Mt = P->d_Mt; A.Minv = P->d_Minv; A.q = q; A.ldq = ldq; A.ldo = ldo; A.qf = qf; A.of = of;
  A.zero_mask = zero_mask; A.accumulate = accumulate; A.scale = scale; A.out = out; A.part = P->d_part;
  A.slot_ext = P->d_slot_ext; A.ext_slots = P->d_ext_slots; A.next = P->d_slot_ext ? P->next : 0;
  A.face = P->face; A.send = P->d_send; A.recv = P->d_recv;
  A.wform = P->wform; A.kh = P->kh; A.kd = P->kd; A.Ms = P->d_Ms;
  if (P->wform == 1) {
    // axis form: d_Wt holds u' = sqrt(|kd| w3 Jg) e_3, so W = sgn(kd) [(kh / kd) |u'|^2 I + u' u'^T]:
    // the sweep forms the bracket (one FP64 multiply less per node and field), the sign goes into
    // the output scale
    A.kh = P->kh / P->kd;
    A.scale = (P->kd < 0.0) ? -scale : scale;
  }
  A.io = 0; A.tper = P->d_tper; A.sv = P->d_sv; A.tchunk = P->d_tchunk; A.ng = P->nglobal;
  A.seg = P->seg; A.bnd = P->d_bnd; A.prow = P->d_prow;
  return A;
}

bool use_plane(const hv_lap_plan* P, int nf) {
  return P->d_gt && P->d_Mt && P->kernel == 1 && hv::plane_supported(P->N, P->TX, P->TY, nf);
}
// The packed metric of a plan has ONE layout (P->kernel): the line-tile kernel may only run on a
// line-layout plan; field counts the plane kernel lacks on a plane-layout plan fall back to the
// element-parallel path.
bool use_tiles(const hv_lap_plan* P, int nf) {
  return use_plane(P, nf) ||
         (P->d_gt && P->d_Mt && P->kernel == 0 && hv::tile_supported(P->N, P->TX, P->TY, nf));
}

// alpha = 2 through the tile-ordered intermediate (plane kernel, N = 4, 2x2 tiles, 4 fields, one GPU)
bool use_yt(const hv_lap_plan* P, int nf, const double* out) {
  int64_t lay[5];
  return P->d_yt && P->d_tper && P->d_sv && P->seg <= 0 && use_plane(P, nf) && hv::plane_yt_layout(P->N, P->TX, P->TY, nf, lay) &&
         !(P->d_slot_ext && P->next > 0) && (reinterpret_cast<uintptr_t>(out) & 15) == 0;
}

// tile sweep over [t0, t1) (+ packing of the interface sums when pack != 0; no-op on one GPU)
int lap_local(const hv_lap_plan* P, const double* q, int64_t ldq, int nf, const hv::FieldMap& qf, double* out,
              int64_t ldo, const hv::FieldMap& of, double scale, unsigned zero_mask, cudaStream_t st, int accumulate,
              int64_t t0 = 0, int64_t t1 = -1, int pack = 1) {
  if ((reinterpret_cast<uintptr_t>(out) & 15) != 0)
    HV_FAIL(HV_ERR_INVALID, "hv_lap_local: the output must be 16-byte aligned");
  hv::TileArgs A = tile_args(P, q, ldq, qf, out, ldo, of, scale, zero_mask, accumulate);
  A.tile0 = t0;
  A.tile1 = (t1 < 0) ? P->ntiles : t1;
  const int rc = use_plane(P, nf) ? hv::laplacian_plane(A, P->N, nf, P->D, st) : hv::laplacian_tile(A, P->N, nf, P->D, st);
  if (rc) return rc;
  return pack ? hv::slot_pack(A, nf, st) : HV_OK;
}

int lap_finish(const hv_lap_plan* P, int nf, double* out, int64_t ldo, const hv::FieldMap& of, double scale,
               unsigned zero_mask, cudaStream_t st, int accumulate) {
  const hv::TileArgs A = tile_args(P, nullptr, 0, hv::FieldMap{}, out, ldo, of, scale, zero_mask, accumulate);
  return hv::slot_fixup(A, nf, st);
}

// Run one whole Laplacian pass (single GPU) with the best available kernel for this plan.
int lap_pass(const hv_lap_plan* P, const double* q, int64_t ldq, int nf, const hv::FieldMap& qf, double* out,
             int64_t ldo, const hv::FieldMap& of, double scale, unsigned zero_mask, cudaStream_t st,
             int accumulate = 0) {
  // the sweeps write output rows with 16-byte stores: an output not 16-byte aligned (a caller's
  // offset view) takes the element-parallel path, which stores doubles
  const bool aligned = (reinterpret_cast<uintptr_t>(out) & 15) == 0;
  if (use_tiles(P, nf) && aligned) {
    if (P->d_slot_ext && P->next > 0)
      HV_FAIL(HV_ERR_INVALID, "multi-GPU plan: use hv_lap_local / exchange / hv_lap_finish");
    int rc = lap_local(P, q, ldq, nf, qf, out, ldo, of, scale, zero_mask, st, accumulate);
    if (rc) return rc;
    return lap_finish(P, nf, out, ldo, of, scale, zero_mask, st, accumulate);
  }
  if (zero_mask && !accumulate) {
    const int64_t tot = P->nglobal * ldo;
    zero_cols_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(out, P->nglobal, ldo, ~zero_mask);
    HV_LAUNCH_CHECK();
  }
  return hv::laplacian_v1(P, q, ldq, nf, qf, out, ldo, of, scale, accumulate, st);
}

int field_maps(int nf, const int32_t* h_qf, int64_t ldq, const int32_t* h_of, int64_t ldo, hv::FieldMap& qf,
               hv::FieldMap& of) {
  if (nf < 1 || nf > 5 || !h_of || ldo < 1) HV_FAIL(HV_ERR_INVALID, "bad field map");
  for (int f = 0; f < nf; ++f) {
    if (h_of[f] < 0 || h_of[f] >= ldo) HV_FAIL(HV_ERR_INVALID, "output field index out of range");
    of.f[f] = h_of[f];
    if (h_qf) {
      if (h_qf[f] < 0 || h_qf[f] >= ldq) HV_FAIL(HV_ERR_INVALID, "input field index out of range");
      qf.f[f] = h_qf[f];
    }
  }
  return HV_OK;
}

}  // namespace

extern "C" int hv_tile_pack_metric(int N, int TX, int TY, int64_t ntiles, int nlay, const int32_t* d_elem,
                                   const double* d_W, int64_t nloc, int layout, double* d_Wt, void* stream) {
  if (N < 1 || N > 8 || TX < 1 || TY < 1 || ntiles <= 0 || nlay <= 0 || !d_elem || !d_W || !d_Wt)
    HV_FAIL(HV_ERR_INVALID, "hv_tile_pack_metric: bad arguments");
  if (layout >= 1 && layout <= 3 && hv::plane_supported(N, TX, TY, 4))
    return hv::plane_pack(N, TX, TY, ntiles, nlay, d_elem, d_W, nloc, layout - 1, d_Wt, (cudaStream_t)stream);
  if (layout >= 2) HV_FAIL(HV_ERR_UNSUPPORTED, "hv_tile_pack_metric: axis / isotropic form needs the plane kernel");
  return hv::tile_pack(N, TX * TY, ntiles, nlay, d_elem, d_W, nloc, d_Wt, (cudaStream_t)stream);
}

extern "C" int64_t hv_plane_metric_doubles(int N, int TX, int TY, int wform) {
  if (N < 1 || N > 7 || TX < 1 || TY < 1 || wform < 0 || wform > 2) return -1;
  return hv::plane_metric_doubles(N, TX, TY, wform);
}

extern "C" int hv_plane_chunk_rows(int N, int TX, int TY) { return hv::plane_chunk_rows(N, TX, TY); }

extern "C" int hv_plane_yt_layout(int N, int TX, int TY, int F, int64_t* out) {
  if (!out) return -1;
  return hv::plane_yt_layout(N, TX, TY, F, out) ? 0 : -1;
}

extern "C" int hv_tile_pack_minv(int64_t rows, int gts, int mts, const int32_t* d_gt, const double* d_Minv,
                                 double* d_Mt, void* stream) {
  if (rows <= 0 || gts <= 0 || mts <= 0 || !d_gt || !d_Minv || !d_Mt) HV_FAIL(HV_ERR_INVALID, "hv_tile_pack_minv: bad args");
  return hv::tile_pack_minv(rows, gts, mts, d_gt, d_Minv, d_Mt, (cudaStream_t)stream);
}

extern "C" int hv_lap_local(const hv_lap_plan* P, const double* d_q, int64_t ldq, int nf, const int32_t* h_qf,
                            double* d_out, int64_t ldo, const int32_t* h_of, double scale, uint32_t zero_mask,
                            int accumulate, void* stream) {
  int rc = check_plan(P);
  if (rc) return rc;
  hv::FieldMap qf{}, of{};
  if ((rc = field_maps(nf, h_qf, ldq, h_of, ldo, qf, of))) return rc;
  if (!h_qf || !d_q || !d_out) HV_FAIL(HV_ERR_INVALID, "hv_lap_local: null argument");
  if (!use_tiles(P, nf)) HV_FAIL(HV_ERR_UNSUPPORTED, "hv_lap_local needs a tile plan");
  return lap_local(P, d_q, ldq, nf, qf, d_out, ldo, of, scale, zero_mask, (cudaStream_t)stream, accumulate);
}

extern "C" int hv_lap_local_tiles(const hv_lap_plan* P, const double* d_q, int64_t ldq, int nf, const int32_t* h_qf,
                                  double* d_out, int64_t ldo, const int32_t* h_of, double scale, uint32_t zero_mask,
                                  int accumulate, int64_t t0, int64_t t1, int pack, void* stream) {
  int rc = check_plan(P);
  if (rc) return rc;
  hv::FieldMap qf{}, of{};
  if ((rc = field_maps(nf, h_qf, ldq, h_of, ldo, qf, of))) return rc;
  if (!h_qf || !d_q || !d_out) HV_FAIL(HV_ERR_INVALID, "hv_lap_local_tiles: null argument");
  if (!use_tiles(P, nf)) HV_FAIL(HV_ERR_UNSUPPORTED, "hv_lap_local_tiles needs a tile plan");
  if (t0 < 0 || t1 > P->ntiles || t0 > t1) HV_FAIL(HV_ERR_INVALID, "hv_lap_local_tiles: bad tile range");
  return lap_local(P, d_q, ldq, nf, qf, d_out, ldo, of, scale, zero_mask, (cudaStream_t)stream, accumulate, t0, t1,
                   pack);
}

extern "C" int hv_lap_finish(const hv_lap_plan* P, double* d_out, int64_t ldo, int nf, const int32_t* h_of,
                             double scale, uint32_t zero_mask, int accumulate, void* stream) {
  int rc = check_plan(P);
  if (rc) return rc;
  hv::FieldMap qf{}, of{};
  if ((rc = field_maps(nf, nullptr, 0, h_of, ldo, qf, of))) return rc;
  if (!d_out) HV_FAIL(HV_ERR_INVALID, "hv_lap_finish: null output");
  return lap_finish(P, nf, d_out, ldo, of, scale, zero_mask, (cudaStream_t)stream, accumulate);
}

extern "C" int hv_laplacian(const hv_lap_plan* P, const double* d_q, int64_t ldq, int nf, const int32_t* h_qf,
                            double* d_out, int64_t ldo, const int32_t* h_of, double scale, void* stream) {
  int rc = check_plan(P);
  if (rc) return rc;
  if (nf < 1 || nf > 5 || !d_q || !d_out || !h_qf || !h_of || ldq < 1 || ldo < 1)
    HV_FAIL(HV_ERR_INVALID, "hv_laplacian: bad arguments");
  hv::FieldMap qf{}, of{};
  for (int f = 0; f < nf; ++f) {
    if (h_qf[f] < 0 || h_qf[f] >= ldq || h_of[f] < 0 || h_of[f] >= ldo)
      HV_FAIL(HV_ERR_INVALID, "hv_laplacian: field index out of range");
    qf.f[f] = h_qf[f];
    of.f[f] = h_of[f];
  }
  return lap_pass(P, d_q, ldq, nf, qf, d_out, ldo, of, scale, 0u, (cudaStream_t)stream);
}

namespace {

// hv_hyperdiffusion; stage 0 = the whole op, stages 1..4 = one kernel of alpha = 2 on a tile plan
// (pass-1 sweep, pass-1 fix-up, pass-2 sweep, pass-2 fix-up; hv_hyperdiffusion_stage)
int hyperdiffusion(const hv_lap_plan* P, const double* d_q, int64_t ldq, int nvar, const int32_t* h_vars, int alpha,
                   double* d_out, int64_t ldo, int accumulate, cudaStream_t st, int stage) {
  int rc = check_plan(P);
  if (rc) return rc;
  if (alpha != 1 && alpha != 2) HV_FAIL(HV_ERR_INVALID, "alpha must be 1 or 2");
  if (nvar < 0 || nvar > 5 || !d_q || !d_out || ldo < 1 || ldo > 32 || ldq < 1)
    HV_FAIL(HV_ERR_INVALID, "hv_hyperdiffusion: bad arguments");
  unsigned keep = 0;
  hv::FieldMap qf{}, of{}, yf{};
  for (int v = 0; v < nvar; ++v) {
    if (h_vars[v] == 0) HV_FAIL(HV_ERR_INVALID, "hyper-diffusing density is out of scope");
    if (h_vars[v] < 0 || h_vars[v] >= ldq || h_vars[v] >= ldo) HV_FAIL(HV_ERR_INVALID, "variable index out of range");
    qf.f[v] = of.f[v] = h_vars[v];
    yf.f[v] = v;
    keep |= 1u << h_vars[v];
  }
  const unsigned zmask = ((ldo >= 32) ? 0xffffffffu : ((1u << ldo) - 1u)) & ~keep;
  if (stage && (alpha != 2 || nvar == 0 || !use_tiles(P, nvar) || (P->d_slot_ext && P->next > 0) ||
                (reinterpret_cast<uintptr_t>(d_out) & 15) != 0))
    HV_FAIL(HV_ERR_UNSUPPORTED, "hv_hyperdiffusion_stage: alpha = 2 on a single-GPU tile plan only");
  if (nvar == 0) {
    if (accumulate) return HV_OK;
    const int64_t tot = P->nglobal * ldo;
    zero_cols_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(d_out, P->nglobal, ldo, 0u);
    HV_LAUNCH_CHECK();
    return HV_OK;
  }
  const double sign = (alpha % 2 == 1) ? 1.0 : -1.0;  // (-1)^(alpha+1)
  if (alpha == 1) return lap_pass(P, d_q, ldq, nvar, qf, d_out, ldo, of, sign, zmask, st, accumulate);
  const bool all = stage == 0;
  if (use_yt(P, nvar, d_out)) {
    // pass 1: q -> tile-ordered y blocks + perimeter partial rows, whose fix-up writes the compact slot
    // rows; pass 2: blocks and slot rows by bulk copy -> out rows (+ the usual slot fix-up)
    hv::TileArgs A1 = tile_args(P, d_q, ldq, qf, P->d_yt, 0, yf, 1.0, 0u, 0);
    // the input by bulk copies of its gid runs when the plan has a chunk table (rows of 5 doubles)
    A1.io = (P->d_tchunk && ldq == 5 && (reinterpret_cast<uintptr_t>(d_q) & 15) == 0) ? 3 : 1;
    if ((all || stage == 1) && (rc = hv::laplacian_plane(A1, P->N, nvar, P->D, st))) return rc;
    if ((all || stage == 2) && (rc = hv::slot_fixup(A1, nvar, st))) return rc;
    hv::TileArgs A2 = tile_args(P, P->d_yt, 0, yf, d_out, ldo, of, sign, zmask, accumulate);
    A2.io = 2;
    if ((all || stage == 3) && (rc = hv::laplacian_plane(A2, P->N, nvar, P->D, st))) return rc;
    if (all || stage == 4) return lap_finish(P, nvar, d_out, ldo, of, sign, zmask, st, accumulate);
    return HV_OK;
  }
  if (all) {
    rc = lap_pass(P, d_q, ldq, nvar, qf, P->d_y, nvar, yf, 1.0, 0u, st);
    if (rc) return rc;
    return lap_pass(P, P->d_y, nvar, nvar, yf, d_out, ldo, of, sign, zmask, st, accumulate);
  }
  if (stage == 1) return lap_local(P, d_q, ldq, nvar, qf, P->d_y, nvar, yf, 1.0, 0u, st, 0);
  if (stage == 2) return lap_finish(P, nvar, P->d_y, nvar, yf, 1.0, 0u, st, 0);
  if (stage == 3) return lap_local(P, P->d_y, nvar, nvar, yf, d_out, ldo, of, sign, zmask, st, accumulate);
  if (stage == 4) return lap_finish(P, nvar, d_out, ldo, of, sign, zmask, st, accumulate);
  HV_FAIL(HV_ERR_INVALID, "hv_hyperdiffusion_stage: stage must be 1..4");
}

}  // namespace

extern "C" int hv_hyperdiffusion(const hv_lap_plan* P, const double* d_q, int64_t ldq, int nvar,
                                 const int32_t* h_vars, int alpha, double* d_out, int64_t ldo, int accumulate,
                                 void* stream) {
  return hyperdiffusion(P, d_q, ldq, nvar, h_vars, alpha, d_out, ldo, accumulate, (cudaStream_t)stream, 0);
}

extern "C" int hv_hyperdiffusion_stage(const hv_lap_plan* P, const double* d_q, int64_t ldq, int nvar,
                                       const int32_t* h_vars, double* d_out, int64_t ldo, int stage, void* stream) {
  if (stage < 1 || stage > 4) HV_FAIL(HV_ERR_INVALID, "hv_hyperdiffusion_stage: stage must be 1..4");
  return hyperdiffusion(P, d_q, ldq, nvar, h_vars, 2, d_out, ldo, 0, (cudaStream_t)stream, stage);
}
