/*
 * hv_b200.h -- C-ABI of the B200-native EBG hyper-diffusion / Euler-RHS library.
 *
 * The reference (hevicore, pure Python/numpy) has no native FFI; its operator
 * entry points are Python functions.  Each export below replaces the numerical
 * body of one reference function (file:line relative to
 * /root/reference/pkg/src/hevicore/), and the Python mirror package
 * paper_2311_11425_b200 binds them through ctypes (INTEGRATION.md shows the
 * binding a maintainer would add to the reference itself).
 *
 * Conventions
 *  - Plain pointers and sizes only.  "d_" pointers are CUDA device pointers,
 *    "h_" pointers are host pointers.  `stream` is a cudaStream_t passed as
 *    void* (0 = legacy default stream).  All device work is asynchronous on
 *    `stream`; functions that must report data-dependent errors (J <= 0,
 *    M <= 0, ...) synchronise the stream before returning.
 *  - Element arrays use the reference layout (nelem, n, n, n) with k fastest;
 *    the global state is (nglobal, ld) row-major (reference: (nglobal, 5)).
 *  - Return value: HV_OK (0) or an HV_ERR_* code; hv_last_error() gives a
 *    thread-local message.  The Python layer maps the codes onto the
 *    reference's exception types (ValueError / RuntimeError).
 *  - Only equal polynomial degree in the three directions is supported on the
 *    device (all BASELINE configurations); 1 <= N <= 8.
 */
#ifndef HV_B200_H
#define HV_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HV_ABI_VERSION 6

#define HV_OK 0
#define HV_ERR_INVALID 1        /* ValueError: bad argument / config                  */
#define HV_ERR_DEGENERATE 2     /* ValueError: J<=0, eigenvalue<=0, mass<=0 or ==0    */
#define HV_ERR_NONCONFORMING 3  /* RuntimeError: mesh.py:127-128,139-140              */
#define HV_ERR_CUDA 4           /* RuntimeError: CUDA runtime failure                 */
#define HV_ERR_NCCL 5           /* RuntimeError: collective failure                   */
#define HV_ERR_UNSUPPORTED 6    /* NotImplementedError                                */

int hv_abi_version(void);
const char* hv_last_error(void);
/* Number of CUDA kernels this library has launched in the process (bench.py's gpu_launches). */
int64_t hv_launch_count(void);
/* Measurement probe, not on the operator path: `blocks` x `threads` threads each run 8 independent
 * chains of `iters` dependent FP64 FMAs (2 * 8 * iters * blocks * threads FLOPs); bench.py times it
 * with CUDA events for the measured FP64 peak.  d_out: >= blocks * threads doubles. */
int hv_probe_dfma(double* d_out, int64_t iters, int blocks, int threads, void* stream);
/* Test probe, not on the operator path: d_out[i] = x_i^y with the power function the Euler kernels use
 * for the equation of state (state.py:84-101 calls numpy's power; csrc/hv_pow.cuh: <= 1 ulp for positive
 * normal x, the library pow otherwise). */
int hv_probe_pow(int64_t n, const double* d_x, double y, double* d_out, void* stream);
/* Test probe: counts in *d_bad (zeroed by the caller) the pairs (a_j, b_i), j = 0, 97, 194, ..., whose
 * quotient by the Euler kernels' reciprocal-and-correction division (csrc/hv_pow.cuh div_rcp) differs
 * bitwise from IEEE a_j / b_i. */
int hv_probe_div(int64_t n, const double* d_a, const double* d_b, unsigned long long* d_bad, void* stream);

/* ---------------------------------------------------------------- host mesh
 * Replaces Mesh._number_gridpoints (mesh.py:86-107): bit-exact gid
 * (first-appearance rank of each cluster of points within `tol`).
 * h_coords: (nelem, 3, n1, n2, n3); h_gid: (nelem*n1*n2*n3). */
int hv_number_gridpoints(const double* h_coords, int64_t nelem, int n1, int n2, int n3, double tol,
                         int64_t* h_gid, int64_t* nglobal);
/* mesh.py:106-107: xg[gid[p]] = pts[p], last writer wins. h_xg: (nglobal, 3). */
int hv_last_writer_coords(const double* h_coords, const int64_t* h_gid, int64_t nelem, int n1, int n2,
                          int n3, int64_t nglobal, double* h_xg);
/* Replaces Mesh._build_columns (mesh.py:109-145). h_col_gid: (nglobal/n_z, n_z). */
int hv_build_columns(const int64_t* h_gid, int64_t nelem, int n1, int n2, int n3, const int64_t* h_elem_layer,
                     const int64_t* h_elem_hcol, int64_t nglobal, int64_t nlay, int64_t* h_col_gid,
                     int64_t* h_col_of, int64_t* h_level_of, double* h_flux_mask, int64_t* ncol);
/* DSS gather map behind assembly.dss (assembly.py:17-26): for node g, the
 * local flat indices h_idx[h_off[g] .. h_off[g+1]) in increasing flat order,
 * so a sequential sum reproduces np.add.at bit for bit. */
int hv_build_dss_csr(const int64_t* h_gid, int64_t nloc, int64_t nglobal, int64_t* h_off, int32_t* h_idx);

/* ------------------------------------------------------------ metric setup
 * Replaces _covariant_basis/_jacobian/_cross/curl_invariant_metrics/
 * cross_product_metrics (metrics.py:49-110).  scheme 0 = curl-invariant,
 * 1 = cross-product.  Rounding-faithful to numpy's einsum order (bit-exact
 * with the reference on the reference's numpy build).
 * h_D: (n,n) derivative matrix (host); d_coords (nelem,3,n,n,n); outputs
 * d_dxdxi (nelem,3,3,n,n,n) [nullable], d_J (nelem,n,n,n), d_grad (nelem,3,3,n,n,n).
 * Returns HV_ERR_DEGENERATE if any J <= 0 (synchronises). */
int hv_metric_terms(int scheme, int N, const double* h_D, const double* d_coords, int64_t nelem,
                    double* d_dxdxi, double* d_J, double* d_grad, void* stream);

/* Sequential-order DSS of `ncomp` element fields through the CSR map:
 * d_out[g*ncomp + c] = sum_{p in csr(g)} d_fe[c*cstride + p]  (assembly.py:17-26). */
int hv_dss_csr(const double* d_fe, int ncomp, int64_t cstride, const int64_t* d_off, const int32_t* d_idx,
               int64_t nglobal, double* d_out, void* stream);

/* GlobalMass (assembly.py:54-64) and project_metrics_to_columns
 * (metrics.py:121-142).  d_w3 (n^3).  Outputs: d_M, d_Minv (nglobal) and,
 * if d_Jg != NULL, the projected d_Jg (nglobal) and d_gz (nglobal,3).
 * Returns HV_ERR_DEGENERATE for M <= 0 (synchronises). */
int hv_mass_and_projection(int N, const double* d_w3, const double* d_J, const double* d_grad, int64_t nelem,
                           const int64_t* d_off, const int32_t* d_idx, int64_t nglobal, double* d_M,
                           double* d_Minv, double* d_Jg, double* d_gz, void* stream);

/* The same two reductions split for the multi-GPU slab decomposition: raw
 * flat-order sums per node d_S (nglobal, 5) = [sum w3 J, sum (w3 J) J,
 * sum (w3 J) grad_zeta_c] (the host adds the neighbours' interface sums in
 * rank order), then M = S0, Minv = 1/M, Jg = S1/M, gz = S2..4/M (d_Jg nullable). */
int hv_mass_proj_sums(int N, const double* d_w3, const double* d_J, const double* d_grad, int64_t nelem,
                      const int64_t* d_off, const int32_t* d_idx, int64_t nglobal, double* d_S, void* stream);
int hv_mass_proj_finalize(int64_t nglobal, const double* d_S, double* d_M, double* d_Minv, double* d_Jg, double* d_gz,
                          void* stream);

/* build_viscous_metric (hyperdiff.py:54-81) fused with the packing of the
 * Laplacian metric W = w3 * Jg[gid] * G_nu (6 unique components).
 * mode 0 = scaled: nu_m*vals_m = ((a_m * lam_m) / b) * vals_m with host-computed
 *          a_m = c_m**(1/alpha) * 4, b = N**2 * dt**(1/alpha) (reference order);
 * mode 1 = constant (nu_m = h_nu[m]); mode 2 = anisotropic (nu_h, nu_h, nu_v) in h_nu.
 * Outputs (all nullable): d_Gnu (nelem*n^3, 3, 3), d_lam (.., 3), d_evecs (.., 3, 3),
 * d_W packed per DESIGN.md §3 (6, nelem*n^3) component-major.
 * Returns HV_ERR_DEGENERATE if an eigenvalue of G is <= 0 (synchronises). */
int hv_viscous_metric(int N, int mode, const double* h_a, double b, const double* h_nu, const double* d_grad,
                      int64_t nelem, const double* d_w3, const double* d_Jg, const int32_t* d_gid32,
                      double* d_Gnu, double* d_lam, double* d_evecs, double* d_W, void* stream);
/* Axis form of the Laplacian metric for scaled mode with c_1 == c_2 (every BASELINE config):
 * then G_nu = sum_m k_m e_m e_m^T (hyperdiff.py:80, k_m = nu_m vals_m = a_m / b) collapses to
 * k_h I + (k_v - k_h) e_3 e_3^T, e_3 the eigenvector of the largest eigenvalue of G (the same
 * Jacobi eigensolve as hv_viscous_metric), so W = w3 Jg G_nu = kh |u|^2 I + kd u u^T with
 * u = sqrt(w3 Jg[gid]) e_3.  ncomp = 3 writes d_U (3, nelem*n^3) component-major, half the bytes of
 * d_W, as u' = sqrt(scale w3 Jg[gid]) e_3 with scale = |kd| (what a wform-1 plan expects: the sweep
 * then forms (kh / kd) |u'|^2 d + u' (u' . d) and the sign of kd goes into the output scale).
 * Isotropic form (c_1 == c_2 == c_3, so k_v == k_h and G_nu = k_h I): ncomp = 1 writes
 * d_U[p] = scale * w3 Jg[gid] with scale = k_h, one double per node (no eigensolve).
 * Returns HV_ERR_DEGENERATE like hv_viscous_metric (ncomp = 3). */
int hv_viscous_axis(int N, const double* d_grad, int64_t nelem, const double* d_w3, const double* d_Jg,
                    const int32_t* d_gid32, int ncomp, double scale, double* d_U, void* stream);

/* ------------------------------------------------------------- hot path
 * Laplacian plan: everything laplacian_apply (hyperdiff.py:84-94) reads. */
typedef struct hv_lap_plan {
  int N;                       /* polynomial degree                               */
  double D[81];                /* (N+1)x(N+1) derivative matrix, row-major         */
  int64_t nelem, nglobal;
  const int32_t* d_gid;        /* (nelem*n^3) local -> global                      */
  const int64_t* d_off;        /* DSS CSR offsets (nglobal+1)                      */
  const int32_t* d_idx;        /* DSS CSR local indices (nelem*n^3)                */
  const double* d_W;           /* packed metric (6, nelem*n^3)                     */
  const double* d_Minv;        /* (nglobal)                                        */
  double* d_work;              /* element workspace, >= 5*nelem*n^3 doubles        */
  double* d_y;                 /* gridpoint workspace, >= 5*nglobal doubles        */
  /* optional tile-sweep plan (tiles.py); d_gt == NULL selects the
   * element-parallel path */
  int TX, TY, nlay, n_z;
  int64_t ntiles, nslot;
  const int32_t* d_gt;         /* (ntiles, nlay, GTS) tile node gids, (TX*N+1, TY*N+1, N+1)
                                  per layer padded to GTS = multiple of 4, -1 = absent */
  const int32_t* d_code;       /* (ntiles, TX*N+1, TY*N+1) -1 or partial row         */
  const int32_t* d_tmeta;      /* (ntiles, 2) active tile extent                     */
  const int32_t* d_slot_col;   /* (nslot) shared column ids                           */
  const int32_t* d_slot_row0;  /* (nslot) first partial row                           */
  const int32_t* d_slot_nc;    /* (nslot) owning tiles per shared column              */
  const int32_t* d_col_gid;    /* (ncol, n_z) int32 column gids                       */
  const double* d_Wt;          /* tiled packed metric                                 */
  const double* d_Mt;          /* Minv in tile order (ntiles, nlay, MTS)              */
  double* d_part;              /* partial rows (rows, n_z, F), >= rows*n_z*5 doubles   */
  int kernel;                  /* 0: line-tile kernel (lap_tile.cu), 1: plane-owner kernel (lap_plane.cu) */
  /* multi-GPU slab interface (parallel.py); d_slot_ext == NULL on one GPU */
  const int32_t* d_slot_ext;   /* (nslot) -1 or side*face + jf, side 0 = lower rank, 1 = upper   */
  const int32_t* d_ext_slots;  /* (next) slots with d_slot_ext >= 0                             */
  int64_t next;
  int face;                    /* column nodes per slab face                                   */
  double* d_send;              /* (2*face, n_z, F) local interface sums (NCCL send payload),   *
                                * F = fields of the pass; allocate for 5                        */
  double* d_recv;              /* (2*face, n_z, F) neighbour sums (NCCL receive buffer)        */
  /* form of d_Wt for the plane kernel (kernel == 1): 0 = the 6 components of W;
   * 1 = axis form (scaled mode with c_1 == c_2, hyperdiff.py:71-80: G_nu = k_h I + (k_v - k_h) e_3 e_3^T):
   * d_Wt holds u' = sqrt(|kd| w3 Jg[gid]) e_3 (3 components, hv_viscous_axis with scale = |kd|) and
   * W = kh |u|^2 I + kd u u^T = sgn(kd) [(kh / kd) |u'|^2 I + u' u'^T]; kd != 0;
   * 2 = isotropic form (c_1 == c_2 == c_3): s = kh w3 Jg[gid] (1 component), W = s I */
  int wform;
  double kh, kd;
  const double* d_Ms;          /* (nslot, n_z) Minv of the shared column nodes in slot order, or NULL */
  /* tile-ordered intermediate of H_nu's alpha = 2 (plane kernel, N = 4, 2x2 tiles, 4 fields; DESIGN.md
   * §4.2): pass 1 writes L q of the tile-owned nodes into d_yt in the sweep's own per-tile-layer
   * block layout and the perimeter nodes' partial sums into d_part; the slot fix-up writes their
   * final values as compact rows d_sv; pass 2 loads blocks and slot rows with bulk copies instead
   * of gathering by gid.  d_yt == NULL keeps the (nglobal, F) path. */
  const int32_t* d_tper;       /* (ntiles, NPER + 96): per tile the level offsets u*YUS + v of its slot
                                * columns in slot order, then 32 runs (first slot, count, position)   */
  double* d_yt;                /* (ntiles, nlay + 1, block) doubles (hv_plane_yt_layout)             */
  const int32_t* d_tchunk;     /* (ntiles, U*V + 1 + 128) or NULL: per tile the row-buffer row of each
                                * column's level 1, the number of runs, then 32 x (gid at layer 1, gid
                                * stride per layer, rows, row) -- pass 1 then bulk-copies its input's
                                * (nglobal, 5) rows (lattice-numbered meshes, tiles.build_chunk_table) */
  double* d_sv;                /* (nslot * n_z * 4) final values of the slot column nodes: [nslot][4]
                                * for z = 0, then per layer lb [nslot][N][4] for z = lb*N + 1 + kk   */
  /* vertical segments (plane kernel, N <= 4, one GPU): seg > 0 sweeps each tile as segments of seg
   * layers, one CTA each (more CTAs for meshes with few tiles); the levels between segments leave raw
   * sums in d_bnd that the slot fix-up completes.  seg = 0: whole columns. */
  int seg;
  double* d_bnd;               /* (ntiles, nseg - 1, 2, U*V, 5) boundary-level sums                      */
  const int32_t* d_prow;       /* (rows) partial row -> tile * U*V + u*V + v                             */
} hv_lap_plan;

/* Split Laplacian pass for the multi-GPU slab decomposition (the host runs the
 * neighbour exchange of d_send -> d_recv in between, ncclSend/ncclRecv):
 *   hv_lap_local : tile sweep; final values for tile-owned nodes, partial rows
 *                  for shared ones, local interface sums packed into d_send;
 *   hv_lap_finish: fixed-order sums of the shared nodes (interface: lower rank
 *                  first), times scale * Minv, into out.
 * Same argument meaning as hv_laplacian; zero_mask lists out columns to zero,
 * accumulate != 0 adds into out. */
int hv_lap_local(const hv_lap_plan* plan, const double* d_q, int64_t ldq, int nf, const int32_t* h_qf, double* d_out,
                 int64_t ldo, const int32_t* h_of, double scale, uint32_t zero_mask, int accumulate, void* stream);
/* hv_lap_local on the tiles [t0, t1) only (pack != 0: then pack the interface sums).  The
 * tile plan puts the tiles holding slab-interface columns first, so a pass can sweep them,
 * start the neighbour exchange and sweep the interior tiles while it is in flight. */
int hv_lap_local_tiles(const hv_lap_plan* plan, const double* d_q, int64_t ldq, int nf, const int32_t* h_qf,
                       double* d_out, int64_t ldo, const int32_t* h_of, double scale, uint32_t zero_mask, int accumulate,
                       int64_t t0, int64_t t1, int pack, void* stream);
int hv_lap_finish(const hv_lap_plan* plan, double* d_out, int64_t ldo, int nf, const int32_t* h_of, double scale,
                  uint32_t zero_mask, int accumulate, void* stream);

/* Reorder the packed metric W (6, nelem*n^3) into the tile-sweep layout
 * (layout 0: line-tile kernel, [t][l][pair][k][e][i*n+j][2]; layout 1: plane kernel,
 * [t][l][pair][i][k][e][j][2]; layout 2: plane kernel, axis form, d_W = U (3, nelem*n^3) of
 * hv_viscous_axis -> [t][l][c][i][k][e][j]; layout 3: plane kernel, isotropic form, d_W = s (nelem*n^3)
 * -> [t][l][i][k][e][j]) using d_elem (ntiles, nlay, TX*TY),
 * -1 for the absent elements of ragged tiles. */
/* Minv in tile order: d_Mt[r*mts + c] = d_Minv[d_gt[r*gts + c]] for the rows r = (tile, layer)
 * (0 for absent nodes and padding). */
int hv_tile_pack_minv(int64_t rows, int gts, int mts, const int32_t* d_gt, const double* d_Minv, double* d_Mt,
                      void* stream);
int hv_tile_pack_metric(int N, int TX, int TY, int64_t ntiles, int nlay, const int32_t* d_elem, const double* d_W,
                        int64_t nloc, int layout, double* d_Wt, void* stream);
/* Doubles per tile-layer of the plane kernel's packed metric in form wform (0: 6 components,
 * 1: axis, 2: isotropic -- rows padded for conflict-free shared-memory reads where tuned);
 * d_Wt of hv_tile_pack_metric holds ntiles * nlay of them.  -1 for bad arguments. */
int64_t hv_plane_metric_doubles(int N, int TX, int TY, int wform);
/* Block layout of the tile-ordered intermediate (d_yt): out[0..4] = (level stride, u stride, field
 * stride, doubles per tile-layer block, perimeter columns NPER per tile); the v stride is 1.
 * Perimeter column p of a tile: p < V: (u, v) = (0, p); p < 2V: (U-1, p-V); then (1 + r % (U-2),
 * 0 or V-1) for r = p - 2V (U = TX*N+1, V = TY*N+1).  Returns 0, or -1 when the plane kernel has
 * no tile-ordered mode for (N, TX, TY, F). */
int hv_plane_yt_layout(int N, int TX, int TY, int F, int64_t* out);
/* Row-buffer capacity (rows) of the plane kernel's bulk-copied pass-1 input (d_tchunk), -1 when the
 * plane kernel has no such mode for (N, TX, TY). */
int hv_plane_chunk_rows(int N, int TX, int TY);

/* y = scale * Minv * DSS(sum_m weak_m(W_mn d_n q)) on nf fields.
 * Input field f is d_q[g*ldq + h_qf[f]], output d_out[g*ldo + h_of[f]].
 * (hyperdiff.py:84-94 applied to nf fields in one pass; 1 <= nf <= 5.) */
int hv_laplacian(const hv_lap_plan* plan, const double* d_q, int64_t ldq, int nf, const int32_t* h_qf,
                 double* d_out, int64_t ldo, const int32_t* h_of, double scale, void* stream);

/* hyperdiffusion_apply (hyperdiff.py:97-106): out (nglobal, ldo) gets
 * (-1)^(alpha+1) L^alpha q on the nvar listed variables and 0 on every other
 * column of out (out[:,0] = 0 as in the reference). q is (nglobal, ldq).
 * accumulate != 0: out += H_nu(q) instead (rhs_horizontal's `out += ...`,
 * euler.py:130-133), other columns untouched. */
int hv_hyperdiffusion(const hv_lap_plan* plan, const double* d_q, int64_t ldq, int nvar, const int32_t* h_vars,
                      int alpha, double* d_out, int64_t ldo, int accumulate, void* stream);
/* One kernel of hv_hyperdiffusion's alpha = 2 on a single-GPU tile plan, for per-kernel timing
 * (bench.py): stage 1 = pass-1 sweep, 2 = pass-1 fix-up, 3 = pass-2 sweep, 4 = pass-2 fix-up;
 * stages 1..4 in order equal hv_hyperdiffusion(alpha = 2, accumulate = 0).  HV_ERR_UNSUPPORTED
 * for plans without a tile sweep. */
int hv_hyperdiffusion_stage(const hv_lap_plan* plan, const double* d_q, int64_t ldq, int nvar, const int32_t* h_vars,
                            double* d_out, int64_t ldo, int stage, void* stream);

/* ------------------------------------------------------------ Euler RHS
 * EulerOps._precompute element part (euler.py:39-59): per element node the
 * record read by hv_euler_rhs, component-major (18, nelem*n^3): grad xi (3),
 * grad eta (3), grad zeta gathered (3), Jg gathered (1), dPhi_m (3), flux mask
 * (1), Phi (1), rhat (3).  d_Phi_g / d_mask_g are gridpoint arrays. */
int hv_euler_setup(int N, const double* h_D, int64_t nelem, const int32_t* d_gid, const double* d_grad,
                   const double* d_Jg, const double* d_gz, const double* d_Phi_g, const double* d_mask_g,
                   const double* d_coords, int sphere, double* d_M, void* stream);
/* rhs_full (dirs = 7, coriolis 0 = rhat) / rhs_horizontal without H_nu (dirs = 3,
 * coriolis 1 = zetahat) for set_id 0 = 2NC, 1 = 2C, 2 = 3C (euler.py:111-129,
 * 159-224): element fluxes -> flat-order DSS -> Minv.  out (nglobal, ldo>=5)
 * receives the 5 tendencies (accumulate != 0: added). d_work >= 5*nelem*n^3. */
int hv_euler_rhs(int N, const double* h_D, int set_id, int dirs, int coriolis, double P_A, double R, double gamma,
                 double omega, int64_t nelem, int64_t nglobal, const int32_t* d_gid, const int32_t* d_elem_layer,
                 int nlay, const double* d_w3,
                 const double* d_M, const int64_t* d_off, const int32_t* d_idx, const double* d_Minv,
                 const double* d_q, int64_t ldq, double* d_work, double* d_out, int64_t ldo, int accumulate,
                 void* stream);

/* V(q), the vertical (zeta) operator of the HEVI split, column by column
 * (EulerOps.rhs_vertical / column_apply / _col_acc, euler.py:61-94,138-144,231-272):
 * per column of d_col_gid (ncol, n_z) int32 the layer accumulators, the zeta DSS
 * along the column and the division by the column mass DSS(w_z J).  h_w: the
 * (N+1) zeta quadrature weights.  out (nglobal, ldo) gets the 5 tendencies of
 * every gridpoint (accumulate != 0: added). */
int hv_euler_vertical(int N, const double* h_D, const double* h_w, int set_id, double P_A, double R, double gamma,
                      int64_t ncol, int nlay, int n_z, const int32_t* d_col_gid, const double* d_Jg,
                      const double* d_gz, const double* d_mask_g, const double* d_Phi_g, const double* d_q,
                      int64_t ldq, double* d_out, int64_t ldo, int accumulate, void* stream);

/* LHEVI column systems.
 * hv_column_jacobian: band batch of I - lam dV/dq for the columns of d_qcol
 *   (ncol, n_z, 5) (EulerOps.column_jacobian, euler.py:274-417), written to d_band
 *   (ncol, 2kl+ku+1, 5 n_z), kl = ku = 5 (N+1) - 1, LAPACK band layout.  d_col_gid
 *   (ncol, n_z) int32 maps the column nodes to gridpoints (J_g, grad zeta, mask, Phi).
 * hv_band_lu_factor: in-place batched band LU with partial pivoting
 *   (linalg.banded_lu_factor_batch, linalg.py:112-163); d_ipiv (nb, M) int32 pivot
 *   rows, d_info (nb) 0 or 1 + the first column with a zero pivot (SingularMatrixError).
 * hv_band_solve: d_x (nb, M) <- solution of the factored systems for the right-hand
 *   sides in d_x (linalg.banded_solve_batch, linalg.py:166-194). */
int hv_column_jacobian(int N, const double* h_D, const double* h_w, int set_id, double P_A, double R, double gamma,
                       double lam, int64_t ncol, int nlay, int n_z, const int32_t* d_col_gid, const double* d_qcol,
                       const double* d_Jg, const double* d_gz, const double* d_mask_g, const double* d_Phi_g,
                       double* d_band, void* stream);
int hv_band_lu_factor(double* d_data, int64_t nb, int kl, int ku, int M, int32_t* d_ipiv, int32_t* d_info,
                      void* stream);
int hv_band_solve(const double* d_data, const int32_t* d_ipiv, int64_t nb, int kl, int ku, int M, double* d_x,
                  void* stream);

/* hv_euler_rhs on a single-column tile plan (the N = 7 plan): the element accumulators of
 * each column are assembled on chip (vertical DSS carried between layers, tile-owned nodes
 * finished in the sweep, side-face nodes via partial rows + the fixed-order slot fix-up), no
 * (5 x nloc) work array.  d_elem: (ntiles, nlay) element of each tile layer. */
int hv_euler_rhs_tiles(const hv_lap_plan* plan, const int32_t* d_elem, const double* d_w3, int set_id, int dirs,
                       int coriolis, double P_A, double R, double gamma, double omega, const double* d_M,
                       const double* d_q, int64_t ldq, double* d_out, int64_t ldo, int accumulate, void* stream);

/* Multi-GPU Euler RHS (SURVEY §8(e) "other phases"): each rank runs hv_euler_rhs /
 * hv_euler_rhs_tiles with a unit mass (the raw DSS sums of its slab, euler.py:101-103 before the
 * division), the slab-face rows are exchanged and added in rank order, then
 * out[g, f] (+)= Minv[g] * raw[g, f] for f < nf (accumulate != 0: added, e.g. onto H_nu). */
int hv_rows_minv(double* d_out, int64_t ldo, const double* d_raw, int64_t ldr, const double* d_Minv, int64_t ng,
                 int nf, int accumulate, void* stream);

/* EulerOps.diagnostics (euler.py:421-456): d_out[7] = mass, energy_internal, energy_kinetic,
 * energy_potential, energy_total, p_surface_min, w_vertical_max.  d_M: the global mass (nglobal),
 * d_xg (nglobal, 3) only for the sphere (radial velocity), d_col_gid (ncol, n_z) int32 (surface
 * nodes = first column level), d_work >= 7 * 592 doubles.  Deterministic two-stage reduction. */
int hv_euler_diagnostics(int set_id, double P_A, double R, double gamma, double c_v, int sphere, int64_t ng,
                         const double* d_q, const double* d_M, const double* d_Phi_g, const double* d_xg, int64_t ncol,
                         int n_z, const int32_t* d_col_gid, double* d_work, double* d_out, void* stream);

/* assembly.elem_deriv / weak_deriv_acc (assembly.py:29-51) on (nelem, n, n, n) element data:
 * weak = 0: sum_a D[i,a] f_a along axis; weak = 1: -sum_a D[a,i] (w3 f)_a (d_w3: n^3 weights). */
int hv_elem_deriv(int N, const double* h_D, const double* d_w3, int64_t nelem, const double* d_f, int axis, int weak,
                  double* d_out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HV_B200_H */
