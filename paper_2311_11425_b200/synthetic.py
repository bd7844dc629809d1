"""Seeded synthetic inputs for the five BASELINE.json configurations (host, numpy).

No public benchmark suite is involved: BASELINE.json names only synthetic
meshes and states, so these generators stand in for them.
All arrays are generated on the HOST with ``numpy.random.default_rng(seed)``
(PCG64) and copied to the device, so the CUDA path and the CPU oracle see
bitwise-identical inputs within one process.  The smooth states go through
numpy's transcendental functions and a BLAS contraction (``T @ A``), whose
last-ulp rounding can depend on the host CPU's SIMD level; the parity
fixtures therefore store the exact input bytes (tests/golden/*.npz
``state``, checked against this generator in the build container by
tests/test_oracle_golden.py) and the GPU-side tests read those.

Interpretation choices for the config text (recorded, not guessed silently;
DESIGN.md §7 repeats them):

* c1/c2/c5 geometry: vertex lattice, interior vertices displaced by
  U(-0.1, 0.1) x element spacing per axis, boundary vertices fixed, trilinear
  map to the LGL nodes.  c2 uses the perturbation too (c5 says "same ...
  perturbed geometry generator").  c2's real aspect ratio is 2.5:1.
* c2/c5 state: 5 fields of sum_{0<=kx,ky,kz<=8, k!=0} a_k prod_d cos(2 pi k_d
  x_d / L_d + phi_{d,k_d}) with a_k ~ N(0,1)/|k|^2 and one phase per (axis,
  wavenumber) so the sum factorises, plus 1e-3 N(0,1) white noise.
* c3 state: sum over (kx,ky,kz) in [0,4]^3 and vertical k in [0,3] of
  a * prod_d cos(k_d xhat_d + phi) * cos(pi k zeta + psi), xhat = x/|x|,
  zeta = height/z_top, a ~ N(0,1)/(1+|k|^2+k^2), plus 1e-3 N(0,1) noise.
* c4 state: isentropic background with the Exner function held fixed when
  theta is perturbed: pi = 1 - g z/(c_p theta0), P = p0 pi^(c_p/R),
  rho = P/(R (theta0+theta') pi), Theta = rho theta; U = V = W = 0; z from
  the last-writer gridpoint coordinates (mesh.py:107 semantics).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .basis import lobatto

GEOM_SEED = 0
STATE_SEED = 1


# ------------------------------------------------------------------ geometry
def perturbed_box_coords(nx, ny, nv, N, extents, frac=0.1, seed=GEOM_SEED, perturb=True, ia_range=None):
    """Trilinear map of a (optionally) perturbed vertex lattice to LGL nodes.

    Element order e = (ia*ny + ib)*nv + l, the box order of mesh.py:246-257
    generalised to nx != ny.  ``ia_range = (ia0, ia1)`` generates only the
    x-slab ia0 <= ia < ia1 of the same global lattice (multi-GPU slabs: the
    vertex perturbation is drawn for the whole lattice, so every rank sees the
    same bits on a shared face); its elements are numbered locally.
    Returns coords (nelem,3,n,n,n), elem_layer, elem_hcol.
    """
    x1 = lobatto(N).nodes
    n = N + 1
    Lx, Ly, Lz = extents
    hx, hy, hz = Lx / nx, Ly / ny, Lz / nv
    vx = np.linspace(0.0, Lx, nx + 1)
    vy = np.linspace(0.0, Ly, ny + 1)
    vz = np.linspace(0.0, Lz, nv + 1)
    V = np.empty((nx + 1, ny + 1, nv + 1, 3))
    V[..., 0] = vx[:, None, None]
    V[..., 1] = vy[None, :, None]
    V[..., 2] = vz[None, None, :]
    if perturb:
        rng = np.random.default_rng(seed)
        d = rng.uniform(-frac, frac, size=(nx + 1, ny + 1, nv + 1, 3))
        d *= np.array([hx, hy, hz])
        interior = np.zeros((nx + 1, ny + 1, nv + 1), dtype=bool)
        interior[1:-1, 1:-1, 1:-1] = True
        V[interior] += d[interior]
    if ia_range is not None:
        ia0, ia1 = ia_range
        V = V[ia0:ia1 + 1]
        nx = ia1 - ia0
    s = 0.5 * (1.0 + x1)            # exact 0 and 1 at the end nodes
    S = (1.0 - s, s)
    nel = nx * ny * nv
    coords = np.empty((nx, ny, nv, 3, n, n, n))
    # separable trilinear map: contract the corner index along x, then y, then z
    for c in range(3):
        Vc = V[..., c]
        tx = [[Vc[0:nx, b:b + ny, d:d + nv, None] * S[0] + Vc[1:nx + 1, b:b + ny, d:d + nv, None] * S[1]
               for d in (0, 1)] for b in (0, 1)]                               # (nx,ny,nv,i)
        txy = [tx[0][d][..., :, None] * S[0][None, :] + tx[1][d][..., :, None] * S[1][None, :]
               for d in (0, 1)]                                                 # (nx,ny,nv,i,j)
        coords[:, :, :, c] = (txy[0][..., None] * S[0] + txy[1][..., None] * S[1])
    coords = coords.reshape(nel, 3, n, n, n)
    ia, ib, l = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nv), indexing="ij")
    layer = l.reshape(-1).astype(np.int64)
    hcol = (ia * ny + ib).reshape(-1).astype(np.int64)
    return coords, layer, hcol


def box_window_coords(ne, nv_full, N, extents, ia0, nx, ib0, ny, nv):
    """Elements [ia0, ia0+nx) x [ib0, ib0+ny) x layers [0, nv) of the ne x ne x nv_full box of
    ``build_box`` (mesh.py:231-258), with the same node coordinates bit for bit (the same
    linspace breakpoints and node formula), numbered locally e = (ia*ny + ib)*nv + l.

    Parity cases at a large config's own element geometry (config 4: 156.25 x 156.25 x 625 m
    elements) without the full mesh.  Returns coords (nelem,3,n,n,n), elem_layer, elem_hcol.
    """
    x1 = lobatto(N).nodes
    Lx, Ly, Lz = extents
    xs = np.linspace(0.0, Lx, ne + 1)
    ys = np.linspace(0.0, Ly, ne + 1)
    lev = np.linspace(0.0, 1.0, nv_full + 1) * Lz
    n = N + 1
    coords = np.empty((nx * ny * nv, 3, n, n, n))
    e = 0
    for a in range(nx):
        ia = ia0 + a
        x = 0.5 * (xs[ia] + xs[ia + 1]) + 0.5 * (xs[ia + 1] - xs[ia]) * x1
        for b in range(ny):
            ib = ib0 + b
            y = 0.5 * (ys[ib] + ys[ib + 1]) + 0.5 * (ys[ib + 1] - ys[ib]) * x1
            for l in range(nv):
                z = 0.5 * (lev[l] + lev[l + 1]) + 0.5 * (lev[l + 1] - lev[l]) * x1
                X, Y, Z = np.meshgrid(x, y, z, indexing="ij")
                coords[e] = np.stack([X, Y, Z])
                e += 1
    idx = np.arange(nx * ny * nv)
    return coords, (idx % nv).astype(np.int64), (idx // nv).astype(np.int64)


# ------------------------------------------------------------------- states
def _eval_modes(axes_fn, A, npts, nk, nfields, chunk, device):
    """out[p, f] = sum_k c0[p, kx] * (T[p, (rest)] @ A)[kx, f] chunk by chunk.

    ``axes_fn(s0, s1, xp)`` returns (c0 (m, nk), T (m, K)) for points s0:s1.
    With ``device`` (a torch device) the contraction runs there in float64
    (input generation only; the result is copied back to the host).
    """
    if device is None:
        out = np.empty((npts, nfields))
        for s0 in range(0, npts, chunk):
            s1 = min(npts, s0 + chunk)
            c0, T = axes_fn(s0, s1, np)
            U = (T @ A).reshape(s1 - s0, nk, nfields)
            out[s0:s1] = np.einsum("pk,pkf->pf", c0, U)
        return out
    import torch

    At = torch.from_numpy(A).to(device)
    out = torch.empty((npts, nfields), dtype=torch.float64, device=device)
    big = chunk * 64
    for s0 in range(0, npts, big):
        s1 = min(npts, s0 + big)
        c0, T = axes_fn(s0, s1, torch)
        U = (T @ At).reshape(s1 - s0, nk, nfields)
        out[s0:s1] = torch.einsum("pk,pkf->pf", c0, U)
    return out.cpu().numpy()


def keyed_normal(keys, nfields, seed=STATE_SEED, block_bits=20):
    """N(0,1) samples indexed by integer node keys instead of by local node order: key k takes row
    k mod 2^b of the block rng(seed, k >> b).  Ranks that share a node (slab faces) draw the same
    value for it without generating the whole global array."""
    keys = np.asarray(keys, dtype=np.int64)
    out = np.empty((keys.shape[0], nfields))
    blk = keys >> block_bits
    order = np.argsort(blk, kind="stable")
    bs = blk[order]
    cuts = np.flatnonzero(np.diff(bs)) + 1
    for part in np.split(order, cuts):
        if part.size == 0:
            continue
        b = int(blk[part[0]])
        draw = np.random.default_rng([seed, b]).standard_normal((1 << block_bits, nfields))
        out[part] = draw[keys[part] & ((1 << block_bits) - 1)]
    return out


def fourier_state(xg, extents, kmax=8, noise=1e-3, seed=STATE_SEED, nfields=5, chunk=1 << 16, device=None,
                  noise_keys=None):
    """Random Fourier modes (|k|^-2 amplitudes) plus white noise, (ng, nfields).

    ``noise_keys`` (ng,) int64: draw the white noise per global node key (keyed_normal) instead of
    in local node order -- multi-GPU slabs, whose shared face nodes must hold the same state on both
    ranks (the smooth part is a function of the coordinates, which agree bitwise on the faces)."""
    rng = np.random.default_rng(seed)
    nk = kmax + 1
    amp = rng.standard_normal((nfields, nk, nk, nk))
    kk = np.arange(nk, dtype=float)
    k2 = kk[:, None, None] ** 2 + kk[None, :, None] ** 2 + kk[None, None, :] ** 2
    k2[0, 0, 0] = np.inf
    amp = amp / k2[None]
    phase = rng.uniform(0.0, 2.0 * np.pi, size=(3, nk))
    white = rng.standard_normal((xg.shape[0], nfields)) if noise_keys is None else keyed_normal(
        noise_keys, nfields, seed)
    A = np.ascontiguousarray(amp.transpose(2, 3, 1, 0).reshape(nk * nk, nk * nfields))   # [(ky,kz),(kx,f)]
    if device is not None:
        import torch

        xgd = torch.from_numpy(np.ascontiguousarray(xg)).to(device)
        kkd, phd = torch.from_numpy(kk).to(device), torch.from_numpy(phase).to(device)

    def axes(s0, s1, xp):
        if xp is np:
            x, k_, ph = xg[s0:s1], kk, phase
        else:
            x, k_, ph = xgd[s0:s1], kkd, phd
        cs = [xp.cos(2.0 * np.pi * k_[None, :] * (x[:, d:d + 1] / extents[d]) + ph[d][None, :]) for d in range(3)]
        T = (cs[1][:, :, None] * cs[2][:, None, :]).reshape(s1 - s0, nk * nk)
        return cs[0], T

    return _eval_modes(axes, A, xg.shape[0], nk, nfields, chunk, device) + noise * white


def sphere_state(xg, radius, z_top, kmax=4, kvert=3, noise=1e-3, seed=STATE_SEED, nfields=5,
                 chunk=1 << 16, device=None):
    """Smooth spherical-harmonic-like data (restricted separable waves) plus noise."""
    rng = np.random.default_rng(seed)
    nk, nz = kmax + 1, kvert + 1
    amp = rng.standard_normal((nfields, nk, nk, nk, nz))
    kk = np.arange(nk, dtype=float)
    kz = np.arange(nz, dtype=float)
    k2 = (1.0 + kk[:, None, None, None] ** 2 + kk[None, :, None, None] ** 2
          + kk[None, None, :, None] ** 2 + kz[None, None, None, :] ** 2)
    amp = amp / k2[None]
    phase = rng.uniform(0.0, 2.0 * np.pi, size=(3, nk))
    vphase = rng.uniform(0.0, 2.0 * np.pi, size=nz)
    white = rng.standard_normal((xg.shape[0], nfields))
    A = np.ascontiguousarray(amp.transpose(2, 3, 4, 1, 0).reshape(nk * nk * nz, nk * nfields))
    if device is not None:
        import torch

        cvt = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(device)  # noqa: E731
        xgd, kkd, kzd, phd, vpd = cvt(xg), cvt(kk), cvt(kz), cvt(phase), cvt(vphase)

    def axes(s0, s1, xp):
        if xp is np:
            x, k_, kz_, ph, vp = xg[s0:s1], kk, kz, phase, vphase
        else:
            x, k_, kz_, ph, vp = xgd[s0:s1], kkd, kzd, phd, vpd
        r = xp.sqrt(x[:, 0] * x[:, 0] + x[:, 1] * x[:, 1] + x[:, 2] * x[:, 2])
        xh = x / r[:, None]
        zeta = (r - radius) / z_top
        cs = [xp.cos(k_[None, :] * xh[:, d:d + 1] + ph[d][None, :]) for d in range(3)]
        cv = xp.cos(np.pi * kz_[None, :] * zeta[:, None] + vp[None, :])
        T = (cs[1][:, :, None, None] * cs[2][:, None, :, None] * cv[:, None, None, :]).reshape(
            s1 - s0, nk * nk * nz)
        return cs[0], T

    return _eval_modes(axes, A, xg.shape[0], nk, nfields, chunk, device) + noise * white


def bubble_state_2c(xg, c_p=1004.5, c_v=717.5, g=9.80616, theta0=300.0, p0=1.0e5,
                    amp=0.5, radius=2000.0, centre=(5000.0, 5000.0, 2000.0)):
    """Set-2C state (rho, U, V, W, Theta) of the c4 warm bubble."""
    R = c_p - c_v
    z = xg[:, 2]
    dx = xg[:, 0] - centre[0]
    dy = xg[:, 1] - centre[1]
    dz = xg[:, 2] - centre[2]
    r = np.sqrt(dx * dx + dy * dy + dz * dz)
    tp = np.where(r < radius, amp * 0.5 * (1.0 + np.cos(np.pi * r / radius)), 0.0)
    exner = 1.0 - g * z / (c_p * theta0)
    P = p0 * exner ** (c_p / R)
    theta = theta0 + tp
    rho = P / (R * theta * exner)
    out = np.zeros((xg.shape[0], 5))
    out[:, 0] = rho
    out[:, 4] = rho * theta
    return out


# ------------------------------------------------------------------ configs
@dataclass
class Workload:
    """One BASELINE.json configuration, ready to build."""

    name: str
    geometry: str
    N: int
    alpha: int
    c: tuple
    dt: float
    operator: str                  # "laplacian" | "hyperdiff" | "euler+hyperdiff"
    nx: int = 0
    ny: int = 0
    nv: int = 0
    extents: tuple = (1.0, 1.0, 1.0)
    perturb: bool = False
    ne: int = 0                    # sphere panels per edge
    radius: float = 6.371e6
    z_top: float = 1.0e4
    set_name: str = "2C"
    fields_out: int = 4            # DOF-updates per global node per op
    notes: dict = field(default_factory=dict)


def workload(name, scale=1, slabs=1):
    """Named config.  ``scale`` shrinks element counts (parity cases), ``slabs`` = GPUs for c5."""
    if name == "c1":
        return Workload("c1", "box", 4, 1, (1.0, 1.0, 1.0), 1.0, "laplacian",
                        nx=8 // scale or 1, ny=8 // scale or 1, nv=4 // scale or 1,
                        extents=(8000.0, 8000.0, 2000.0), perturb=True, fields_out=5)
    if name == "c2":
        return Workload("c2", "box", 4, 2, (0.05, 0.05, 0.0), 0.5, "hyperdiff",
                        nx=32 // scale, ny=32 // scale, nv=8 // scale,
                        extents=(1.0e5 / scale, 1.0e5 / scale, 1.0e4 / scale), perturb=True)
    if name == "c3":
        return Workload("c3", "sphere", 4, 2, (0.1, 0.1, 0.01), 300.0, "hyperdiff",
                        ne=30 // scale, nv=10 // scale or 1, radius=6.371e6, z_top=1.0e4)
    if name == "c4":
        return Workload("c4", "box", 7, 2, (0.02, 0.02, 0.02), 0.1, "euler+hyperdiff",
                        nx=64 // scale, ny=64 // scale, nv=16 // scale,
                        extents=(1.0e4, 1.0e4, 1.0e4), perturb=False, set_name="2C",
                        fields_out=5)
    if name == "c5":
        e = 128 // scale
        v = 32 // scale
        return Workload("c5", "box", 4, 2, (0.05, 0.05, 0.0), 0.5, "hyperdiff",
                        nx=e * slabs, ny=e, nv=v,
                        extents=(3125.0 * e * slabs, 3125.0 * e, 1250.0 * v), perturb=True)
    raise ValueError(f"unknown workload {name!r}")


def make_mesh(w):
    """Build the product ``Mesh`` for a workload (numbering on the host in C++)."""
    from . import mesh as hm

    if w.geometry == "sphere":
        cfg = hm.MeshConfig("sphere", panels_per_edge=w.ne, n_elem_vertical=w.nv, degree=w.N,
                            radius=w.radius, z_top=w.z_top)
        return hm.build_cubed_sphere(cfg)
    if w.nx == w.ny and not w.perturb:
        cfg = hm.MeshConfig("box", panels_per_edge=w.nx, n_elem_vertical=w.nv, degree=w.N,
                            box_extents=tuple(w.extents))
        return hm.build_box(cfg)
    return hm.build_box_lattice(w.nx, w.ny, w.nv, w.N, w.extents, perturb=w.perturb)


def make_state(w, mesh, device=None):
    """Host state (ng, 5) for a workload (``device``: evaluate the smooth part there)."""
    if w.name in ("c1",):
        rng = np.random.default_rng(STATE_SEED)
        return rng.standard_normal((mesh.nglobal, 5))
    if w.name in ("c2", "c5"):
        return fourier_state(mesh.xg, w.extents, device=device)
    if w.name == "c3":
        return sphere_state(mesh.xg, w.radius, w.z_top, device=device)
    if w.name == "c4":
        return bubble_state_2c(mesh.xg)
    raise ValueError(w.name)
