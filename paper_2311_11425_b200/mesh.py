"""Cubed-sphere and box spectral-element meshes with host C++ connectivity.

Mirror of the reference ``mesh`` module (mesh.py:23-262).  Element
coordinates are generated on the host with the reference's formulas (same
bits); the global numbering, last-writer gridpoint coordinates and the column
structure come from the C++ connectivity builder in ``libhv_b200.so``
(``hv_number_gridpoints`` / ``hv_build_columns``), bit-exact with the
reference's KD-tree + union-find + ``np.unique`` construction
(tests/test_mesh_numbering.py).  The device-side copies (int32 gid, DSS CSR
map, coordinates) are built lazily by :meth:`Mesh.device`.

Beyond the reference API, :func:`build_box_lattice` builds the rectangular,
optionally perturbed boxes of the BASELINE configs and records the panel
grid of element columns (``hgrid``) that the tile-sweep kernels use.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .basis import Basis1D, lobatto

__all__ = ["MeshConfig", "Mesh", "build_box", "build_cubed_sphere", "build_mesh", "build_box_lattice"]


@dataclass
class MeshConfig:
    """Mesh parameters (mesh.py:23-50)."""

    geometry: str
    panels_per_edge: int = 1
    n_elem_vertical: int = 1
    degree: int = 4
    degree_xi: int = None
    degree_eta: int = None
    degree_zeta: int = None
    radius: float = 6.371e6
    z_top: float = 3.0e4
    box_extents: tuple = (1.0, 1.0, 1.0)
    vertical_map: object = None

    def __post_init__(self):
        if self.geometry not in ("sphere", "box"):
            raise ValueError(f"unknown geometry {self.geometry!r}")
        if self.panels_per_edge < 1 or self.n_elem_vertical < 1:
            raise ValueError("element counts must be >= 1")
        if self.z_top <= 0:
            raise ValueError("z_top must be positive")
        for name in ("degree_xi", "degree_eta", "degree_zeta"):
            if getattr(self, name) is None:
                setattr(self, name, self.degree)
        if min(self.degree_xi, self.degree_eta, self.degree_zeta) < 1:
            raise ValueError("polynomial degrees must be >= 1")
        if self.geometry == "box" and min(self.box_extents) <= 0:
            raise ValueError("degenerate box extents")


class Mesh:
    """Element coordinates plus global numbering and column structure (mesh.py:53-171).

    coords (nelem,3,n1,n2,n3); gid (nelem,n1,n2,n3) int64; xg (nglobal,3);
    col_gid (ncol,n_z); col_of, level_of (nglobal,); flux_mask (nglobal,).
    """

    def __init__(self, cfg, coords, bases, elem_layer, elem_hcol, hgrid=None):
        self.cfg = cfg
        self.coords = np.ascontiguousarray(coords, dtype=np.float64)
        self.bases = bases
        self.nelem = self.coords.shape[0]
        self.shape = self.coords.shape[2:]
        self.elem_layer = np.ascontiguousarray(elem_layer, dtype=np.int64)
        self.elem_hcol = np.ascontiguousarray(elem_hcol, dtype=np.int64)
        self.n_z = cfg.n_elem_vertical * cfg.degree_zeta + 1
        self.hgrid = hgrid  # (npanel, nx, ny) with hcol = (p*nx + ia)*ny + ib, or None
        self._dev = None
        self._number_gridpoints()
        self._build_columns()

    def _dedupe_tol(self):
        """mesh.py:81-84."""
        if self.cfg.geometry == "sphere":
            return 1e-7 * self.cfg.radius / max(1.0, 10.0 * self.cfg.panels_per_edge)
        return 1e-9 * max(self.cfg.box_extents)

    def _number_gridpoints(self):
        L = _lib.lib()
        n1, n2, n3 = self.shape
        gid = np.empty(self.nelem * n1 * n2 * n3, dtype=np.int64)
        ng = C.c_int64(0)
        _lib.check(L.hv_number_gridpoints(self.coords.ctypes.data, self.nelem, n1, n2, n3,
                                          float(self._dedupe_tol()), gid.ctypes.data, C.addressof(ng)))
        self.nglobal = int(ng.value)
        self.gid = gid.reshape((self.nelem,) + tuple(self.shape))
        self.xg = np.zeros((self.nglobal, 3))
        _lib.check(L.hv_last_writer_coords(self.coords.ctypes.data, gid.ctypes.data, self.nelem, n1, n2, n3,
                                           self.nglobal, self.xg.ctypes.data))

    def _build_columns(self):
        L = _lib.lib()
        n1, n2, n3 = self.shape
        nlay = self.cfg.n_elem_vertical
        if self.nglobal % self.n_z:
            raise RuntimeError("column extraction missed gridpoints")
        ncol_max = self.nglobal // self.n_z
        col_gid = np.empty((ncol_max, self.n_z), dtype=np.int64)
        self.col_of = np.empty(self.nglobal, dtype=np.int64)
        self.level_of = np.empty(self.nglobal, dtype=np.int64)
        self.flux_mask = np.empty(self.nglobal)
        ncol = C.c_int64(0)
        _lib.check(L.hv_build_columns(self.gid.ctypes.data, self.nelem, n1, n2, n3, self.elem_layer.ctypes.data,
                                      self.elem_hcol.ctypes.data, self.nglobal, nlay, col_gid.ctypes.data,
                                      self.col_of.ctypes.data, self.level_of.ctypes.data,
                                      self.flux_mask.ctypes.data, C.addressof(ncol)))
        self.col_gid = col_gid[: ncol.value]
        self.ncol = int(ncol.value)
        self.elem_col = self.col_of[self.gid[:, :, :, 0]]

    # ---------------------------------------------------------------- geometry
    def height(self, x=None):
        """Height above the reference surface (mesh.py:149-154)."""
        x = self.xg if x is None else x
        if self.cfg.geometry == "sphere":
            return np.linalg.norm(x, axis=-1) - self.cfg.radius
        return x[..., 2]

    def lonlat(self, x=None):
        """(mesh.py:156-161)."""
        x = self.xg if x is None else x
        r = np.linalg.norm(x, axis=-1)
        return np.arctan2(x[..., 1], x[..., 0]), np.arcsin(np.clip(x[..., 2] / r, -1.0, 1.0))

    def summary(self):
        c = self.cfg
        return (f"geometry: {c.geometry}\nelements: {self.nelem}\ngridpoints: {self.nglobal}\n"
                f"columns: {self.ncol}\nn_z: {self.n_z}\n"
                f"degrees: {c.degree_xi} {c.degree_eta} {c.degree_zeta}\n")

    # ------------------------------------------------------------------ device
    @property
    def degree(self):
        c = self.cfg
        if not (c.degree_xi == c.degree_eta == c.degree_zeta):
            raise NotImplementedError("the B200 kernels support equal degrees in the three directions only")
        return c.degree_xi

    def device(self):
        """Device mirror (int32 gid, DSS CSR map, coords, w3), built once."""
        if self._dev is None:
            from .device import DeviceMesh

            self._dev = DeviceMesh(self)
        return self._dev


def _vertical_levels(cfg):
    """mesh.py:174-181."""
    s = np.linspace(0.0, 1.0, cfg.n_elem_vertical + 1)
    if cfg.vertical_map is not None:
        s = np.asarray([cfg.vertical_map(v) for v in s])
        if abs(s[0]) > 0 or abs(s[-1] - 1) > 1e-15 or np.any(np.diff(s) <= 0):
            raise ValueError("vertical_map must be increasing with endpoints 0, 1")
    return s


def _panel(p, t1, t2):
    """Unnormalised panel directions of the equiangular cube (mesh.py:184-192)."""
    one = np.ones_like(t1)
    if p == 0:
        return one, t1, t2
    if p == 1:
        return -t1, one, t2
    if p == 2:
        return -one, -t1, t2
    if p == 3:
        return t1, -one, t2
    if p == 4:
        return -t2, t1, one
    return t2, t1, -one


def build_cubed_sphere(cfg):
    """Equiangular cubed-sphere shell with radial extrusion (mesh.py:195-228)."""
    if cfg.geometry != "sphere":
        raise ValueError("config geometry must be 'sphere'")
    bx, be, bz = lobatto(cfg.degree_xi), lobatto(cfg.degree_eta), lobatto(cfg.degree_zeta)
    ne, nv = cfg.panels_per_edge, cfg.n_elem_vertical
    ang = np.linspace(-np.pi / 4, np.pi / 4, ne + 1)
    lev = _vertical_levels(cfg)
    # radial node positions of every layer: (nv, n3)
    r_lay = np.empty((nv, bz.npts))
    for l in range(nv):
        z0, z1 = cfg.z_top * lev[l], cfg.z_top * lev[l + 1]
        r_lay[l] = cfg.radius + (0.5 * (z0 + z1) + 0.5 * (z1 - z0) * bz.nodes)
    coords = np.empty((6, ne, ne, nv, 3, bx.npts, be.npts, bz.npts))
    for p in range(6):
        for ia in range(ne):
            a = 0.5 * (ang[ia] + ang[ia + 1]) + 0.5 * (ang[ia + 1] - ang[ia]) * bx.nodes
            for ib in range(ne):
                b = 0.5 * (ang[ib] + ang[ib + 1]) + 0.5 * (ang[ib + 1] - ang[ib]) * be.nodes
                t1, t2 = np.meshgrid(np.tan(a), np.tan(b), indexing="ij")
                dx, dy, dz = _panel(p, t1, t2)
                nrm = np.sqrt(dx * dx + dy * dy + dz * dz)
                d = np.stack([dx / nrm, dy / nrm, dz / nrm])
                coords[p, ia, ib] = d[None, :, :, :, None] * r_lay[:, None, None, None, :]
    nel = 6 * ne * ne * nv
    coords = coords.reshape(nel, 3, bx.npts, be.npts, bz.npts)
    idx = np.arange(nel)
    layer = (idx % nv).astype(np.int64)
    hcol = (idx // nv).astype(np.int64)
    return Mesh(cfg, coords, (bx, be, bz), layer, hcol, hgrid=(6, ne, ne))


def build_box(cfg):
    """Tensor-product brick, zeta along z (mesh.py:231-258)."""
    if cfg.geometry != "box":
        raise ValueError("config geometry must be 'box'")
    bx, be, bz = lobatto(cfg.degree_xi), lobatto(cfg.degree_eta), lobatto(cfg.degree_zeta)
    Lx, Ly, Lz = cfg.box_extents
    ne, nv = cfg.panels_per_edge, cfg.n_elem_vertical
    xs = np.linspace(0.0, Lx, ne + 1)
    ys = np.linspace(0.0, Ly, ne + 1)
    lev = _vertical_levels(cfg) * Lz
    X1 = 0.5 * (xs[:-1] + xs[1:])[:, None] + 0.5 * (xs[1:] - xs[:-1])[:, None] * bx.nodes[None, :]
    Y1 = 0.5 * (ys[:-1] + ys[1:])[:, None] + 0.5 * (ys[1:] - ys[:-1])[:, None] * be.nodes[None, :]
    Z1 = 0.5 * (lev[:-1] + lev[1:])[:, None] + 0.5 * (lev[1:] - lev[:-1])[:, None] * bz.nodes[None, :]
    n1, n2, n3 = bx.npts, be.npts, bz.npts
    coords = np.empty((ne, ne, nv, 3, n1, n2, n3))
    coords[:, :, :, 0] = X1[:, None, None, :, None, None]
    coords[:, :, :, 1] = Y1[None, :, None, None, :, None]
    coords[:, :, :, 2] = Z1[None, None, :, None, None, :]
    nel = ne * ne * nv
    idx = np.arange(nel)
    return Mesh(cfg, coords.reshape(nel, 3, n1, n2, n3), (bx, be, bz), (idx % nv).astype(np.int64),
                (idx // nv).astype(np.int64), hgrid=(1, ne, ne))


def build_mesh(cfg):
    return build_cubed_sphere(cfg) if cfg.geometry == "sphere" else build_box(cfg)


def build_box_lattice(nx, ny, nv, N, extents, perturb=True, frac=0.1, seed=0):
    """Rectangular nx x ny x nv box, trilinear map of an (optionally) perturbed
    vertex lattice (BASELINE configs 1, 2, 5; see synthetic.perturbed_box_coords)."""
    from .synthetic import perturbed_box_coords

    coords, layer, hcol = perturbed_box_coords(nx, ny, nv, N, extents, frac=frac, seed=seed, perturb=perturb)
    cfg = MeshConfig("box", panels_per_edge=max(nx, ny), n_elem_vertical=nv, degree=N,
                     box_extents=tuple(float(e) for e in extents))
    b = lobatto(N)
    return Mesh(cfg, coords, (b, b, b), layer, hcol, hgrid=(1, nx, ny))


def build_box_window(ne, nv_full, N, extents, ia0, nx, ib0, ny, nv):
    """A window of ``build_box``'s elements at their own coordinates (synthetic.box_window_coords):
    parity cases at a large configuration's element geometry (config 4)."""
    from .synthetic import box_window_coords

    coords, layer, hcol = box_window_coords(ne, nv_full, N, extents, ia0, nx, ib0, ny, nv)
    cfg = MeshConfig("box", panels_per_edge=max(nx, ny), n_elem_vertical=nv, degree=N,
                     box_extents=tuple(float(e) for e in extents))
    b = lobatto(N)
    return Mesh(cfg, coords, (b, b, b), layer, hcol, hgrid=(1, nx, ny))
