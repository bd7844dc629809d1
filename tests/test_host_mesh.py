"""Host C++ connectivity (libhv_b200.so) vs the reference: bit-exact gid/xg/columns.

Also pins the device metric arithmetic: the host build of metric_math.h
(hv_debug_metric_terms_host) must reproduce the reference's numpy metrics
bit for bit, which fixes the operation order the sm_100a kernel executes.
"""

from __future__ import annotations

import ctypes as C
import hashlib

import numpy as np
import pytest

from cases import CASES
from conftest import golden
from paper_2311_11425_b200 import _lib, basis, mesh as hm, synthetic
from product_cases import product_mesh


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _unused_product_mesh(name):
    c = CASES[name]
    if c["kind"] == "lattice":
        return hm.build_box_lattice(c["nx"], c["ny"], c["nv"], c["N"], c["extents"])
    if c["kind"] == "sphere":
        return hm.build_cubed_sphere(hm.MeshConfig("sphere", panels_per_edge=c["ne"], n_elem_vertical=c["nv"],
                                                   degree=c["N"], radius=c["radius"], z_top=c["z_top"]))
    return hm.build_box(hm.MeshConfig("box", panels_per_edge=c["ne"], n_elem_vertical=c["nv"], degree=c["N"],
                                      box_extents=c["extents"]))


@pytest.mark.parametrize("name", list(CASES))
def test_numbering_bit_exact(name):
    m = product_mesh(name)
    g = golden(name)
    assert m.nglobal == int(g["ng"])
    assert sha(m.gid) == str(g["sha_gid"])
    assert sha(m.xg) == str(g["sha_xg"])
    assert sha(m.col_gid) == str(g["sha_col_gid"])
    assert sha(m.flux_mask) == str(g["sha_flux_mask"])


@pytest.mark.parametrize("name", list(CASES))
def test_metric_order_host_build(name):
    m = product_mesh(name)
    g = golden(name)
    L = _lib.lib()
    N = m.degree
    n = N + 1
    D = np.ascontiguousarray(basis.lobatto(N).diff_matrix)
    for scheme, key in ((0, "sha_grad"), (1, "sha_grad_cross")):
        dx = np.empty((m.nelem, 3, 3, n, n, n))
        J = np.empty((m.nelem, n, n, n))
        gr = np.empty((m.nelem, 3, 3, n, n, n))
        _lib.check(L.hv_debug_metric_terms_host(scheme, N, D.ctypes.data, m.coords.ctypes.data, m.nelem,
                                                dx.ctypes.data, J.ctypes.data, gr.ctypes.data))
        assert sha(gr) == str(g[key]), (name, scheme)
        assert sha(J) == str(g["sha_J"])
        assert sha(dx) == str(g["sha_dxdxi"])


def test_sphere_numbering_larger():
    """Cubed-sphere corners (valence-3 columns) at a size the oracle still finishes."""
    from oracle import hevi_oracle as O

    cfg = hm.MeshConfig("sphere", panels_per_edge=5, n_elem_vertical=2, degree=3, radius=6.371e6, z_top=1.0e4)
    m = hm.build_cubed_sphere(cfg)
    coords, layer, hcol = O.sphere_coords(5, 2, 3, 6.371e6, 1.0e4)
    assert np.array_equal(coords, m.coords)
    gid, ng, xg = O.number_points(coords, O.dedupe_tol("sphere", 5))
    assert ng == m.nglobal and np.array_equal(gid, m.gid) and np.array_equal(xg, m.xg)
    col_gid, col_of, level_of, mask = O.build_columns(gid, ng, layer, hcol, 3)
    assert np.array_equal(col_gid, m.col_gid) and np.array_equal(mask, m.flux_mask)
    assert np.array_equal(col_of, m.col_of) and np.array_equal(level_of, m.level_of)


def test_box_builder_matches_reference_formula():
    from oracle import hevi_oracle as O

    m = hm.build_box(hm.MeshConfig("box", panels_per_edge=3, n_elem_vertical=2, degree=5,
                                   box_extents=(3.0, 2.0, 1.0)))
    coords, layer, hcol = O.box_coords(3, 2, 5, (3.0, 2.0, 1.0))
    assert np.array_equal(coords, m.coords)
    assert np.array_equal(layer, m.elem_layer) and np.array_equal(hcol, m.elem_hcol)


def test_dss_csr_flat_order():
    m = product_mesh("box_p_n4")
    L = _lib.lib()
    gid = m.gid.reshape(-1)
    off = np.empty(m.nglobal + 1, dtype=np.int64)
    idx = np.empty(gid.size, dtype=np.int32)
    _lib.check(L.hv_build_dss_csr(gid.ctypes.data, gid.size, m.nglobal, off.ctypes.data, idx.ctypes.data))
    # sequential sums through the map == np.add.at
    rng = np.random.default_rng(3)
    fe = rng.standard_normal(gid.size)
    ref = np.zeros(m.nglobal)
    np.add.at(ref, gid, fe)
    got = np.zeros(m.nglobal)
    for g in range(m.nglobal):
        s = 0.0
        for o in range(off[g], off[g + 1]):
            s = s + fe[idx[o]]
        got[g] = s
    assert np.array_equal(got, ref)
    assert np.all(np.diff(off) >= 1)
    # valence histogram of an interior-perturbed box: {1, 2, 4, 8}
    assert set(np.unique(np.diff(off))) <= {1, 2, 4, 8}


def test_nonconforming_columns_raise():
    m = product_mesh("box_p_n2_const")
    layer = m.elem_layer.copy()
    layer[0], layer[1] = layer[1], layer[0]  # element order inside a column no longer stacks
    with pytest.raises(RuntimeError):
        hm.Mesh(m.cfg, m.coords, m.bases, layer, m.elem_hcol)


def test_error_mapping():
    L = _lib.lib()
    with pytest.raises(ValueError):
        _lib.check(L.hv_number_gridpoints(None, 0, 1, 1, 1, 0.0, None, None))
