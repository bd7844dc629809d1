"""Host tile plan (tiles.py) invariants, CPU only.

The sweep kernels trust the plan: every element is swept exactly once, every
tile column-node either belongs to one tile (reduced on chip) or is a slot whose
partial rows are numbered densely in (column, tile) order, and for a slab the
interface tiles come first (parallel.py overlaps their exchange with the rest).
"""

from __future__ import annotations

import numpy as np
import pytest

from paper_2311_11425_b200 import mesh as hm, parallel
from paper_2311_11425_b200.tiles import build_tile_plan


def _check_plan(m, p):
    N, n = m.degree, m.degree + 1
    # every element exactly once, ragged tiles padded with -1
    e = p.elem[p.elem >= 0]
    assert np.array_equal(np.sort(e), np.arange(m.nelem))
    # tile node gids reproduce the element gids
    gt = p.gt[:, :, :p.nodes].reshape(p.ntiles, p.nlay, p.U, p.V, n)
    for a in range(p.TX):
        for b in range(p.TY):
            eab = p.elem[:, :, a, b]
            sel = eab >= 0
            sub = gt[:, :, a * N:a * N + n, b * N:b * N + n, :][sel]
            assert np.array_equal(sub, m.gid[eab[sel]])
    # column-node ownership: count tiles per column
    col = np.where(gt[:, 0, :, :, 0] >= 0, m.col_of[np.maximum(gt[:, 0, :, :, 0], 0)], -1)
    owners = np.zeros(m.ncol, dtype=np.int64)
    for t in range(p.ntiles):
        c = np.unique(col[t][col[t] >= 0])
        owners[c] += 1
    assert np.all(owners >= 1)
    # slots: partial rows dense, unique, grouped by column in tile order
    rows = p.code[p.code >= 0]
    assert len(rows) == p.npart and np.array_equal(np.sort(rows), np.arange(p.npart))
    assert np.array_equal(p.slot_nc, owners[p.slot_col])
    if p.nslot:
        assert np.array_equal(p.slot_row0[1:], np.cumsum(p.slot_nc)[:-1]) and p.slot_row0[0] == 0
    for t in range(p.ntiles):
        for u, v in zip(*np.nonzero(p.code[t] >= 0)):
            s = np.searchsorted(p.slot_col, col[t, u, v])
            assert p.slot_col[s] == col[t, u, v]
            assert p.slot_row0[s] <= p.code[t, u, v] < p.slot_row0[s] + p.slot_nc[s]
    # columns owned by one tile (and not interface) never get a slot
    single = np.nonzero(owners == 1)[0]
    ext = p.slot_col[p.slot_ext >= 0]
    assert set(p.slot_col.tolist()) & set(single.tolist()) == set(ext.tolist()) & set(single.tolist())
    return col


@pytest.mark.parametrize("nx,ny,nv,N,TX,TY", [(4, 4, 2, 4, 2, 2), (5, 3, 3, 4, 2, 2), (3, 2, 2, 2, 2, 2),
                                              (3, 3, 2, 3, 1, 1), (1, 5, 1, 4, 2, 2)])
def test_box_tile_plan(nx, ny, nv, N, TX, TY):
    m = hm.build_box_lattice(nx, ny, nv, N, (100.0 * nx, 120.0 * ny, 50.0 * nv))
    p = build_tile_plan(m, TX, TY)
    assert p is not None and p.next_tiles == 0
    assert p.ntiles == -(-nx // TX) * -(-ny // TY)
    _check_plan(m, p)


def test_sphere_tile_plan():
    m = hm.build_cubed_sphere(hm.MeshConfig("sphere", panels_per_edge=3, n_elem_vertical=2, degree=3,
                                             radius=6.371e6, z_top=3.0e4))
    p = build_tile_plan(m, 2, 2)
    assert p is not None and p.ntiles == 6 * 4
    _check_plan(m, p)
    # cube edges and corners: columns shared by up to 3 tiles across panels
    assert p.slot_nc.max() >= 3


@pytest.mark.parametrize("rank", [0, 1, 2])
def test_slab_interface_tiles_first(rank):
    world, nxp, ny, nv, N = 3, 5, 4, 2, 4
    L = parallel.SlabLayout(rank, world, nxp, ny, nv, N, elem_size=(100.0, 120.0, 50.0))
    m = L.build_mesh()
    ext = L.ext_cols(m)
    p = build_tile_plan(m, 2, 2, ext)
    assert p is not None
    col = _check_plan(m, p)
    touches = np.array([np.isin(col[t][col[t] >= 0], list(ext)).any() for t in range(p.ntiles)])
    assert p.next_tiles == touches.sum()
    assert np.all(touches[:p.next_tiles]) and not np.any(touches[p.next_tiles:])
    # every interface column is a slot carrying its (side * face + jf) code
    slot_of = dict(zip(p.slot_col.tolist(), p.slot_ext.tolist()))
    assert all(slot_of[c] == code for c, code in ext.items())
    assert np.array_equal(np.sort(p.ext_slots), np.nonzero(p.slot_ext >= 0)[0])
    assert len(p.ext_slots) == len(ext) == L.face * ((rank > 0) + (rank < world - 1))


def test_plan_rejects_unstructured():
    m = hm.build_box_lattice(2, 2, 2, 3, (200.0, 240.0, 100.0))
    m.hgrid = None
    assert build_tile_plan(m, 2, 2) is None


def _chunk_model_ok(p, ct, ld=5):
    """Every node (u, v, k >= 1) of every layer >= 1 sits where the chunk table's runs put its gid."""
    UV, N = p.U * p.V, p.N
    gt = p.gt[:, :, :UV * p.n].reshape(p.ntiles, p.nlay, UV, p.n)
    for t in range(p.ntiles):
        colrow, nr = ct[t, :UV], ct[t, UV]
        runs = ct[t, UV + 1:UV + 1 + 4 * nr].reshape(-1, 4)
        # runs: disjoint row ranges with a spare row between them, start row parity = gid parity
        rr = sorted((int(p0), int(p0 + nrow)) for _, _, nrow, p0 in runs)
        assert all(b[0] > a[1] for a, b in zip(rr, rr[1:]))
        assert all((g1 - p0) % 2 == 0 and st % 2 == 0 for g1, st, _, p0 in runs)
        for l in range(1, p.nlay):
            row = np.full(rr[-1][1] + 1, -1, dtype=np.int64)
            for g1, st, nrow, p0 in runs:
                row[p0:p0 + nrow] = g1 + st * (l - 1) + np.arange(nrow)
            got = row[colrow[:, None] + np.arange(N)[None, :]]
            assert np.array_equal(got, gt[t, l, :, 1:])


@pytest.mark.parametrize("perturb", [True, False])
def test_chunk_table_lattice_box(perturb):
    """Lattice-numbered boxes (configs 1, 2, 5): the bulk-copy runs of pass 1's input reproduce the
    tile node gids of every layer >= 1 (lap_plane.cu IO 3)."""
    from paper_2311_11425_b200.tiles import build_chunk_table

    m = hm.build_box_lattice(6, 4, 3, 4, (6000.0, 4000.0, 1500.0), perturb=perturb)
    p = build_tile_plan(m, 2, 2)
    ct = build_chunk_table(p, 360)
    assert ct is not None
    _chunk_model_ok(p, ct)
    assert ct[:, p.U * p.V].max() <= 32


def test_chunk_table_rejects_what_it_cannot_model():
    """Single-layer meshes and capacities below the runs: no table (the gather path runs)."""
    from paper_2311_11425_b200.tiles import build_chunk_table

    m1 = hm.build_box_lattice(4, 4, 1, 4, (4000.0, 4000.0, 500.0))
    assert build_chunk_table(build_tile_plan(m1, 2, 2), 360) is None
    m = hm.build_box_lattice(4, 4, 2, 4, (4000.0, 4000.0, 1000.0))
    assert build_chunk_table(build_tile_plan(m, 2, 2), 200) is None


def test_chunk_table_sphere_if_modelled():
    """The cubed sphere's numbering: either modelled exactly or rejected (never a wrong table)."""
    from paper_2311_11425_b200.tiles import build_chunk_table

    m = hm.build_cubed_sphere(hm.MeshConfig("sphere", panels_per_edge=4, n_elem_vertical=3, degree=4,
                                            radius=6.371e6, z_top=1e4))
    p = build_tile_plan(m, 2, 2)
    ct = build_chunk_table(p, 360)
    if ct is not None:
        _chunk_model_ok(p, ct)
