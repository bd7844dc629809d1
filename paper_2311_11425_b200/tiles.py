"""Tile plan for the fused sweep kernels (host setup, numpy index bookkeeping).

A tile is a TX x TY patch of element columns inside one panel of the
(panel, ia, ib) column grid; one CTA sweeps it bottom to top, one layer of
TX*TY elements per step.  Inside the tile the element nodes are addressed on
the structured tile grid (u, v, k) = (px*N + i, py*N + j, k); shared faces
between the tile's elements are summed on chip and the top face of a layer is
carried in registers into the next layer, so only the column-nodes on the
tile perimeter that another tile also owns need an off-chip combination
("partial rows", summed in fixed order by the fix-up kernel).

Every structural assumption is verified against the mesh's own gid: if an
element's gid does not match the tile grid (non-extruded or oddly oriented
mesh) the plan is rejected and the operators use the element-parallel path.
"""

from __future__ import annotations

import os

import numpy as np

__all__ = ["TilePlan", "build_tile_plan", "tile_shape"]


def tile_shape(N, F=4):
    """(TX, TY) of the compiled sweep kernels: 2x2 columns for the plane-owner kernel
    (lap_plane.cu, N <= 4) and the line kernel (lap_tile.cu, N = 5, 6); single columns at
    N = 7 (the 6-component metric of an N = 7 element layer is 24.6 KB), where the default is
    the split-plane kernel (H = 4); ``HV_N7_KERNEL=plane2x2`` selects 2x2 tiles for it
    (measured slower)."""
    if N == 7 and os.environ.get("HV_N7_KERNEL", "") != "plane2x2":
        return (1, 1)
    return (2, 2)


class TilePlan:
    """Host arrays of one tile plan (see module docstring)."""

    def __init__(self, **kw):
        self.__dict__.update(kw)


def build_tile_plan(mesh, TX, TY, ext_cols=None, _order=None):
    """Tile plan of ``mesh``; ``ext_cols`` maps column id -> interface code
    (side * face + jf) for column nodes also owned by a neighbouring rank
    (parallel.py): they become slots even when a single local tile owns them,
    and the tiles holding them come first (``next_tiles`` of them) so that one
    pass can sweep them, ship the interface sums and sweep the interior tiles
    while the exchange is in flight."""
    N = mesh.degree
    n = N + 1
    if mesh.hgrid is None:
        return None
    npan, nx, ny = mesh.hgrid
    nlay = mesh.cfg.n_elem_vertical
    nhcol = npan * nx * ny
    if mesh.nelem != nhcol * nlay:
        return None
    # (hcol, layer) -> element
    order = np.lexsort((mesh.elem_layer, mesh.elem_hcol))
    if not (np.array_equal(mesh.elem_hcol[order], np.repeat(np.arange(nhcol), nlay))
            and np.array_equal(mesh.elem_layer[order], np.tile(np.arange(nlay), nhcol))):
        return None
    stack = order.reshape(nhcol, nlay)
    # tiles
    tiles = []
    for p in range(npan):
        for a0 in range(0, nx, TX):
            for b0 in range(0, ny, TY):
                tiles.append((p, a0, b0, min(TX, nx - a0), min(TY, ny - b0)))
    tiles = np.array(tiles, dtype=np.int64)
    if _order is not None:
        tiles = tiles[_order]
    nt = len(tiles)
    U, V = TX * N + 1, TY * N + 1
    NE = TX * TY
    # element of (tile, layer, px, py); -1 outside ragged tiles
    px = np.arange(TX)[None, :, None]
    py = np.arange(TY)[None, None, :]
    act = (px < tiles[:, 3][:, None, None]) & (py < tiles[:, 4][:, None, None])
    ia = tiles[:, 1][:, None, None] + px
    ib = tiles[:, 2][:, None, None] + py
    hc = (tiles[:, 0][:, None, None] * nx + np.minimum(ia, nx - 1)) * ny + np.minimum(ib, ny - 1)
    elem = np.where(act[:, None], stack[hc][:, :, :, :].transpose(0, 3, 1, 2), -1)  # (nt, nlay, TX, TY)
    # tile node gids: scatter every active element onto the tile grid and check
    # that elements sharing a tile node agree (the structural hypothesis)
    gid = mesh.gid
    gt = np.full((nt, nlay, U, V, n), -1, dtype=np.int64)
    for a in range(TX):
        for b in range(TY):
            e_ab = elem[:, :, a, b]
            m = e_ab >= 0
            if not np.any(m):
                continue
            ref = gid[np.where(m, e_ab, 0)]                              # (nt, nlay, n, n, n)
            sub = gt[:, :, a * N:a * N + n, b * N:b * N + n, :]
            mm = np.broadcast_to(m[..., None, None, None], sub.shape)
            clash = mm & (sub >= 0) & (sub != ref)
            if np.any(clash):
                return None
            sub[mm] = ref[mm]
    # vertical stacking: top level of layer l == bottom level of layer l+1
    if nlay > 1:
        top, bot = gt[:, :-1, :, :, N], gt[:, 1:, :, :, 0]
        if not np.array_equal(top, bot):
            return None
    # column ids of the tile column-nodes and the sharing between tiles
    col = np.where(gt[:, 0, :, :, 0] >= 0, mesh.col_of[np.maximum(gt[:, 0, :, :, 0], 0)], -1)  # (nt, U, V)
    flat = col.reshape(nt, -1)
    tid = np.repeat(np.arange(nt), flat.shape[1])
    cf = flat.reshape(-1)
    m = cf >= 0
    pairs = np.unique(np.stack([cf[m], tid[m]], axis=1), axis=0)          # (col, tile) sorted by col then tile
    cnt = np.bincount(pairs[:, 0], minlength=mesh.ncol)
    is_ext = np.zeros(mesh.ncol, dtype=bool)
    ext_code = np.full(mesh.ncol, -1, dtype=np.int64)
    if ext_cols:
        kk = np.fromiter(ext_cols.keys(), dtype=np.int64)
        is_ext[kk] = True
        ext_code[kk] = np.fromiter(ext_cols.values(), dtype=np.int64)
    shared_cols = np.nonzero((cnt >= 2) | (is_ext & (cnt >= 1)))[0]
    nslot = len(shared_cols)
    slot_of_col = np.full(mesh.ncol, -1, dtype=np.int64)
    slot_of_col[shared_cols] = np.arange(nslot)
    slot_nc = cnt[shared_cols]
    slot_row0 = np.zeros(nslot, dtype=np.int64)
    if nslot:
        slot_row0[1:] = np.cumsum(slot_nc)[:-1]
    # rank of each (col, tile) pair among the col's tiles
    first = np.searchsorted(pairs[:, 0], pairs[:, 0], side="left")
    rank = np.arange(len(pairs)) - first
    code = np.full((nt, U, V), -1, dtype=np.int64)
    pkey = pairs[:, 0] * nt + pairs[:, 1]
    tq = np.broadcast_to(np.arange(nt)[:, None, None], col.shape)
    mq = col >= 0
    if nslot and np.any(mq):
        k = col[mq] * nt + tq[mq]
        idx = np.searchsorted(pkey, k)
        sl = slot_of_col[col[mq]]
        rows = np.where(sl >= 0, slot_row0[np.maximum(sl, 0)] + rank[idx], -1)
        code[mq] = rows
    npart = int(slot_nc.sum()) if nslot else 0
    nodes = U * V * n
    gts = (nodes + 3) & ~3
    mts = (nodes + 1) & ~1
    gtp = np.full((nt, nlay, gts), -1, dtype=np.int32)
    gtp[:, :, :nodes] = gt.reshape(nt, nlay, nodes)
    slot_ext = ext_code[shared_cols].astype(np.int32)
    ext_slots = np.nonzero(slot_ext >= 0)[0].astype(np.int32)
    ext_tile = np.zeros(nt, dtype=bool)
    if ext_cols:
        ext_tile = (np.where(col >= 0, is_ext[np.maximum(col, 0)], False)).reshape(nt, -1).any(axis=1)
        if _order is None and not np.all(ext_tile[:ext_tile.sum()]):
            # interface tiles first (stable), rebuild with that order
            return build_tile_plan(mesh, TX, TY, ext_cols,
                                   _order=np.concatenate([np.nonzero(ext_tile)[0], np.nonzero(~ext_tile)[0]]))
    return TilePlan(next_tiles=int(ext_tile.sum()), N=N, n=n, TX=TX, TY=TY, U=U, V=V, NE=NE, nlay=nlay, ntiles=nt, tiles=tiles, elem=elem,
                    slot_ext=slot_ext, ext_slots=ext_slots,
                    gt=gtp, gts=gts, mts=mts, nodes=nodes, code=code.astype(np.int32), nslot=nslot,
                    slot_col=shared_cols.astype(np.int32), slot_row0=slot_row0.astype(np.int32),
                    slot_nc=slot_nc.astype(np.int32), npart=npart, n_z=mesh.n_z,
                    tmeta=tiles[:, 3:5].astype(np.int32))
