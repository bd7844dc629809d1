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


def build_chunk_table(tp, rows_cap, row_ld=5):
    """Bulk-copy description of a tile plan's q input (lap_plane.cu IO 3), or None.

    On lattice-numbered meshes (first-appearance order over elements, local nodes (i, j, k), k
    fastest: mesh.py:86-107) the new nodes of an element are one contiguous gid range and a tile
    column's levels k = 1..N of a layer are consecutive gids.  For every tile this finds the runs
    of consecutive gids that hold its levels 1..N (the same runs in every layer >= 1, each start
    advancing by a fixed stride per layer), places them in the kernel's row buffer (AoS rows of
    ``row_ld`` doubles; a start row with the parity of its gid so that both ends of a bulk copy are
    16-byte aligned, one spare row between runs, the element chunks 68 rows apart so that the
    lanes of the four elements hit different bank groups), and returns per tile
    ``[colrow (U*V) | nruns | 32 x (gid at layer 1, stride, rows, dst row)]`` as int32.
    Verified against ``tp.gt`` for every layer; None if any tile does not fit the model.
    """
    U, V, n, N, nlay = tp.U, tp.V, tp.n, tp.N, tp.nlay
    if nlay < 2:
        return None
    UV = U * V
    gt = tp.gt[:, :, :UV * n].reshape(tp.ntiles, nlay, UV, n).astype(np.int64)
    if np.any(gt < 0):
        return None
    lev = gt[:, :, :, 1:]                                       # (t, l, uv, N) levels 1..N
    # levels of a column consecutive in every layer
    if not np.all(np.diff(lev, axis=3) == 1):
        return None
    width = UV + 1 + 4 * 32
    out = np.zeros((tp.ntiles, width), dtype=np.int32)
    col0 = lev[:, :, :, 0]                                      # (t, l, uv) gid of level 1
    for t in range(tp.ntiles):
        c1 = col0[t, 1]
        order = np.argsort(c1, kind="stable")
        s = c1[order]
        # columns whose level-1 gids are N apart continue the same run
        brk = np.nonzero(np.diff(s) != N)[0] + 1
        starts = np.concatenate([[0], brk])
        ends = np.concatenate([brk, [len(s)]])
        if len(starts) > 32:
            return None
        # every layer: a run's columns keep their offsets (one stride per run)
        runs = []
        for a, b in zip(starts, ends):
            cols = order[a:b]
            ct = col0[t]                                          # (nlay, UV)
            st = ct[1:][:, cols] - ct[1][cols][None, :]           # (nlay-1, ncols)
            if not np.all(st == st[:, :1]):
                return None
            d = st[:, 0]
            stride = int(d[1] - d[0]) if len(d) > 1 else 0
            if not np.array_equal(d, stride * np.arange(nlay - 1)):
                return None
            runs.append((int(c1[cols[0]]), stride, (b - a) * N, cols))
        # placement: big runs (element chunks) first, 68 rows apart; then the faces.  When that does not
        # fit the row buffer (e.g. cubed-sphere tiles at panel edges), packed with one spare row only.
        runs.sort(key=lambda r: -r[2])
        if any(st % 2 for _, st, _, _ in runs):
            return None                                          # parity must not change between layers
        for aligned in (True, False):
            cur, big = 0, 0
            colrow = np.zeros(UV, dtype=np.int64)
            meta = []
            for g1, stride, nrows, cols in runs:
                p = cur + (1 if cur else 0)
                if aligned and nrows >= 4 * N * N:
                    p = max(p, 68 * big)
                    big += 1
                if (p - g1) % 2:
                    p += 1
                colrow[cols] = p + N * np.arange(len(cols))
                meta.append((g1, stride, nrows, p))
                cur = p + nrows
            if cur + 1 <= rows_cap:
                break
        else:
            return None
        out[t, :UV] = colrow
        out[t, UV] = len(meta)
        for r, m in enumerate(meta):
            out[t, UV + 1 + 4 * r:UV + 5 + 4 * r] = m
    return out
