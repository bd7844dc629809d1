"""Multi-GPU slab decomposition.

CPU (gloo, world_size 2): slab layout, interface matching across ranks through
the same DistTransport the GPU path uses, local->global maps, rank-order sums.
GPU (one device, several ranks in one process): the whole device pipeline
(setup exchange, split passes, interface slots) against the single-mesh result.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

from paper_2311_11425_b200 import parallel


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        L = parallel.SlabLayout(rank, world, nx_per=3, ny=2, nv=2, N=3, elem_size=(100.0, 120.0, 50.0))
        m = L.build_mesh()
        faces = L.face_columns(m)
        face = L.face
        # every rank sends the coordinates of its face column nodes (all levels) to its neighbours
        send = torch.zeros((2, face, m.n_z, 5), dtype=torch.float64)
        recv = torch.zeros_like(send)
        for s, cols in faces.items():
            xyz = m.xg[m.col_gid[cols]]                     # (face, n_z, 3)
            send[s, :, :, :3] = torch.from_numpy(xyz)
            send[s, :, :, 3] = rank
        parallel.DistTransport(rank, world).exchange(send, recv)
        ok = True
        for s, cols in faces.items():
            xyz = m.xg[m.col_gid[cols]]
            ok &= bool(np.array_equal(recv[s, :, :, :3].numpy(), xyz))      # bitwise identical faces
            ok &= bool(np.all(recv[s, :, :, 3].numpy() == (rank - 1 if s == 0 else rank + 1)))
        # rank-order combination is the same expression on both sides
        a = torch.tensor([0.1 * (rank + 1)], dtype=torch.float64)
        b = torch.tensor([0.7 / (rank + 3)], dtype=torch.float64)
        q.put((rank, ok, sorted(faces), float(parallel.combine_interface(a, b, 0)), m.nglobal))
    finally:
        dist.destroy_process_group()


def test_slab_interfaces_gloo_world2():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(r[1] for r in res)
    assert res[0][2] == [1] and res[1][2] == [0]


def test_local_to_global_map_and_counts():
    from paper_2311_11425_b200 import mesh as hm

    world, nxp, ny, nv, N = 3, 2, 3, 2, 2
    g = hm.build_box_lattice(nxp * world, ny, nv, N, (100.0 * nxp * world, 120.0 * ny, 50.0 * nv))
    seen = np.zeros(g.nglobal, dtype=int)
    for r in range(world):
        L = parallel.SlabLayout(r, world, nxp, ny, nv, N, elem_size=(100.0, 120.0, 50.0))
        m = L.build_mesh()
        l2g = L.local_to_global(m, g)
        assert np.all(l2g >= 0) and len(np.unique(l2g)) == m.nglobal
        assert np.array_equal(m.xg, g.xg[l2g]) or np.allclose(m.xg, g.xg[l2g], rtol=0, atol=1e-9)
        seen[l2g] += 1
        faces = L.face_columns(m)
        assert sorted(faces) == [s for s, ok in ((0, r > 0), (1, r < world - 1)) if ok]
    # interface column nodes are owned by exactly two slabs, all others by one
    n_face = (ny * N + 1) * (nv * N + 1)
    assert np.sum(seen == 2) == (world - 1) * n_face and np.all(seen >= 1)


def test_lattice_keyed_state_agrees_on_slab_faces():
    """The multi-GPU bench state (synthetic.fourier_state with noise keyed on the global lattice node,
    SlabLayout.lattice_keys) is one global field: every rank holds, on every node, exactly the value
    the single global mesh holds there, so the slab-face nodes two ranks share agree bitwise."""
    from paper_2311_11425_b200 import mesh as hm, synthetic

    world, nxp, ny, nv, N = 3, 2, 3, 2, 3
    esz = (100.0, 120.0, 50.0)
    ext = (esz[0] * nxp * world, esz[1] * ny, esz[2] * nv)
    g = hm.build_box_lattice(nxp * world, ny, nv, N, ext)
    G = parallel.SlabLayout(0, 1, nxp * world, ny, nv, N, elem_size=esz)
    gkeys = G.lattice_keys(g)
    assert len(np.unique(gkeys)) == g.nglobal
    qg = synthetic.fourier_state(g.xg, ext, noise_keys=gkeys)
    for r in range(world):
        L = parallel.SlabLayout(r, world, nxp, ny, nv, N, elem_size=esz)
        m = L.build_mesh()
        l2g = L.local_to_global(m, g)
        assert np.array_equal(L.lattice_keys(m), gkeys[l2g])
        q = synthetic.fourier_state(m.xg, L.extents, noise_keys=L.lattice_keys(m))
        assert np.array_equal(q, qg[l2g])


@pytest.mark.gpu
@pytest.mark.parametrize("world,nxp", [(2, 2), (3, 2), (2, 6)])
def test_slab_pipeline_matches_single_mesh(world, nxp):
    import torch

    from cases import rel_l2
    from paper_2311_11425_b200 import euler, hyperdiff, mesh as hm, metrics, state, synthetic

    ny, nv, N = 3, 2, 4
    esz = (100.0, 120.0, 50.0)
    ext = (esz[0] * nxp * world, esz[1] * ny, esz[2] * nv)
    cfg = hyperdiff.HyperDiffConfig(alpha=2, c=(0.05, 0.05, 0.0))
    g = hm.build_box_lattice(nxp * world, ny, nv, N, ext)
    gm = metrics.project_metrics_to_columns(metrics.curl_invariant_metrics(g), g)
    gvm = hyperdiff.build_viscous_metric(g, gm, cfg, dt=0.5)
    gops = euler.EulerOps(g, gm, state.PhysConstants(omega=0.0), "2C", hyper=(cfg, gvm))
    q = synthetic.fourier_state(g.xg, ext)
    ref = hyperdiff.hyperdiffusion_apply(state.StateField("2C", q), cfg, gvm, gops)
    layouts = [parallel.SlabLayout(r, world, nxp, ny, nv, N, elem_size=esz) for r in range(world)]
    ops = parallel.setup_loopback(layouts, cfg, 0.5)
    maps = [L.local_to_global(op.mesh, g) for L, op in zip(layouts, ops)]
    for op in ops:   # interface tiles first; with nxp = 6 the interior launch is not empty
        assert 0 < op.next_tiles <= op.plan.ntiles
        if nxp == 6:
            assert op.next_tiles < op.plan.ntiles
    # slab mass / projected metrics equal the single-mesh ones (rank-order sums)
    for op, l2g in zip(ops, maps):
        assert rel_l2(op.ops.mass.d_M.cpu().numpy(), gops.mass.M[l2g]) <= 1e-15
        assert rel_l2(op.mets.Jg, gm.Jg[l2g]) <= 1e-15
    qs = [torch.from_numpy(q[l2g]).cuda() for l2g in maps]
    outs = [torch.empty_like(x) for x in qs]
    parallel.run_loopback(ops, qs, outs)
    got = np.zeros_like(ref)
    for o, l2g in zip(outs, maps):
        got[l2g] = o.cpu().numpy()
    assert rel_l2(got, ref) <= 1e-13
    # interface nodes: both owning slabs hold bitwise identical values
    vals = {}
    for o, l2g in zip(outs, maps):
        oo = o.cpu().numpy()
        for li, gi in enumerate(l2g):
            if gi in vals:
                assert np.array_equal(vals[gi], oo[li])
            vals[gi] = oo[li]


@pytest.mark.gpu
def test_slab_apply_stream_overlap_matches_sequential():
    """SlabHyperDiffusion.apply (interface tiles on a side stream, exchange enqueued behind them,
    interior tiles concurrently) equals the sequential pass with the same (here: empty) neighbour
    sums, bit for bit."""
    import torch

    from paper_2311_11425_b200 import hyperdiff, synthetic

    class NoNeighbour:
        calls = 0

        def start(self, send, recv):
            NoNeighbour.calls += 1
            return []

        def wait(self, works):
            pass

        def exchange(self, send, recv):
            pass

    layout = parallel.SlabLayout(0, 2, 6, 3, 2, 4, elem_size=(100.0, 120.0, 50.0))
    cfg = hyperdiff.HyperDiffConfig(alpha=2, c=(0.05, 0.05, 0.0))
    op = parallel.setup_distributed(layout, cfg, 0.5, NoNeighbour())
    assert 0 < op.next_tiles < op.plan.ntiles
    q = torch.from_numpy(synthetic.fourier_state(op.mesh.xg, layout.extents)).cuda()
    out1 = torch.empty_like(q)
    op.apply(q, out1, NoNeighbour())
    out2 = torch.empty_like(q)
    for k in range(cfg.alpha):
        op.pass_local(k, q, out2, "all")
        op.pass_finish()
    torch.cuda.synchronize()
    assert torch.equal(out1, out2)
    assert NoNeighbour.calls == cfg.alpha
