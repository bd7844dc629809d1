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


def _global_problem(world, nxp, ny, nv, N, esz, cfg, dt, set_name="2C"):
    from paper_2311_11425_b200 import euler, hyperdiff, mesh as hm, metrics, state

    ext = (esz[0] * nxp * world, esz[1] * ny, esz[2] * nv)
    g = hm.build_box_lattice(nxp * world, ny, nv, N, ext)
    gm = metrics.project_metrics_to_columns(metrics.curl_invariant_metrics(g), g)
    gvm = hyperdiff.build_viscous_metric(g, gm, cfg, dt=dt)
    gops = euler.EulerOps(g, gm, state.PhysConstants(omega=0.0), set_name, hyper=(cfg, gvm))
    return g, gops, gvm


@pytest.mark.gpu
@pytest.mark.parametrize("world,nxp,N", [(2, 2, 4), (3, 2, 3), (2, 1, 7)])
def test_slab_euler_rhs_matches_single_mesh(world, nxp, N):
    """S + H_nu across slabs (SURVEY §8(e) "other phases": the 5-field face exchange of the Euler
    RHS DSS) equals the single-mesh rhs_full_hyper; interface rows bitwise equal on both owners."""
    import torch

    from cases import random_state, rel_l2
    from paper_2311_11425_b200 import hyperdiff, state

    ny, nv = 2, 2
    esz = (100.0, 120.0, 50.0)
    cfg = hyperdiff.HyperDiffConfig(alpha=2, c=(0.05, 0.05, 0.0))
    g, gops, gvm = _global_problem(world, nxp, ny, nv, N, esz, cfg, 0.5)
    q = random_state(g.nglobal, "2C")
    ref = gops.rhs_full_hyper(state.StateField("2C", q))
    layouts = [parallel.SlabLayout(r, world, nxp, ny, nv, N, elem_size=esz) for r in range(world)]
    ops = parallel.setup_loopback(layouts, cfg, 0.5)
    maps = [L.local_to_global(op.mesh, g) for L, op in zip(layouts, ops)]
    qs = [torch.from_numpy(q[l2g]).cuda() for l2g in maps]
    outs = [torch.empty_like(x) for x in qs]
    parallel.run_loopback_euler(ops, qs, outs)
    got = np.zeros_like(ref)
    vals = {}
    for o, l2g in zip(outs, maps):
        oo = o.cpu().numpy()
        got[l2g] = oo
        for li, gi in enumerate(l2g):
            if gi in vals:
                assert np.array_equal(vals[gi], oo[li])
            vals[gi] = oo[li]
    assert rel_l2(got, ref) <= 1e-13, rel_l2(got, ref)


def _slab_proc(rank, world, port, nxp, N, q_global_path, outq):
    """One rank of the 2-process test: gloo process group, halos staged through host memory
    (HostStagedTransport), both ranks on cuda:0 (no kernel waits on the other process)."""
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2311_11425_b200 import hyperdiff

        torch.cuda.set_device(0)
        ny, nv, esz = 2, 2, (100.0, 120.0, 50.0)
        cfg = hyperdiff.HyperDiffConfig(alpha=2, c=(0.05, 0.05, 0.0))
        L = parallel.SlabLayout(rank, world, nxp, ny, nv, N, elem_size=esz)
        tr = parallel.HostStagedTransport(rank, world)
        op = parallel.setup_distributed(L, cfg, 0.5, tr)
        z = np.load(q_global_path)
        l2g = z[f"l2g{rank}"]
        q = torch.from_numpy(np.ascontiguousarray(z["q"][l2g])).cuda()
        h = torch.empty_like(q)
        op.apply(q, h, tr)
        s = torch.empty_like(q)
        op.rhs_full_hyper(q, s, tr)
        torch.cuda.synchronize()
        outq.put((rank, h.cpu().numpy(), s.cpu().numpy(), op.ops.mass.d_M.cpu().numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("N", [4, 7])
def test_two_process_slabs_host_staged(tmp_path, N):
    """Two processes (torch.distributed gloo, world 2), each building its slab with
    setup_distributed (cross-rank mass / projection) and applying H_nu and S + H_nu through the
    DistTransport API, against the single-mesh results and the CPU oracle."""
    import torch.multiprocessing as mp

    from cases import random_state, rel_l2
    from oracle import hevi_oracle as O
    from paper_2311_11425_b200 import hyperdiff, state

    world, nxp, ny, nv = 2, 2, 2, 2
    esz = (100.0, 120.0, 50.0)
    cfg = hyperdiff.HyperDiffConfig(alpha=2, c=(0.05, 0.05, 0.0))
    g, gops, gvm = _global_problem(world, nxp, ny, nv, N, esz, cfg, 0.5)
    q = random_state(g.nglobal, "2C")
    maps = [parallel.SlabLayout(r, world, nxp, ny, nv, N, elem_size=esz).local_to_global(
        parallel.SlabLayout(r, world, nxp, ny, nv, N, elem_size=esz).build_mesh(), g) for r in range(world)]
    path = tmp_path / "q.npz"
    np.savez(path, q=q, **{f"l2g{r}": m for r, m in enumerate(maps)})
    ctx = mp.get_context("spawn")
    outq = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_slab_proc, args=(r, world, port, nxp, N, str(path), outq)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((outq.get(timeout=300) for _ in procs), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    H = np.zeros((g.nglobal, 5))
    S = np.zeros((g.nglobal, 5))
    M = np.zeros(g.nglobal)
    for (r, h, s, m), l2g in zip(res, maps):
        for arr, loc in ((H, h), (S, s)):
            arr[l2g] = loc
        M[l2g] = m
    # the two ranks agree bitwise on the shared face nodes
    shared = np.intersect1d(maps[0], maps[1])
    pos0 = {v: i for i, v in enumerate(maps[0])}
    pos1 = {v: i for i, v in enumerate(maps[1])}
    i0 = np.array([pos0[v] for v in shared])
    i1 = np.array([pos1[v] for v in shared])
    assert np.array_equal(res[0][1][i0], res[1][1][i1]) and np.array_equal(res[0][2][i0], res[1][2][i1])
    st = state.StateField("2C", q)
    assert rel_l2(M, gops.mass.M) <= 1e-15
    assert rel_l2(H, hyperdiff.hyperdiffusion_apply(st, cfg, gvm, gops)) <= 1e-13
    assert rel_l2(S, gops.rhs_full_hyper(st)) <= 1e-13
    # and the CPU oracle on the global mesh
    coords, layer, hcol = g.coords, g.elem_layer, g.elem_hcol
    om = O.OracleMesh.from_coords("box", N, coords, layer, hcol,
                                  O.dedupe_tol("box", max(g.cfg.panels_per_edge, 1), extents=g.cfg.box_extents))
    _, J, grad = O.curl_metrics(om)
    Jg, gz = O.project_columns(om, J, grad)
    _, Minv = O.lumped_mass(om, J)
    Gnu, _, _ = O.viscous_metric(om, grad, 2, c=cfg.c, dt=0.5)
    Ho = O.hyperdiffusion(om, Gnu, O.gather(om.gid, Jg), Minv, q, 2)
    assert rel_l2(H, Ho) <= 1e-12
    So = O.OracleEuler(om, J, grad, Jg, gz, O.Consts(omega=0.0), "2C").rhs_full(q) + Ho
    assert rel_l2(S, So) <= 1e-12
