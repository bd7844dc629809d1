"""Multi-GPU slab decomposition of the hyper-diffusion operator.

The paper scales by horizontal domain decomposition keeping vertical columns
whole; the reference code itself is serial.  Here one process
drives one GPU and owns an x-slab of ``nx_per`` element rows of the global
(nx_per * world) x ny x nv box (config 5), built as a standalone local mesh.
The only inter-rank coupling of H_nu is the direct-stiffness summation of the
column nodes on the two slab faces:

* setup: the raw flat-order sums behind M, J_g and grad zeta
  (hv_mass_proj_sums) are exchanged on the face nodes and added in global rank
  order before the divisions (hv_mass_proj_finalize);
* every Laplacian pass: hv_lap_local (tile sweep; the face column nodes are
  slots, their local sums packed into a send buffer), one neighbour exchange
  of (2, face, n_z, 5) doubles, hv_lap_finish (fixed-order sums, lower rank
  first, so both ranks hold bitwise identical interface values).

Transports: ``DistTransport`` (torch.distributed point-to-point: NCCL for CUDA
tensors over NVLink, gloo for CPU tensors in the CPU tests) and
``LoopbackTransport`` (several ranks inside one process on one GPU, used to
test the whole device pipeline without inter-process waits).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .basis import lobatto
from .device import torch_mod

__all__ = ["SlabLayout", "DistTransport", "HostStagedTransport", "LoopbackTransport", "SlabHyperDiffusion",
           "run_loopback", "run_loopback_euler", "halo_views"]

ELEM_SIZE_C5 = (3125.0, 3125.0, 1250.0)


class SlabLayout:
    """Rank ``rank`` of ``world`` owns element rows ia in [rank*nx_per, (rank+1)*nx_per)."""

    def __init__(self, rank, world, nx_per, ny, nv, N, elem_size=ELEM_SIZE_C5, perturb=True):
        if not (0 <= rank < world):
            raise ValueError("rank out of range")
        self.rank, self.world = rank, world
        self.nx_per, self.ny, self.nv, self.N = nx_per, ny, nv, N
        self.nx_g = nx_per * world
        self.extents = (elem_size[0] * self.nx_g, elem_size[1] * ny, elem_size[2] * nv)
        self.perturb = perturb
        self.face = ny * N + 1

    def build_mesh(self):
        from .mesh import Mesh, MeshConfig
        from .synthetic import perturbed_box_coords

        ia0 = self.rank * self.nx_per
        coords, layer, hcol = perturbed_box_coords(self.nx_g, self.ny, self.nv, self.N, self.extents,
                                                   perturb=self.perturb, ia_range=(ia0, ia0 + self.nx_per))
        cfg = MeshConfig("box", panels_per_edge=max(self.nx_g, self.ny), n_elem_vertical=self.nv, degree=self.N,
                         box_extents=tuple(float(x) for x in self.extents))
        b = lobatto(self.N)
        return Mesh(cfg, coords, (b, b, b), layer, hcol, hgrid=(1, self.nx_per, self.ny))

    def face_columns(self, mesh):
        """{side: column ids (face,) ordered along the face}; side 0 = lower rank, 1 = upper rank."""
        N, ny, nv = self.N, self.ny, self.nv
        out = {}
        for side, ia, i in ((0, 0, 0), (1, self.nx_per - 1, N)):
            if (side == 0 and self.rank == 0) or (side == 1 and self.rank == self.world - 1):
                continue
            cols = np.empty(self.face, dtype=np.int64)
            for ib in range(ny):
                e = (ia * ny + ib) * nv          # layer 0 element of column (ia, ib)
                for j in range(N + 1):
                    cols[ib * N + j] = mesh.col_of[mesh.gid[e, i, j, 0]]
            out[side] = cols
        return out

    def ext_cols(self, mesh):
        return {int(c): side * self.face + jf for side, cols in self.face_columns(mesh).items()
                for jf, c in enumerate(cols)}

    def lattice_keys(self, mesh):
        """Global vertex-lattice index of every local node, (I * (ny N + 1) + J) * (nv N + 1) + K with
        I = ia_global N + i, J = ib N + j, K = l N + k: the same key on every rank that holds the node
        (state generation keyed on it, synthetic.fourier_state(noise_keys=...))."""
        N, ny, nv = self.N, self.ny, self.nv
        n = N + 1
        keys = np.empty(mesh.nglobal, dtype=np.int64)
        ii, jj, kk = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
        ii, jj, kk = ii.reshape(-1), jj.reshape(-1), kk.reshape(-1)
        nyl, nzl = ny * N + 1, nv * N + 1
        step = 1 << 16
        for e0 in range(0, mesh.nelem, step):
            e = np.arange(e0, min(mesh.nelem, e0 + step))
            ia = e // (ny * nv) + self.rank * self.nx_per
            ib = (e // nv) % ny
            l = e % nv
            I = ia[:, None] * N + ii[None, :]
            J = ib[:, None] * N + jj[None, :]
            K = l[:, None] * N + kk[None, :]
            keys[mesh.gid[e0:e0 + len(e)].reshape(len(e), -1)] = (I * nyl + J) * nzl + K
        return keys

    def local_to_global(self, mesh, global_mesh):
        """Global gid of every local node (tests / gathering results)."""
        N3 = mesh.gid.shape[1:]
        l2g = np.full(mesh.nglobal, -1, dtype=np.int64)
        ny, nv = self.ny, self.nv
        e_l = np.arange(mesh.nelem)
        ia_l = e_l // (ny * nv)
        rest = e_l % (ny * nv)
        e_g = (ia_l + self.rank * self.nx_per) * ny * nv + rest
        l2g[mesh.gid.reshape(mesh.nelem, -1)] = global_mesh.gid[e_g].reshape(mesh.nelem, -1)
        return l2g


class DistTransport:
    """Neighbour exchange with torch.distributed point-to-point ops (NCCL or gloo).

    ``start`` enqueues the sends / receives (with NCCL they run on the communicator's stream,
    ordered after the work already queued on the current stream) and returns the handles;
    ``wait`` makes the current stream (NCCL) or the host (gloo) wait for them."""

    def __init__(self, rank, world):
        self.rank, self.world = rank, world

    def start(self, send, recv):
        import torch.distributed as dist

        ops = []
        if self.rank > 0:
            ops += [dist.P2POp(dist.isend, send[0], self.rank - 1), dist.P2POp(dist.irecv, recv[0], self.rank - 1)]
        if self.rank < self.world - 1:
            ops += [dist.P2POp(dist.isend, send[1], self.rank + 1), dist.P2POp(dist.irecv, recv[1], self.rank + 1)]
        return dist.batch_isend_irecv(ops) if ops else []

    @staticmethod
    def wait(works):
        for r in works:
            r.wait()

    def exchange(self, send, recv):
        self.wait(self.start(send, recv))


class HostStagedTransport(DistTransport):
    """DistTransport over a CPU backend (gloo) for CUDA halo buffers: the send buffer is copied to
    the host after the work queued on the current stream, exchanged, and copied back onto the
    current stream in ``wait``.  Multi-process tests on one GPU (no kernel ever waits on another
    process's kernel) and hosts without NCCL peers."""

    def start(self, send, recv):
        import torch.distributed as dist

        hs = send.detach().to("cpu")                   # synchronises with the producing stream
        hr = torch_mod().empty_like(hs)
        ops = []
        if self.rank > 0:
            ops += [dist.P2POp(dist.isend, hs[0], self.rank - 1), dist.P2POp(dist.irecv, hr[0], self.rank - 1)]
        if self.rank < self.world - 1:
            ops += [dist.P2POp(dist.isend, hs[1], self.rank + 1), dist.P2POp(dist.irecv, hr[1], self.rank + 1)]
        return (dist.batch_isend_irecv(ops) if ops else [], hs, hr, recv)

    @staticmethod
    def wait(works):
        reqs, hs, hr, recv = works
        for r in reqs:
            r.wait()
        recv.copy_(hr.to(recv.device), non_blocking=False)


def halo_views(halo, F):
    """(send, recv) as (2, face * n_z * F) views of the plan's halo buffers: the pass packs F-wide
    rows (slot_pack / slot_fixup), so only F of the 5 allocated doubles per row travel."""
    send, recv = halo
    per = send.shape[1] * send.shape[2] * F
    return send.view(-1)[:2 * per].view(2, per), recv.view(-1)[:2 * per].view(2, per)


class LoopbackTransport:
    """All ranks in one process: recv[1] of rank r <- send[0] of rank r+1 and vice versa."""

    @staticmethod
    def exchange_all(bufs):
        for r in range(len(bufs) - 1):
            s_lo, r_lo = bufs[r + 1]
            s_hi, r_hi = bufs[r]
            r_hi[1].copy_(s_lo[0])
            r_lo[0].copy_(s_hi[1])


def combine_interface(mine, other, side):
    """Interface sum in global rank order (side 0: the neighbour is the lower rank)."""
    return (other + mine) if side == 0 else (mine + other)


class SlabMass:
    """GlobalMass-like holder of the cross-rank mass (assembly.py:54-64)."""

    def __init__(self, d_M, d_Minv):
        self.d_M, self.d_Minv = d_M, d_Minv

    @property
    def M(self):
        return self.d_M.cpu().numpy()

    @property
    def Minv(self):
        return self.d_Minv.cpu().numpy()


class SlabHyperDiffusion:
    """H_nu on one slab; the setup and each pass are split into local / exchange / finish stages."""

    def __init__(self, layout, cfg, dt, set_name="2C"):
        from . import metrics as hmet

        torch = torch_mod()
        self.layout, self.cfg, self.dt, self.set_name = layout, cfg, dt, set_name
        self.mesh = m = layout.build_mesh()
        self.mets0 = hmet.curl_invariant_metrics(m)
        dev = m.device()
        self.S = torch.empty((m.nglobal, 5), dtype=torch.float64, device="cuda")
        _lib.check(_lib.lib().hv_mass_proj_sums(dev.N, dev.w3.data_ptr(), self.mets0.d_J.data_ptr(),
                                                self.mets0.d_grad.data_ptr(), dev.nelem, dev.off.data_ptr(),
                                                dev.idx.data_ptr(), m.nglobal, self.S.data_ptr(), _lib.stream_handle()))
        self.faces = layout.face_columns(m)
        self.face_gid = {s: torch.from_numpy(m.col_gid[c].reshape(-1)).cuda() for s, c in self.faces.items()}
        self.setup_send = torch.zeros((2, layout.face, m.n_z, 5), dtype=torch.float64, device="cuda")
        self.setup_recv = torch.zeros_like(self.setup_send)
        for s, gi in self.face_gid.items():
            self.setup_send[s].view(-1, 5).copy_(self.S[gi])
        self.ops = None

    # ---- setup (after the exchange of setup_send -> setup_recv)
    def setup_finish(self):
        from . import euler, hyperdiff, metrics as hmet
        from .state import PhysConstants

        torch = torch_mod()
        m = self.mesh
        for s, gi in self.face_gid.items():
            self.S[gi] = combine_interface(self.S[gi], self.setup_recv[s].view(-1, 5), s)
        ng = m.nglobal
        M = torch.empty(ng, dtype=torch.float64, device="cuda")
        Minv = torch.empty_like(M)
        Jg = torch.empty_like(M)
        gz = torch.empty((ng, 3), dtype=torch.float64, device="cuda")
        _lib.check(_lib.lib().hv_mass_proj_finalize(ng, self.S.data_ptr(), M.data_ptr(), Minv.data_ptr(),
                                                    Jg.data_ptr(), gz.data_ptr(), _lib.stream_handle()))
        self.mets = hmet.MetricTerms(self.mets0.scheme, m, self.mets0.d_J, self.mets0.d_grad, Jg, gz, projected=True)

        mass = SlabMass(M, Minv)
        self.vm = hyperdiff.build_viscous_metric(m, self.mets, self.cfg, dt=self.dt)
        self.ops = euler.EulerOps(m, self.mets, PhysConstants(omega=0.0), self.set_name, hyper=(self.cfg, self.vm),
                                  mass=mass, ext_cols=self.layout.ext_cols(m))
        self.ops.ext_face = self.layout.face
        self.plan = self.ops.lap_plan(self.vm)
        if self.ops.ext_cols and self.ops.halo is None:
            raise NotImplementedError("slab decomposition needs the tile-sweep kernels (N <= 7, extruded mesh)")
        nv = len(self.cfg.variables)
        self.y = torch.empty((ng, nv), dtype=torch.float64, device="cuda")
        return self

    @property
    def halo(self):
        return self.ops.halo

    # ---- one pass: local stage (tile sweep + pack), exchange, finish stage (slots)
    @property
    def next_tiles(self):
        """Tiles holding slab-interface columns (the tile plan puts them first)."""
        return self.ops._tile_arrays()[0].next_tiles

    def pass_local(self, k, q, out, part="all"):
        """Tile sweep of pass k: ``part`` = "all", "ext" (interface tiles + interface sums
        packed into the send buffer) or "int" (the remaining tiles, no packing)."""
        vars_ = list(self.cfg.variables)
        nv = len(vars_)
        if k == 0:
            qf, ldq = vars_, q.shape[1]
            dst, ldo, of = self.y, nv, list(range(nv))
            scale, zmask = 1.0, 0
        else:
            qf, ldq = list(range(nv)), nv
            dst, ldo, of = out, out.shape[1], vars_
            scale = 1.0 if self.cfg.alpha % 2 == 1 else -1.0
            zmask = ((1 << ldo) - 1) & ~sum(1 << v for v in vars_)
        src = q if k == 0 else self.y
        if self.cfg.alpha == 1:
            dst, ldo, of = out, out.shape[1], vars_
            zmask = ((1 << ldo) - 1) & ~sum(1 << v for v in vars_)
        self._cur = (dst, ldo, of, scale, zmask)
        qa = (C.c_int32 * nv)(*qf)
        oa = (C.c_int32 * nv)(*of)
        nt, ne = self.plan.ntiles, self.next_tiles
        t0, t1, pack = {"all": (0, nt, 1), "ext": (0, ne, 1), "int": (ne, nt, 0)}[part]
        _lib.check(_lib.lib().hv_lap_local_tiles(C.byref(self.plan), src.data_ptr(), ldq, nv, qa, dst.data_ptr(), ldo,
                                                 oa, scale, zmask, 0, t0, t1, pack, _lib.stream_handle()))

    def pass_finish(self):
        dst, ldo, of, scale, zmask = self._cur
        oa = (C.c_int32 * len(of))(*of)
        _lib.check(_lib.lib().hv_lap_finish(C.byref(self.plan), dst.data_ptr(), ldo, len(of), oa, scale, zmask, 0,
                                            _lib.stream_handle()))

    # ---- one process per GPU: the interface tiles on a high-priority side stream, their sums
    # shipped as soon as they are packed, while the interior tiles run on the compute stream
    def apply(self, q, out, transport):
        torch = torch_mod()
        main = torch.cuda.current_stream()
        if getattr(self, "_side", None) is None:
            self._side = torch.cuda.Stream(priority=-1)
        side = self._side
        for k in range(self.cfg.alpha):
            side.wait_stream(main)
            with torch.cuda.stream(side):
                self.pass_local(k, q, out, "ext")
                send, recv = halo_views(self.halo, len(self.cfg.variables))
                works = transport.start(send, recv)
            self.pass_local(k, q, out, "int")
            main.wait_stream(side)
            transport.wait(works)
            self.pass_finish()
        return out


    # ---- Euler RHS across slabs (the same face exchange, 5 fields)
    def _raw_euler(self):
        """EulerOps of this slab whose DSS divides by a unit mass: its rhs_full gives the slab's raw
        DSS sums of the element accumulators (euler.py:101-103 before Minv)."""
        if getattr(self, "_eraw", None) is None:
            from . import euler
            from .state import PhysConstants

            torch = torch_mod()
            ones = torch.ones(self.mesh.nglobal, dtype=torch.float64, device="cuda")
            self._eraw = euler.EulerOps(self.mesh, self.mets, PhysConstants(omega=0.0), self.set_name,
                                        mass=SlabMass(ones, ones))
            self._raw = torch.empty((self.mesh.nglobal, 5), dtype=torch.float64, device="cuda")
            self._esend = torch.zeros((2, self.layout.face * self.mesh.n_z * 5), dtype=torch.float64, device="cuda")
            self._erecv = torch.zeros_like(self._esend)
        return self._eraw

    def euler_local(self, q):
        """Raw slab sums of S(q) and their face rows packed into the send buffer."""
        eo = self._raw_euler()
        eo._rhs(q, 7, 0, out=self._raw)
        for s, gi in self.face_gid.items():
            self._esend[s].view(-1, 5).copy_(self._raw[gi])
        return self._esend, self._erecv

    def euler_finish(self, out, accumulate=True):
        """Complete the face rows in global rank order, then out (+)= Minv * raw."""
        for s, gi in self.face_gid.items():
            self._raw[gi] = combine_interface(self._raw[gi], self._erecv[s].view(-1, 5), s)
        _lib.check(_lib.lib().hv_rows_minv(out.data_ptr(), out.shape[1], self._raw.data_ptr(), 5,
                                           self.ops.mass.d_Minv.data_ptr(), self.mesh.nglobal, 5, int(bool(accumulate)),
                                           _lib.stream_handle()))
        return out

    def rhs_full_hyper(self, q, out, transport):
        """S(q) + H_nu(q) on this slab (config 4's quantity, euler.py:111-118 + hyperdiff.py:97-106), both
        DSS's completed across the slab faces."""
        self.apply(q, out, transport)
        send, recv = self.euler_local(q)
        transport.exchange(send, recv)
        return self.euler_finish(out)


def setup_distributed(layout, cfg, dt, transport):
    """Collective construction of one rank's operator (setup exchange included)."""
    op = SlabHyperDiffusion(layout, cfg, dt)
    transport.exchange(op.setup_send, op.setup_recv)
    return op.setup_finish()


def run_loopback(ops, qs, outs):
    """H_nu on all slabs of one process (1-GPU test of the device pipeline), in the same
    interface-tiles / exchange / interior-tiles / finish order as ``apply``."""
    alpha = ops[0].cfg.alpha
    for k in range(alpha):
        for op, q, o in zip(ops, qs, outs):
            op.pass_local(k, q, o, "ext")
        LoopbackTransport.exchange_all([halo_views(op.halo, len(op.cfg.variables)) for op in ops])
        for op, q, o in zip(ops, qs, outs):
            op.pass_local(k, q, o, "int")
        for op in ops:
            op.pass_finish()
    return outs


def run_loopback_euler(ops, qs, outs):
    """S + H_nu on all slabs of one process (1-GPU test of the slab Euler pipeline)."""
    run_loopback(ops, qs, outs)
    bufs = [op.euler_local(q) for op, q in zip(ops, qs)]
    LoopbackTransport.exchange_all(bufs)
    for op, o in zip(ops, outs):
        op.euler_finish(o)
    return outs


def setup_loopback(layouts, cfg, dt):
    ops = [SlabHyperDiffusion(L, cfg, dt) for L in layouts]
    LoopbackTransport.exchange_all([(op.setup_send, op.setup_recv) for op in ops])
    return [op.setup_finish() for op in ops]
