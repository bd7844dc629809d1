"""EulerOps on the B200: S(q), H(q) and the hyper-diffusion plan (mirror of euler.py:27-144).

``EulerOps`` owns the device-resident operator data (mass, gathered metric,
Laplacian plan) and exposes the reference's entry points.  The hot operators
run in ``libhv_b200.so``.
"""

from __future__ import annotations

import os

import ctypes as C

import numpy as np

from . import _lib
from .assembly import GlobalMass, weights3
from .device import to_dev, torch_mod
from .tiles import build_chunk_table

__all__ = ["EulerOps"]


class EulerOps:
    """euler.py:27-35: mesh, metrics, constants, equation set, optional (cfg, viscous)."""

    def __init__(self, mesh, mets, constants, set_name, hyper=None, mass=None, ext_cols=None):
        """``mass`` / ``ext_cols``: supplied by the multi-GPU slab decomposition (parallel.py):
        the cross-rank mass and the slab-interface column nodes."""
        if set_name not in ("2NC", "2C", "3C"):
            raise ValueError(f"unknown equation set {set_name!r}")
        self.mesh = mesh
        self.metrics = mets
        self.c = constants
        self.set_name = set_name
        self.hyper = hyper
        self.mass = mass if mass is not None else GlobalMass(mesh, mets.d_J)
        self.ext_cols = ext_cols
        self.ext_face = 0
        self.halo = None
        self.w3 = weights3(mesh)
        self._plans = {}
        self._work = None
        self._h = {}

    # ------------------------------------------------------------ host views
    @property
    def Jg_e(self):
        """Projected (or naive) gridpoint J gathered to elements (euler.py:42)."""
        if "Jg_e" not in self._h:
            self._h["Jg_e"] = self.metrics.Jg[self.mesh.gid]
        return self._h["Jg_e"]

    # ------------------------------------------------------------ device plan
    def _workspace(self):
        if self._work is None:
            torch = torch_mod()
            dev = self.mesh.device()
            self._work = (torch.empty(5 * dev.nloc, dtype=torch.float64, device="cuda"),
                          torch.empty(5 * dev.nglobal, dtype=torch.float64, device="cuda"))
        return self._work

    def _tile_arrays(self):
        """Device copy of the tile plan (tiles.py), or None for meshes it does not fit."""
        if "tiles" not in self._h:
            from .tiles import build_tile_plan, tile_shape

            dev = self.mesh.device()
            tp = None
            if os.environ.get("HV_DISABLE_TILES", "0") != "1" and dev.N <= 7:
                tp = build_tile_plan(self.mesh, *tile_shape(dev.N), ext_cols=self.ext_cols)
            if tp is None:
                self._h["tiles"] = None
            else:
                torch = torch_mod()
                d = {k: to_dev(getattr(tp, k)) for k in ("gt", "code", "tmeta", "slot_col", "slot_row0", "slot_nc",
                                                         "slot_ext", "ext_slots")}
                d["elem"] = to_dev(tp.elem.reshape(tp.ntiles, tp.nlay, -1).astype(np.int32))
                d["col_gid"] = to_dev(self.mesh.col_gid.astype(np.int32))
                d["part"] = torch.empty(max(1, tp.npart) * tp.n_z * 5, dtype=torch.float64, device="cuda")
                self._h["tiles"] = (tp, d)
        return self._h["tiles"]

    def _slot_minv(self, d):
        """Minv of the shared column nodes in slot order, (nslot, n_z): the fix-up reads it coalesced."""
        if d["slot_col"].numel() == 0:
            return None
        cols = d["col_gid"][d["slot_col"].long()].long()
        return self.mass.d_Minv[cols].contiguous()

    @staticmethod
    def _segments(tp):
        """Layers per vertical segment of the N <= 4 plane sweep (hv_lap_plan.seg), 0 = whole columns.
        A mesh with fewer tiles than one wave of CTA slots (148 SMs x 4) is swept as two half columns
        (config 2: 256 tiles x 8 layers -> 512 CTAs of 4 layers: 0.114 -> 0.102 ms per H_nu op; 8 or 4
        segments measured 0.132 / 0.114 ms, and config 3's 1350 tiles lose with 2, 0.46 -> 0.52 ms).
        HV_SEG (layers per segment) overrides."""
        env = os.environ.get("HV_SEG", "")
        if env:
            seg = int(env)
        else:
            if tp.ntiles >= 148 * 4 or tp.nlay < 2:
                return 0
            seg = -(-tp.nlay // 2)
        return seg if 0 < seg < tp.nlay else 0

    def _yt_chain(self, tp, d):
        """(tper, yt, sv) for H_nu's tile-ordered intermediate (hv_lap_plan.d_yt), or
        None when the plane kernel has no tile-ordered mode for this plan (or HV_YT=0)."""
        if os.environ.get("HV_YT", "1") == "0":
            return None
        # N = 7: the split-plane kernel with H = 4 only (HV_YT7=0 keeps the rows intermediate there)
        if tp.N == 7 and (os.environ.get("HV_YT7", "1") != "1" or os.environ.get("HV_N7_SPLIT", "") == "2"):
            return None
        lay = np.zeros(5, dtype=np.int64)
        if _lib.lib().hv_plane_yt_layout(tp.N, tp.TX, tp.TY, 4, lay.ctypes.data) != 0:
            return None
        torch = torch_mod()
        blk, nper = int(lay[3]), int(lay[4])
        U, V = tp.U, tp.V
        # perimeter column p -> (u, v), the order of hv_plane_yt_layout
        pu = [0] * V + [U - 1] * V + list(range(1, U - 1)) * 2
        pv = list(range(V)) * 2 + [0] * (U - 2) + [V - 1] * (U - 2)
        assert len(pu) == nper
        rows = tp.code[:, pu, pv]                                             # (ntiles, NPER) partial row or -1
        slot = np.searchsorted(tp.slot_row0, np.maximum(rows, 0), side="right") - 1
        slot = np.where(rows >= 0, slot, -1)
        yus = int(lay[1])
        off = np.asarray(pu) * yus + np.asarray(pv)
        # per tile: its slot columns in slot order (the stage), runs of consecutive slots (one bulk copy each)
        tper = np.full((tp.ntiles, nper + 96), -1, dtype=np.int32)
        tper[:, nper:] = 0
        for t in range(tp.ntiles):
            m = slot[t] >= 0
            order = np.argsort(slot[t][m], kind="stable")
            s_sorted = slot[t][m][order]
            tper[t, :len(s_sorted)] = off[m][order]
            if len(s_sorted):
                brk = np.nonzero(np.diff(s_sorted) != 1)[0] + 1
                starts = np.concatenate([[0], brk])
                cnts = np.diff(np.concatenate([starts, [len(s_sorted)]]))
                if len(starts) > 32:
                    return None
                tper[t, nper:nper + 3 * len(starts):3] = s_sorted[starts]
                tper[t, nper + 1:nper + 3 * len(starts):3] = cnts
                tper[t, nper + 2:nper + 3 * len(starts):3] = starts
        yt = torch.zeros(tp.ntiles * (tp.nlay + 1) * blk, dtype=torch.float64, device="cuda")
        sv = torch.zeros(max(1, tp.nslot) * tp.n_z * 4, dtype=torch.float64, device="cuda")
        return to_dev(tper), yt, sv

    def lap_plan(self, viscous):
        """hv_lap_plan for this (viscous metric, operator set) pair."""
        key = id(viscous)
        if key not in self._plans:
            dev = self.mesh.device()
            W = viscous.packed(self.metrics.d_Jg)
            work, y = self._workspace()
            p = _lib.LapPlan()
            p.N = dev.N
            n = dev.n
            for i in range(n):
                for a in range(n):
                    p.D[i * n + a] = float(dev.D[i, a])
            p.nelem = dev.nelem
            p.nglobal = dev.nglobal
            p.d_gid = dev.gid32.data_ptr()
            p.d_off = dev.off.data_ptr()
            p.d_idx = dev.idx.data_ptr()
            p.d_W = W.data_ptr()
            p.d_Minv = self.mass.d_Minv.data_ptr()
            p.d_work = work.data_ptr()
            p.d_y = y.data_ptr()
            keep = [viscous, W]
            ta = self._tile_arrays()
            if ta is not None:
                torch = torch_mod()
                tp, d = ta
                # plane-owner kernel (lap_plane.cu) for N <= 4 and N = 7 (split planes; the line
                # kernel with HV_N7_KERNEL=line), line-tile kernel otherwise;
                # HV_KERNEL=line forces the line-tile kernel (cross-checks)
                n7p = dev.N == 7 and os.environ.get("HV_N7_KERNEL", "") != "line"
                layout = 1 if (os.environ.get("HV_KERNEL", "") != "line" and (dev.N <= 4 or n7p)) else 0
                # compact forms of W for the plane kernel: isotropic (G_nu = kh I: 1 double per node)
                # or axis (G_nu = kh I + kd e3 e3^T: 3 doubles; N <= 4 -- the N = 7 split-plane kernel
                # spills with it, c4 6.91 -> 7.04 ms); HV_WFORM=0 forces the 6 components (cross-checks),
                # HV_WFORM=1 the axis form also at N = 7 / for isotropic viscosity
                wf = os.environ.get("HV_WFORM", "")
                ax = viscous.axis_form() if layout == 1 and wf != "0" else None
                wform = 0
                if ax is not None and ax[1] == 0.0 and wf != "1":
                    wform = 2
                elif ax is not None and ax[1] != 0.0 and (dev.N <= 4 or wf == "1"):
                    wform = 1
                ncomp = {0: 6, 1: 3, 2: 1}[wform]
                wl = (_lib.lib().hv_plane_metric_doubles(dev.N, tp.TX, tp.TY, wform) if layout == 1
                      else 6 * n * tp.NE * n * n)
                Wt = torch.empty(tp.ntiles * tp.nlay * wl, dtype=torch.float64, device="cuda")
                # isotropic: s = kh w3 Jg; axis: u = sqrt(|kd| w3 Jg) e_3 (the sweep then needs no kd multiply)
                src = viscous.packed_axis(self.metrics.d_Jg, ncomp, ax[0] if wform == 2 else abs(ax[1])) if wform else W
                _lib.check(_lib.lib().hv_tile_pack_metric(dev.N, tp.TX, tp.TY, tp.ntiles, tp.nlay,
                                                          d["elem"].data_ptr(), src.data_ptr(), dev.nloc,
                                                          wform + 1 if wform else layout, Wt.data_ptr(),
                                                          _lib.stream_handle()))
                p.kernel = layout
                if wform:
                    p.wform, p.kh, p.kd = wform, ax[0], ax[1]
                del src
                p.TX, p.TY, p.nlay, p.n_z = tp.TX, tp.TY, tp.nlay, tp.n_z
                p.ntiles, p.nslot = tp.ntiles, tp.nslot
                p.d_gt, p.d_code, p.d_tmeta = d["gt"].data_ptr(), d["code"].data_ptr(), d["tmeta"].data_ptr()
                p.d_slot_col, p.d_slot_row0 = d["slot_col"].data_ptr(), d["slot_row0"].data_ptr()
                p.d_slot_nc, p.d_col_gid = d["slot_nc"].data_ptr(), d["col_gid"].data_ptr()
                Mt = torch.empty(tp.ntiles * tp.nlay * tp.mts, dtype=torch.float64, device="cuda")
                _lib.check(_lib.lib().hv_tile_pack_minv(tp.ntiles * tp.nlay, tp.gts, tp.mts, d["gt"].data_ptr(),
                                                        self.mass.d_Minv.data_ptr(), Mt.data_ptr(),
                                                        _lib.stream_handle()))
                p.d_Wt, p.d_Mt, p.d_part = Wt.data_ptr(), Mt.data_ptr(), d["part"].data_ptr()
                Ms = self._slot_minv(d)
                p.d_Ms = _lib.ptr(Ms)
                keep += [Wt, Mt, Ms]
                seg = self._segments(tp) if layout == 1 and dev.N <= 4 and not self.ext_cols else 0
                yt = self._yt_chain(tp, d) if layout == 1 and not self.ext_cols and not seg else None
                if yt is not None:
                    p.d_tper, p.d_yt, p.d_sv = (x.data_ptr() for x in yt)
                    keep += list(yt)
                    # pass 1's input by bulk copies of gid runs (lattice-numbered meshes; HV_CHUNK=0: gather)
                    cap = _lib.lib().hv_plane_chunk_rows(tp.N, tp.TX, tp.TY)
                    ct = (build_chunk_table(tp, cap) if cap > 0 and os.environ.get("HV_CHUNK", "1") != "0"
                          else None)
                    if ct is not None:
                        ct = to_dev(ct)
                        p.d_tchunk = ct.data_ptr()
                        keep.append(ct)
                if seg:
                    nseg = -(-tp.nlay // seg)
                    t, u, v = np.nonzero(tp.code >= 0)
                    prow = np.zeros(max(1, tp.npart), dtype=np.int32)
                    prow[tp.code[t, u, v]] = (t * tp.U * tp.V + u * tp.V + v).astype(np.int32)
                    bnd = torch.zeros(tp.ntiles * (nseg - 1) * 2 * tp.U * tp.V * 5, dtype=torch.float64,
                                      device="cuda")
                    prow = to_dev(prow)
                    p.seg, p.d_bnd, p.d_prow = seg, bnd.data_ptr(), prow.data_ptr()
                    keep += [bnd, prow]
                if self.ext_cols:
                    face = self.ext_face
                    p.d_slot_ext, p.d_ext_slots = d["slot_ext"].data_ptr(), d["ext_slots"].data_ptr()
                    p.next, p.face = len(tp.ext_slots), face
                    send = torch.zeros((2, face, tp.n_z, 5), dtype=torch.float64, device="cuda")
                    recv = torch.zeros_like(send)
                    p.d_send, p.d_recv = send.data_ptr(), recv.data_ptr()
                    self.halo = (send, recv)
                    keep += [send, recv]
            self._plans[key] = (p, keep)
        return self._plans[key][0]

    # ------------------------------------------------------------ Euler RHS
    _SETS = {"2NC": 0, "2C": 1, "3C": 2}

    @property
    def Phi_g(self):
        """Geopotential g*height at the gridpoints (euler.py:48-53), host."""
        if "Phi_g" not in self._h:
            m = self.mesh
            if m.cfg.geometry == "sphere":
                self._h["Phi_g"] = self.c.g * m.height()
            else:
                self._h["Phi_g"] = self.c.g * m.xg[:, 2]
        return self._h["Phi_g"]

    def _euler_record(self):
        """Per element node RHS record on the device (hv_euler_setup)."""
        if "euler_M" not in self._h:
            torch = torch_mod()
            dev = self.mesh.device()
            M = torch.empty((18, dev.nloc), dtype=torch.float64, device="cuda")
            phi = to_dev(np.ascontiguousarray(self.Phi_g, dtype=np.float64))
            mask = to_dev(np.ascontiguousarray(self.mesh.flux_mask, dtype=np.float64))
            _lib.check(_lib.lib().hv_euler_setup(
                dev.N, dev.D.ctypes.data, dev.nelem, dev.gid32.data_ptr(), self.metrics.d_grad.data_ptr(),
                self.metrics.d_Jg.data_ptr(), self.metrics.d_gz.data_ptr(), phi.data_ptr(), mask.data_ptr(),
                dev.coords.data_ptr(), int(self.mesh.cfg.geometry == "sphere"), M.data_ptr(), _lib.stream_handle()))
            self._h["euler_M"] = M
        return self._h["euler_M"]

    def _euler_tile_plan(self):
        """hv_lap_plan carrying the single-column tile plan for hv_euler_rhs_tiles (N = 7), or None."""
        if "euler_tiles" not in self._h:
            self._h["euler_tiles"] = None
            ta = self._tile_arrays()
            if ta is not None and os.environ.get("HV_EULER_TILES", "1") != "0" and not self.ext_cols:
                tp, d = ta
                if tp.TX == 1 and tp.TY == 1:
                    torch = torch_mod()
                    dev = self.mesh.device()
                    p = _lib.LapPlan()
                    p.N = dev.N
                    n = dev.n
                    for i in range(n):
                        for a in range(n):
                            p.D[i * n + a] = float(dev.D[i, a])
                    p.nelem, p.nglobal = dev.nelem, dev.nglobal
                    p.d_gid, p.d_Minv = dev.gid32.data_ptr(), self.mass.d_Minv.data_ptr()
                    p.TX, p.TY, p.nlay, p.n_z = 1, 1, tp.nlay, tp.n_z
                    p.ntiles, p.nslot = tp.ntiles, tp.nslot
                    p.d_gt, p.d_code, p.d_tmeta = d["gt"].data_ptr(), d["code"].data_ptr(), d["tmeta"].data_ptr()
                    p.d_slot_col, p.d_slot_row0 = d["slot_col"].data_ptr(), d["slot_row0"].data_ptr()
                    p.d_slot_nc, p.d_col_gid = d["slot_nc"].data_ptr(), d["col_gid"].data_ptr()
                    Mt = torch.empty(tp.ntiles * tp.nlay * tp.mts, dtype=torch.float64, device="cuda")
                    _lib.check(_lib.lib().hv_tile_pack_minv(tp.ntiles * tp.nlay, tp.gts, tp.mts, d["gt"].data_ptr(),
                                                            self.mass.d_Minv.data_ptr(), Mt.data_ptr(),
                                                            _lib.stream_handle()))
                    p.d_Mt, p.d_part = Mt.data_ptr(), d["part"].data_ptr()
                    Ms = self._slot_minv(d)
                    p.d_Ms = _lib.ptr(Ms)
                    elem = d["elem"].reshape(tp.ntiles, tp.nlay).contiguous()
                    self._h["euler_tiles"] = (p, [Mt, elem, Ms], elem)
        return self._h["euler_tiles"]

    def _rhs(self, state, dirs, coriolis, out=None, accumulate=False):
        from .hyperdiff import _as_device

        torch = torch_mod()
        data = state.data if hasattr(state, "data") else state
        q, host = _as_device(data)
        if q.dim() != 2 or q.shape[1] != 5:
            raise ValueError("state data must be (nglobal, 5)")
        dev = self.mesh.device()
        M = self._euler_record()
        if out is None:
            out = torch.empty_like(q)
        k = self.c
        et = self._euler_tile_plan()
        if et is not None:
            p, _, elem = et
            _lib.check(_lib.lib().hv_euler_rhs_tiles(
                C.byref(p), elem.data_ptr(), dev.w3.data_ptr(), self._SETS[self.set_name], dirs, coriolis, k.P_A, k.R,
                k.gamma, k.omega, M.data_ptr(), q.data_ptr(), 5, out.data_ptr(), 5, int(bool(accumulate)),
                _lib.stream_handle()))
            return out, host
        work, _ = self._workspace()
        if "elem_layer" not in self._h:
            self._h["elem_layer"] = to_dev(np.ascontiguousarray(self.mesh.elem_layer, dtype=np.int32))
        _lib.check(_lib.lib().hv_euler_rhs(
            dev.N, dev.D.ctypes.data, self._SETS[self.set_name], dirs, coriolis, k.P_A, k.R, k.gamma, k.omega,
            dev.nelem, dev.nglobal, dev.gid32.data_ptr(), self._h["elem_layer"].data_ptr(),
            self.mesh.cfg.n_elem_vertical, dev.w3.data_ptr(), M.data_ptr(), dev.off.data_ptr(),
            dev.idx.data_ptr(), self.mass.d_Minv.data_ptr(), q.data_ptr(), 5, work.data_ptr(), out.data_ptr(), 5,
            int(bool(accumulate)), _lib.stream_handle()))
        return out, host

    # ------------------------------------------------------------ operators
    def rhs_full(self, state, out=None):
        """S(q) with Coriolis 2 omega rhat x u; hyper-diffusion excluded (euler.py:111-118)."""
        o, host = self._rhs(state, 7, 0, out=out)
        return o.cpu().numpy() if host else o

    def rhs_horizontal(self, state, with_hyperdiff=True, out=None):
        """H(q): xi/eta terms, Coriolis 2 omega zetahat x u, plus H_nu (euler.py:122-134)."""
        o, host = self._rhs(state, 3, 1, out=out)
        if self.hyper is not None and with_hyperdiff:
            from .hyperdiff import hyperdiffusion_apply
            from .state import StateField

            cfg, viscous = self.hyper
            data = state.data if hasattr(state, "data") else state
            qd = o.new_tensor(data) if host else data
            hyperdiffusion_apply(StateField(self.set_name, qd), cfg, viscous, self, out=o, accumulate=True)
        return o.cpu().numpy() if host else o

    def rhs_full_hyper(self, state, out=None):
        """S(q) + H_nu(q) in one output (the config-4 quantity; extension)."""
        if self.hyper is None:
            raise ValueError("rhs_full_hyper needs EulerOps(..., hyper=(cfg, viscous))")
        from .hyperdiff import _as_device, hyperdiffusion_apply
        from .state import StateField

        data = state.data if hasattr(state, "data") else state
        qd, host = _as_device(data)
        # H_nu first (plain row writes from the sweep), then S accumulated by the streaming
        # DSS kernel: S + H == H + S bitwise, and the read-modify-write moves out of the sweep
        cfg, viscous = self.hyper
        o = hyperdiffusion_apply(StateField(self.set_name, qd), cfg, viscous, self, out=out)
        self._rhs(qd, 7, 0, out=o, accumulate=True)
        return o.cpu().numpy() if host else o

    def _column_arrays(self):
        if "cols" not in self._h:
            phi = to_dev(np.ascontiguousarray(self.Phi_g, dtype=np.float64))
            mask = to_dev(np.ascontiguousarray(self.mesh.flux_mask, dtype=np.float64))
            cg = to_dev(np.ascontiguousarray(self.mesh.col_gid, dtype=np.int32))
            self._h["cols"] = (cg, mask, phi)
        return self._h["cols"]

    # ------------------------------------------------------------ diagnostics
    DIAG_KEYS = ("mass", "energy_internal", "energy_kinetic", "energy_potential", "energy_total", "p_surface_min",
                 "w_vertical_max")

    def diagnostics(self, state):
        """Quadrature-weighted global integrals and surface extrema (euler.py:421-456), one
        deterministic device reduction (hv_euler_diagnostics)."""
        from .hyperdiff import _as_device

        torch = torch_mod()
        data = state.data if hasattr(state, "data") else state
        q, _ = _as_device(data)
        cg, _, phi = self._column_arrays()
        sphere = int(self.mesh.cfg.geometry == "sphere")
        if sphere and "xg_dev" not in self._h:
            self._h["xg_dev"] = to_dev(np.ascontiguousarray(self.mesh.xg, dtype=np.float64))
        xg = self._h["xg_dev"] if sphere else None
        work = torch.empty(7 * 592, dtype=torch.float64, device="cuda")
        out = torch.empty(7, dtype=torch.float64, device="cuda")
        k = self.c
        _lib.check(_lib.lib().hv_euler_diagnostics(
            self._SETS[self.set_name], k.P_A, k.R, k.gamma, k.c_v, sphere, q.shape[0], q.data_ptr(),
            self.mass.d_M.data_ptr(), phi.data_ptr(), xg.data_ptr() if xg is not None else None, self.mesh.ncol,
            self.mesh.n_z, cg.data_ptr(), work.data_ptr(), out.data_ptr(), _lib.stream_handle()))
        return dict(zip(self.DIAG_KEYS, (float(v) for v in out.cpu().numpy())))

    # ------------------------------------------------------------ LHEVI column systems
    @property
    def nzl(self):
        return self.mesh.device().N + 1

    nvar = 5

    @property
    def kl(self):
        """Half bandwidth nvar * nzl - 1 (euler.py:84-85)."""
        return self.nvar * self.nzl - 1

    ku = kl

    @property
    def Mdim(self):
        return self.nvar * self.mesh.n_z

    @property
    def ncol(self):
        return self.mesh.ncol

    def column_jacobian(self, qcol, lam):
        """Band batch of I - lam dV/dq about the column state qcol (ncol, n_z, 5)
        (euler.py:274-306), LAPACK band layout (ncol, 2 kl + ku + 1, 5 n_z)."""
        from .hyperdiff import _as_device

        torch = torch_mod()
        q, host = _as_device(qcol)
        q = q.contiguous()
        ncol = q.shape[0]
        if tuple(q.shape[1:]) != (self.mesh.n_z, 5) or ncol > self.mesh.ncol:
            raise ValueError("qcol must be (ncol, n_z, 5)")
        dev = self.mesh.device()
        cg, mask, phi = self._column_arrays()
        band = torch.empty((ncol, 2 * self.kl + self.ku + 1, self.Mdim), dtype=torch.float64, device="cuda")
        wz = np.ascontiguousarray(self.mesh.bases[2].weights, dtype=np.float64)
        k = self.c
        _lib.check(_lib.lib().hv_column_jacobian(
            dev.N, dev.D.ctypes.data, wz.ctypes.data, self._SETS[self.set_name], k.P_A, k.R, k.gamma, float(lam),
            ncol, self.mesh.cfg.n_elem_vertical, self.mesh.n_z, cg.data_ptr(), q.data_ptr(),
            self.metrics.d_Jg.data_ptr(), self.metrics.d_gz.data_ptr(), mask.data_ptr(), phi.data_ptr(),
            band.data_ptr(), _lib.stream_handle()))
        return band.cpu().numpy() if host else band

    def column_apply(self, qcol):
        """V on column-gathered states qcol (ncol, n_z, 5) -> (ncol, n_z, 5) (euler.py:231-235)."""
        from .hyperdiff import _as_device

        q, host = _as_device(qcol)
        if tuple(q.shape) != (self.mesh.ncol, self.mesh.n_z, 5):
            raise ValueError("qcol must be (ncol, n_z, 5)")
        torch = torch_mod()
        cg, _, _ = self._column_arrays()
        idx = cg.long()
        qg = torch.empty((self.mesh.nglobal, 5), dtype=torch.float64, device="cuda")
        qg[idx.reshape(-1)] = q.reshape(-1, 5)
        v = self.rhs_vertical(qg)[idx]
        return v.cpu().numpy() if host else v

    def rhs_vertical(self, state, out=None, accumulate=False):
        """V(q) assembled from the independent column evaluations (euler.py:138-144, 231-272)."""
        from .hyperdiff import _as_device

        torch = torch_mod()
        data = state.data if hasattr(state, "data") else state
        q, host = _as_device(data)
        dev = self.mesh.device()
        cg, mask, phi = self._column_arrays()
        if out is None:
            out = torch.empty_like(q)
        wz = np.ascontiguousarray(self.mesh.bases[2].weights, dtype=np.float64)
        k = self.c
        _lib.check(_lib.lib().hv_euler_vertical(
            dev.N, dev.D.ctypes.data, wz.ctypes.data, self._SETS[self.set_name], k.P_A, k.R, k.gamma,
            self.mesh.ncol, self.mesh.cfg.n_elem_vertical, self.mesh.n_z, cg.data_ptr(), self.metrics.d_Jg.data_ptr(),
            self.metrics.d_gz.data_ptr(), mask.data_ptr(), phi.data_ptr(), q.data_ptr(), 5, out.data_ptr(), 5,
            int(bool(accumulate)), _lib.stream_handle()))
        return out.cpu().numpy() if host else out
