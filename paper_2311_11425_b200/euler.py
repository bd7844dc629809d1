"""EulerOps on the B200: S(q), H(q) and the hyper-diffusion plan (mirror of euler.py:27-144).

``EulerOps`` owns the device-resident operator data (mass, gathered metric,
Laplacian plan) and exposes the reference's entry points.  The hot operators
run in ``libhv_b200.so``.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .assembly import GlobalMass, weights3
from .device import torch_mod

__all__ = ["EulerOps"]


class EulerOps:
    """euler.py:27-35: mesh, metrics, constants, equation set, optional (cfg, viscous)."""

    def __init__(self, mesh, mets, constants, set_name, hyper=None):
        if set_name not in ("2NC", "2C", "3C"):
            raise ValueError(f"unknown equation set {set_name!r}")
        self.mesh = mesh
        self.metrics = mets
        self.c = constants
        self.set_name = set_name
        self.hyper = hyper
        self.mass = GlobalMass(mesh, mets.d_J)
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
            self._plans[key] = (p, viscous, W)
        return self._plans[key][0]

    # ------------------------------------------------------------ operators
    def rhs_full(self, state):
        """S(q) (euler.py:111-118)."""
        raise NotImplementedError("rhs_full: fused Euler kernel not built yet")

    def rhs_horizontal(self, state, with_hyperdiff=True):
        """H(q) (euler.py:122-134)."""
        raise NotImplementedError("rhs_horizontal: fused Euler kernel not built yet")
