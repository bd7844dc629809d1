"""Oracle-side construction of the parity cases (test infrastructure)."""

from __future__ import annotations

import numpy as np

from cases import CASES, case_state, window_args
from oracle import hevi_oracle as O
from paper_2311_11425_b200 import synthetic


def oracle_mesh(name, case=None):
    c = CASES[name] if case is None else case
    if c["kind"] == "lattice":
        coords, layer, hcol = synthetic.perturbed_box_coords(c["nx"], c["ny"], c["nv"], c["N"], c["extents"])
        tol = O.dedupe_tol("box", max(c["nx"], c["ny"]), extents=c["extents"])
        return O.OracleMesh.from_coords("box", c["N"], coords, layer, hcol, tol)
    if c["kind"] == "window":
        coords, layer, hcol = synthetic.box_window_coords(*window_args(c))
        tol = O.dedupe_tol("box", max(c["nx"], c["ny"]), extents=c["extents"])
        return O.OracleMesh.from_coords("box", c["N"], coords, layer, hcol, tol)
    if c["kind"] == "sphere":
        coords, layer, hcol = O.sphere_coords(c["ne"], c["nv"], c["N"], c["radius"], c["z_top"])
        tol = O.dedupe_tol("sphere", c["ne"], radius=c["radius"])
        return O.OracleMesh.from_coords("sphere", c["N"], coords, layer, hcol, tol, radius=c["radius"])
    coords, layer, hcol = O.box_coords(c["ne"], c["nv"], c["N"], c["extents"])
    tol = O.dedupe_tol("box", c["ne"], extents=c["extents"])
    return O.OracleMesh.from_coords("box", c["N"], coords, layer, hcol, tol)


class OracleProblem:
    """Mesh + projected curl-invariant metrics + G_nu + mass for one case."""

    def __init__(self, name, case=None):
        c = CASES[name] if case is None else case
        self.name, self.c = name, c
        self.m = m = oracle_mesh(name, c)
        self.dxdxi, self.J, self.grad = O.curl_metrics(m)
        self.Jg0, self.gz0 = O.naive_gridpoint(m, self.J, self.grad)
        self.Jg, self.gz = O.project_columns(m, self.J, self.grad)
        self.M, self.Minv = O.lumped_mass(m, self.J)
        hd = dict(c["hd"])
        alpha = hd.pop("alpha")
        self.alpha = alpha
        self.Gnu, self.lam, self.evecs = O.viscous_metric(m, self.grad, alpha, dt=c["dt"], **hd)
        self.Jg_e = O.gather(m.gid, self.Jg)
        self.state = case_state(name, m.xg, None if case is None else c)

    def hyper(self, data=None):
        return O.hyperdiffusion(self.m, self.Gnu, self.Jg_e, self.Minv,
                                self.state if data is None else data, self.alpha)

    def lap(self, f):
        return O.laplacian(self.m, self.Gnu, self.Jg_e, self.Minv, self.state[:, f])

    def euler(self, set_name, omega=None):
        k = O.Consts(omega=self.c["omega"] if omega is None else omega)
        return O.OracleEuler(self.m, self.J, self.grad, self.Jg, self.gz, k, set_name)
