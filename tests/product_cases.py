"""Product-side construction of the parity cases (runs the CUDA path)."""

from __future__ import annotations

from cases import CASES, window_args
from paper_2311_11425_b200 import euler, hyperdiff, mesh as hm, metrics, state


def product_mesh(name, case=None):
    c = CASES[name] if case is None else case
    if c["kind"] == "lattice":
        return hm.build_box_lattice(c["nx"], c["ny"], c["nv"], c["N"], c["extents"])
    if c["kind"] == "window":
        return hm.build_box_window(*window_args(c))
    if c["kind"] == "sphere":
        return hm.build_cubed_sphere(hm.MeshConfig("sphere", panels_per_edge=c["ne"], n_elem_vertical=c["nv"],
                                                   degree=c["N"], radius=c["radius"], z_top=c["z_top"]))
    return hm.build_box(hm.MeshConfig("box", panels_per_edge=c["ne"], n_elem_vertical=c["nv"], degree=c["N"],
                                      box_extents=c["extents"]))


class ProductProblem:
    def __init__(self, name, set_name="2C", case=None):
        c = CASES[name] if case is None else case
        self.c = c
        self.m = product_mesh(name, c)
        self.mets0 = metrics.curl_invariant_metrics(self.m)
        self.mets = metrics.project_metrics_to_columns(self.mets0, self.m)
        self.cfg = hyperdiff.HyperDiffConfig(**c["hd"])
        self.vm = hyperdiff.build_viscous_metric(self.m, self.mets, self.cfg, dt=c["dt"])
        self.consts = state.PhysConstants(omega=c["omega"])
        self.ops = euler.EulerOps(self.m, self.mets, self.consts, set_name, hyper=(self.cfg, self.vm))
