"""Tensor hyper-diffusion on the B200: viscous metric and the alpha-fold Laplacian.

Mirror of reference hyperdiff.py:18-106.  ``build_viscous_metric`` runs the
per-node eigensolve kernel; ``laplacian_apply`` / ``hyperdiffusion_apply``
run the fused element kernels with on-chip DSS (``hv_laplacian`` /
``hv_hyperdiffusion``).  Inputs may be numpy arrays (copied to the device and
the result copied back, reference semantics) or CUDA tensors (device
resident, result returned as a CUDA tensor).
"""

from __future__ import annotations

import ctypes as C
import os
import weakref
from collections import OrderedDict
from dataclasses import dataclass

import numpy as np

from . import _lib
from .device import torch_mod

__all__ = ["HyperDiffConfig", "ViscousMetric", "scaled_viscosity", "build_viscous_metric",
           "laplacian_apply", "hyperdiffusion_apply"]

_MODES = {"scaled": 0, "constant": 1, "anisotropic": 2}


@dataclass
class HyperDiffConfig:
    """hyperdiff.py:18-37 (same defaults and validation)."""

    alpha: int = 2
    mode: str = "scaled"
    c: tuple = (0.0045, 0.0045, 0.0001)
    nu: tuple = (0.0, 0.0, 0.0)
    nu_h: float = 0.0
    nu_v: float = 0.0
    variables: tuple = (1, 2, 3, 4)
    final_stage_only: bool = False

    def __post_init__(self):
        if self.alpha not in (1, 2):
            raise ValueError("alpha must be 1 or 2")
        if self.mode not in _MODES:
            raise ValueError(f"unknown hyperdiff mode {self.mode!r}")
        if min(self.c) < 0 or min(self.nu) < 0 or self.nu_h < 0 or self.nu_v < 0:
            raise ValueError("coefficients must be >= 0")
        if 0 in self.variables:
            raise ValueError("hyper-diffusing density is out of scope")


def scaled_viscosity(c, lam, N, dt, alpha):
    """nu_i = c_i^(1/alpha) 4 lambda_i / (N^2 dt^(1/alpha)) (hyperdiff.py:54-59); host helper."""
    if dt <= 0:
        raise ValueError("scaled viscosities need dt > 0")
    c = np.asarray(c, dtype=float)
    return (c ** (1.0 / alpha)) * 4.0 * lam / (N**2 * dt ** (1.0 / alpha))


class ViscousMetric:
    """G_nu per element node plus eigen-data of G (hyperdiff.py:40-51).

    Only the parameters and the packed Laplacian metric live on the device;
    ``Gnu`` (nelem,n,n,n,3,3), ``lam`` (..,3) and ``evecs`` (..,3,3) are
    materialised on first access.  No tau tensor is stored.
    """

    def __init__(self, mesh, mets, cfg, params):
        self.mesh, self.mets, self.cfg = mesh, mets, cfg
        self._params = params  # (mode, a[3], b, nu[3])
        self._host = None
        self._packed = {}

    def _run(self, d_Jg=None, want_host=False, W=None):
        torch = torch_mod()
        dev = self.mesh.device()
        mode, a, b, nu = self._params
        a = np.ascontiguousarray(a, dtype=np.float64)
        nu = np.ascontiguousarray(nu, dtype=np.float64)
        G = lam = V = None
        if want_host:
            G = torch.empty((dev.nloc, 3, 3), dtype=torch.float64, device="cuda")
            lam = torch.empty((dev.nloc, 3), dtype=torch.float64, device="cuda")
            V = torch.empty((dev.nloc, 3, 3), dtype=torch.float64, device="cuda")
        _lib.check(_lib.lib().hv_viscous_metric(
            dev.N, mode, a.ctypes.data, float(b), nu.ctypes.data, self.mets.d_grad.data_ptr(), dev.nelem,
            dev.w3.data_ptr(), _lib.ptr(d_Jg), dev.gid32.data_ptr(), _lib.ptr(G), _lib.ptr(lam), _lib.ptr(V),
            _lib.ptr(W), _lib.stream_handle()))
        return G, lam, V

    def _materialise(self):
        if self._host is None:
            G, lam, V = self._run(want_host=True)
            shp = (self.mesh.nelem,) + tuple(self.mesh.shape)
            self._host = (G.cpu().numpy().reshape(shp + (3, 3)), lam.cpu().numpy().reshape(shp + (3,)),
                          V.cpu().numpy().reshape(shp + (3, 3)))
        return self._host

    @property
    def Gnu(self):
        return self._materialise()[0]

    @property
    def lam(self):
        return self._materialise()[1]

    @property
    def evecs(self):
        return self._materialise()[2]

    def axis_form(self):
        """(kh, kd) when G_nu = kh I + kd e_3 e_3^T exactly (scaled mode, c_1 == c_2), else None.

        hyperdiff.py:71-80: k_m = nu_m vals_m = ((a_m lam_m) / b) vals_m = a_m / b to an ulp, so with
        a_1 == a_2 the two horizontal modes share one coefficient and only e_3 carries geometry.
        """
        mode, a, b, _ = self._params
        if mode != 0 or float(a[0]) != float(a[1]):
            return None
        kh = float(a[0]) / float(b)
        return kh, float(a[2]) / float(b) - kh

    def packed_axis(self, d_Jg, ncomp=3, scale=1.0):
        """Axis form u = sqrt(scale w3 Jg[gid]) e_3 (3, nloc), or (ncomp=1, isotropic case) s = scale w3 Jg[gid]
        (1, nloc), for the plane kernel (hv_viscous_axis); not cached (the plan keeps only its
        tile-ordered copy)."""
        torch = torch_mod()
        dev = self.mesh.device()
        U = torch.empty((ncomp, dev.nloc), dtype=torch.float64, device="cuda")
        _lib.check(_lib.lib().hv_viscous_axis(dev.N, self.mets.d_grad.data_ptr(), dev.nelem, dev.w3.data_ptr(),
                                              d_Jg.data_ptr(), dev.gid32.data_ptr(), ncomp, float(scale),
                                              U.data_ptr(), _lib.stream_handle()))
        return U

    def packed(self, d_Jg):
        """W = w3 Jg[gid] G_nu, 6 components (component-major) for this Jg."""
        key = d_Jg.data_ptr()
        if key not in self._packed:
            torch = torch_mod()
            dev = self.mesh.device()
            W = torch.empty((6, dev.nloc), dtype=torch.float64, device="cuda")
            self._run(d_Jg=d_Jg, W=W)
            self._packed = {key: (W, d_Jg)}   # keep one packing alive
        return self._packed[key][0]


def build_viscous_metric(mesh, mets, cfg, dt=None):
    """Assemble G_nu from the metric-tensor eigendecomposition (hyperdiff.py:62-81).

    The scalar prefactors are evaluated on the host exactly as the reference
    does ((c**(1/alpha))*4.0 and N**2 * dt**(1/alpha)); the per-node work
    (G, eigensolve, nu, G_nu, packing) runs on the device and raises
    ValueError on a non-positive eigenvalue like the reference.
    """
    mode = _MODES[cfg.mode]
    a = np.zeros(3)
    b = 0.0
    nu = np.zeros(3)
    if cfg.mode == "scaled":
        if dt is None or dt <= 0:
            raise ValueError("scaled viscosities need dt > 0")
        N = max(mesh.cfg.degree_xi, mesh.cfg.degree_eta, mesh.cfg.degree_zeta)
        a = (np.asarray(cfg.c, dtype=float) ** (1.0 / cfg.alpha)) * 4.0
        b = N**2 * dt ** (1.0 / cfg.alpha)
    elif cfg.mode == "constant":
        nu = np.asarray(cfg.nu, dtype=float)
    else:
        nu = np.array([cfg.nu_h, cfg.nu_h, cfg.nu_v], dtype=float)
    vm = ViscousMetric(mesh, mets, cfg, (mode, a, b, nu))
    vm._run()  # validates eigenvalues (ValueError on degenerate elements)
    return vm


def _as_device(x):
    """(device tensor, was_numpy)."""
    torch = torch_mod()
    if isinstance(x, np.ndarray):
        return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).to("cuda"), True
    if not (x.is_cuda and x.dtype == torch.float64):
        raise ValueError("device inputs must be float64 CUDA tensors")
    return x.contiguous(), False


# Small meshes (configs 1 and 2) are launch-bound: an op is 2-4 kernels of 10-40 us each, about the
# cost of the Python / ctypes call that enqueues them.  The second time an op is asked for with the same
# plan and the same buffers it is captured into a CUDA graph, and replayed from then on.  A graph
# depends only on pointers (the caller's arrays and the plan's own buffers, kept alive by ``ops``), so
# a key hit is always valid while ``ops`` lives; HV_GRAPH=0 disables, HV_GRAPH_MAX is the node bound.
_GRAPHS = OrderedDict()
_GRAPH_CAP = 16


def _run_graphed(ops, key, launch):
    torch = torch_mod()
    if (ops.mesh.nglobal > int(os.environ.get("HV_GRAPH_MAX", 1 << 20)) or os.environ.get("HV_GRAPH", "1") == "0"
            or torch.cuda.is_current_stream_capturing()):
        launch()
        return
    key = (id(ops),) + key
    ent = _GRAPHS.get(key)
    if ent is not None and ent[0]() is not ops:      # a dead EulerOps whose id was reused
        ent = None
    if ent is None:
        launch()
        _GRAPHS[key] = (weakref.ref(ops), None)
        while len(_GRAPHS) > _GRAPH_CAP:
            _GRAPHS.popitem(last=False)
        return
    _GRAPHS.move_to_end(key)
    g = ent[1]
    if g is None:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            launch()
        _GRAPHS[key] = (ent[0], g)
    g.replay()


def laplacian_apply(field_g, viscous, ops):
    """M^-1 DSS(-L_nu q), one field (hyperdiff.py:84-94)."""
    torch = torch_mod()
    q, host = _as_device(field_g)
    if q.dim() != 1:
        raise ValueError("laplacian_apply takes one (nglobal,) field")
    plan = ops.lap_plan(viscous)
    out = torch.empty_like(q)
    qf = (C.c_int32 * 1)(0)
    _run_graphed(ops, ("lap1", id(plan), q.data_ptr(), out.data_ptr()), lambda: _lib.check(
        _lib.lib().hv_laplacian(C.byref(plan), q.data_ptr(), 1, 1, qf, out.data_ptr(), 1, qf, 1.0,
                                _lib.stream_handle())))
    return out.cpu().numpy() if host else out


def laplacian_apply_fields(q, viscous, ops, fields):
    """Several columns of an (nglobal, k) array in one fused pass (extension)."""
    torch = torch_mod()
    qd, host = _as_device(q)
    plan = ops.lap_plan(viscous)
    # every column written by the pass: no need to zero the output first
    full = qd.dim() == 2 and sorted(fields) == list(range(qd.shape[1]))
    out = torch.empty_like(qd) if full else torch.zeros_like(qd)
    fl = (C.c_int32 * len(fields))(*fields)
    _run_graphed(ops, ("lapf", id(plan), qd.data_ptr(), out.data_ptr(), qd.shape[1], tuple(fields), full),
                 lambda: _lib.check(_lib.lib().hv_laplacian(
                     C.byref(plan), qd.data_ptr(), qd.shape[1], len(fields), fl, out.data_ptr(), qd.shape[1], fl,
                     1.0, _lib.stream_handle())))
    return out.cpu().numpy() if host else out


def hyperdiffusion_apply(state, cfg, viscous, ops, out=None, accumulate=False):
    """(-1)^(alpha+1) L^alpha on cfg.variables, zero elsewhere (hyperdiff.py:97-106).

    ``state`` is a StateField (numpy or CUDA data).  With CUDA data an
    ``out`` tensor of the same shape may be supplied to avoid an allocation;
    with ``accumulate=True`` the result is added to ``out`` (rhs_horizontal).
    """
    torch = torch_mod()
    data = state.data if hasattr(state, "data") else state
    q, host = _as_device(data)
    plan = ops.lap_plan(viscous)
    if out is None:
        out = torch.empty_like(q)
    vars_ = (C.c_int32 * len(cfg.variables))(*cfg.variables)
    _run_graphed(ops, ("hnu", id(plan), q.data_ptr(), q.shape[1], out.data_ptr(), out.shape[1], tuple(cfg.variables),
                       cfg.alpha, bool(accumulate)),
                 lambda: _lib.check(_lib.lib().hv_hyperdiffusion(
                     C.byref(plan), q.data_ptr(), q.shape[1], len(cfg.variables), vars_, cfg.alpha, out.data_ptr(),
                     out.shape[1], int(bool(accumulate)), _lib.stream_handle())))
    return out.cpu().numpy() if host else out
