"""Element gather / DSS / derivatives / lumped mass on the device (mirror of assembly.py:6-64).

These are the reference primitives the metrics and tests use; the hot
operators fuse them inside single kernels instead of calling them.  numpy
inputs are copied to the device and results copied back; CUDA tensors stay
on the device.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .device import torch_mod

__all__ = ["weights3", "gather", "dss", "elem_deriv", "weak_deriv_acc", "GlobalMass"]


def weights3(mesh):
    """Tensor-product weights (wx*wy)*wz (assembly.py:6-9); host constant."""
    bx, be, bz = mesh.bases
    return bx.weights[:, None, None] * be.weights[None, :, None] * bz.weights[None, None, :]


def gather(mesh, field_g):
    """field_g[gid] (assembly.py:12-14)."""
    if isinstance(field_g, np.ndarray):
        return field_g[mesh.gid]
    return mesh.device().gather(field_g)


def dss(mesh, field_e):
    """Direct-stiffness summation in flat element order (assembly.py:17-26).

    Runs ``hv_dss_csr`` (sequential per-node sums == np.add.at bit for bit).
    """
    torch = torch_mod()
    host = isinstance(field_e, np.ndarray)
    fe = torch.from_numpy(np.ascontiguousarray(field_e, dtype=np.float64)).cuda() if host else field_e.contiguous()
    dev = mesh.device()
    extra = tuple(fe.shape[4:])
    k = int(np.prod(extra)) if extra else 1
    # component-major copy so each component is a contiguous element field
    fe_c = fe.reshape(dev.nloc, k).t().contiguous()
    out = torch.empty((dev.nglobal, k), dtype=torch.float64, device="cuda")
    _lib.check(_lib.lib().hv_dss_csr(fe_c.data_ptr(), k, dev.nloc, dev.off.data_ptr(), dev.idx.data_ptr(),
                                     dev.nglobal, out.data_ptr(), _lib.stream_handle()))
    out = out.reshape((dev.nglobal,) + extra)
    return out.cpu().numpy() if host else out


def _deriv(mesh, f, axis, weak):
    torch = torch_mod()
    if axis not in (0, 1, 2):
        raise ValueError("axis must be 0, 1 or 2")
    host = isinstance(f, np.ndarray)
    fe = torch.from_numpy(np.ascontiguousarray(f, dtype=np.float64)).cuda() if host else f.contiguous()
    dev = mesh.device()
    if tuple(fe.shape) != (dev.nelem, dev.n, dev.n, dev.n):
        raise ValueError("element data must be (nelem, n, n, n)")
    out = torch.empty_like(fe)
    _lib.check(_lib.lib().hv_elem_deriv(dev.N, dev.D.ctypes.data, dev.w3.data_ptr(), dev.nelem, fe.data_ptr(),
                                        axis, int(weak), out.data_ptr(), _lib.stream_handle()))
    return out.cpu().numpy() if host else out


def elem_deriv(mesh, f, axis):
    """Reference-coordinate derivative along one axis: sum_a D[i, a] f_a (assembly.py:29-36)."""
    return _deriv(mesh, f, axis, False)


def weak_deriv_acc(mesh, f, axis):
    """Weak-form accumulator -sum_a D[a, i] (w3 f)_a (assembly.py:39-51)."""
    return _deriv(mesh, f, axis, True)


class GlobalMass:
    """Diagonal mass DSS(w3 J_elem) and its inverse (assembly.py:54-64).

    ``J_elem`` may be a MetricTerms' device tensor or a numpy array.
    """

    def __init__(self, mesh, J_elem):
        torch = torch_mod()
        dev = mesh.device()
        dJ = J_elem if hasattr(J_elem, "data_ptr") else torch.from_numpy(
            np.ascontiguousarray(J_elem, dtype=np.float64)).cuda()
        self.d_M = torch.empty(dev.nglobal, dtype=torch.float64, device="cuda")
        self.d_Minv = torch.empty_like(self.d_M)
        _lib.check(_lib.lib().hv_mass_and_projection(dev.N, dev.w3.data_ptr(), dJ.data_ptr(), None, dev.nelem,
                                                     dev.off.data_ptr(), dev.idx.data_ptr(), dev.nglobal,
                                                     self.d_M.data_ptr(), self.d_Minv.data_ptr(), None, None,
                                                     _lib.stream_handle()))
        self._h = {}

    @property
    def M(self):
        if "M" not in self._h:
            self._h["M"] = self.d_M.cpu().numpy()
        return self._h["M"]

    @property
    def Minv(self):
        if "Minv" not in self._h:
            self._h["Minv"] = self.d_Minv.cpu().numpy()
        return self._h["Minv"]

    def volume(self):
        return float(self.d_M.sum().item())
