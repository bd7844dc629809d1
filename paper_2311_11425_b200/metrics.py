"""Metric terms on the device: curl-invariant / cross-product metrics and the
column L2 projection (mirror of reference metrics.py:24-142).

``curl_invariant_metrics`` / ``cross_product_metrics`` run the sm_100a
``hv_metric_terms`` kernel, whose arithmetic is rounding-faithful to the
reference's numpy einsum order (bit-exact ``J_elem`` / ``grad_elem``).
``project_metrics_to_columns`` runs ``hv_mass_and_projection`` (sequential
flat-order DSS, bit-exact with ``np.add.at``).  Results live on the device;
the reference-shaped numpy attributes are materialised lazily on access.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .device import torch_mod

__all__ = ["MetricTerms", "curl_invariant_metrics", "cross_product_metrics", "build_metrics",
           "project_metrics_to_columns", "duality_error", "constant_field_divergence"]

_SCHEMES = {"curl-invariant": 0, "cross-product": 1}


class MetricTerms:
    """Per-element metric data plus gridpoint J and grad zeta (metrics.py:24-46).

    Device tensors: ``d_J`` (nelem,n,n,n), ``d_grad`` (nelem,3,3,n,n,n),
    ``d_Jg`` (nglobal,), ``d_gz`` (nglobal,3).  Host views: ``J_elem``,
    ``grad_elem``, ``dxdxi``, ``Jg``, ``gradzeta_g``.
    """

    def __init__(self, scheme, mesh, d_J, d_grad, d_Jg, d_gz, projected=False):
        self.scheme = scheme
        self.mesh = mesh
        self.projected = projected
        self.d_J, self.d_grad, self.d_Jg, self.d_gz = d_J, d_grad, d_Jg, d_gz
        self._host = {}

    def _h(self, key, t):
        if key not in self._host:
            self._host[key] = t.cpu().numpy()
        return self._host[key]

    @property
    def J_elem(self):
        return self._h("J", self.d_J)

    @property
    def grad_elem(self):
        return self._h("grad", self.d_grad)

    @property
    def Jg(self):
        return self._h("Jg", self.d_Jg)

    @property
    def gradzeta_g(self):
        return self._h("gz", self.d_gz)

    @property
    def dxdxi(self):
        if "dx" not in self._host:
            torch = torch_mod()
            dev = self.mesh.device()
            dx = torch.empty_like(self.d_grad)
            J = torch.empty_like(self.d_J)
            g = torch.empty_like(self.d_grad)
            _lib.check(_lib.lib().hv_metric_terms(_SCHEMES[self.scheme], dev.N, dev.D.ctypes.data,
                                                  dev.coords.data_ptr(), dev.nelem, dx.data_ptr(), J.data_ptr(),
                                                  g.data_ptr(), _lib.stream_handle()))
            self._host["dx"] = dx.cpu().numpy()
        return self._host["dx"]


def _element_metrics(mesh, scheme):
    torch = torch_mod()
    dev = mesh.device()
    n = dev.n
    J = torch.empty((dev.nelem, n, n, n), dtype=torch.float64, device="cuda")
    grad = torch.empty((dev.nelem, 3, 3, n, n, n), dtype=torch.float64, device="cuda")
    _lib.check(_lib.lib().hv_metric_terms(_SCHEMES[scheme], dev.N, dev.D.ctypes.data, dev.coords.data_ptr(),
                                          dev.nelem, None, J.data_ptr(), grad.data_ptr(), _lib.stream_handle()))
    # naive gridpoint reduction: last writer in element-loop order (metrics.py:40-46)
    Jg = dev.last_writer(J)
    gz = torch.stack([dev.last_writer(grad[:, 2, c]) for c in range(3)], dim=1).contiguous()
    return MetricTerms(scheme, mesh, J, grad, Jg, gz)


def cross_product_metrics(mesh):
    """grad xi^i = (dx/dxi^j x dx/dxi^k)/J (metrics.py:79-88)."""
    return _element_metrics(mesh, "cross-product")


def curl_invariant_metrics(mesh):
    """Curl-invariant grad xi^i (metrics.py:91-110)."""
    return _element_metrics(mesh, "curl-invariant")


def build_metrics(mesh, scheme):
    if scheme not in _SCHEMES:
        raise ValueError(f"unknown metric scheme {scheme!r}")
    return _element_metrics(mesh, scheme)


def project_metrics_to_columns(metrics, mesh):
    """Mass-weighted L2 projection of J and grad zeta (metrics.py:121-142)."""
    torch = torch_mod()
    dev = mesh.device()
    ng = dev.nglobal
    M = torch.empty(ng, dtype=torch.float64, device="cuda")
    Minv = torch.empty_like(M)
    Jg = torch.empty_like(M)
    gz = torch.empty((ng, 3), dtype=torch.float64, device="cuda")
    _lib.check(_lib.lib().hv_mass_and_projection(dev.N, dev.w3.data_ptr(), metrics.d_J.data_ptr(),
                                                 metrics.d_grad.data_ptr(), dev.nelem, dev.off.data_ptr(),
                                                 dev.idx.data_ptr(), ng, M.data_ptr(), Minv.data_ptr(),
                                                 Jg.data_ptr(), gz.data_ptr(), _lib.stream_handle()))
    out = MetricTerms(metrics.scheme, mesh, metrics.d_J, metrics.d_grad, Jg, gz, projected=True)
    out._mass_cache = (M, Minv)
    return out


# ----------------------------------------------------------- diagnostics (host)
def duality_error(mesh, metrics):
    """max |grad xi^i . dx/dxi^j - delta_ij| (metrics.py:145-154); host diagnostic."""
    err = 0.0
    g, dx = metrics.grad_elem, metrics.dxdxi
    for i in range(3):
        for j in range(3):
            dot = np.einsum("ec...,ec...->e...", g[:, i], dx[:, :, j])
            err = max(err, float(np.max(np.abs(dot - (1.0 if i == j else 0.0)))))
    return err


def constant_field_divergence(mesh, metrics, F):
    """(1/J) sum_m D^m (J F.grad xi^m) (metrics.py:157-170); host diagnostic."""
    F = np.asarray(F, dtype=float)
    D = mesh.bases[0].diff_matrix
    subs = ("ia,eajk->eijk", "ja,eiak->eijk", "ka,eija->eijk")
    J = metrics.J_elem
    div = np.zeros((mesh.nelem,) + tuple(mesh.shape))
    for m in range(3):
        flux = J * np.einsum("c,ec...->e...", F, metrics.grad_elem[:, m])
        div += np.einsum(subs[m], mesh.bases[m].diff_matrix, flux)
    return div / J
