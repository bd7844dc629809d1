"""Batched band LU / solve for the LHEVI column systems on the device.

Mirrors the reference's ``hevicore.linalg`` batch API (linalg.py:112-194):
``banded_lu_factor_batch(data, kl, ku) -> (ipiv, flops)`` factors in place,
``banded_solve_batch(data, ipiv, kl, ku, b) -> (x, flops)``; the data are in
LAPACK band layout ``(nbatch, 2*kl+ku+1, M)``.  Host numpy inputs are copied to
the device and the results copied back (the reference's call signature); device
tensors stay on the device.  Kernels: csrc/column.cu.
"""

from __future__ import annotations

import functools

import numpy as np

from . import _lib
from .device import torch_mod

__all__ = ["SingularMatrixError", "band_rows", "half_bandwidth", "banded_lu_factor_batch", "banded_solve_batch"]


class SingularMatrixError(ArithmeticError):
    """Zero pivot (linalg.py SingularMatrixError): column ``j`` of system ``batch``."""

    def __init__(self, j, batch=None):
        self.j, self.batch = j, batch
        super().__init__(f"zero pivot in column {j}" + ("" if batch is None else f" of system {batch}"))


def band_rows(n_var, N_zeta):
    """Assembled band row count 3 n_var (N_zeta + 1) - 2 (linalg.py:79-81)."""
    return 3 * n_var * (N_zeta + 1) - 2


def half_bandwidth(n_var, N_zeta):
    """kl = ku = n_var (N_zeta + 1) - 1 (linalg.py:84-86)."""
    return n_var * (N_zeta + 1) - 1


@functools.lru_cache(maxsize=64)
def _factor_flops(M, kl, ku):
    f = 0
    for j in range(M):
        lm = min(kl, M - 1 - j)
        nc = min(M - 1, j + ku + kl) - j
        if lm > 0 and nc > 0:
            f += 2 * lm * nc + lm
    return f


@functools.lru_cache(maxsize=64)
def _solve_flops(M, kl, ku):
    f = sum(2 * min(kl, M - 1 - j) for j in range(M - 1))
    f += sum(2 * (min(M - 1, i + ku + kl) - i) + 1 for i in range(M))
    return f


def _dev(a, dtype):
    torch = torch_mod()
    if torch.is_tensor(a):
        if not a.is_cuda or a.dtype != dtype or not a.is_contiguous():
            raise ValueError("device arrays must be contiguous CUDA tensors of the right dtype")
        return a, False
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64 if dtype == torch.float64 else np.int32)).cuda(), True


def banded_lu_factor_batch(data, kl, ku):
    """Factor the batch in place; returns (ipiv (nbatch, M) int64, multiply-add count per system)."""
    torch = torch_mod()
    nb, rows, M = data.shape
    if rows != 2 * kl + ku + 1:
        raise ValueError("band storage has wrong row count")
    d, host = _dev(data, torch.float64)
    ipiv = torch.empty((nb, M), dtype=torch.int32, device="cuda")
    info = torch.empty(nb, dtype=torch.int32, device="cuda")
    _lib.check(_lib.lib().hv_band_lu_factor(d.data_ptr(), nb, kl, ku, M, ipiv.data_ptr(), info.data_ptr(),
                                            _lib.stream_handle()))
    bad = torch.nonzero(info).flatten()
    if bad.numel():
        b = int(bad[0])
        raise SingularMatrixError(int(info[b]) - 1, batch=b if nb > 1 else None)
    if host:
        data[...] = d.cpu().numpy()
        return ipiv.cpu().numpy().astype(np.int64), _factor_flops(M, kl, ku)
    return ipiv, _factor_flops(M, kl, ku)


def banded_solve_batch(data, ipiv, kl, ku, b):
    """Solve the factored systems for right-hand sides b (nbatch, M); returns (x, flops)."""
    torch = torch_mod()
    nb, rows, M = data.shape
    d, host = _dev(data, torch.float64)
    if torch.is_tensor(ipiv):
        ip = ipiv.to(torch.int32).contiguous()
    else:
        ip = torch.from_numpy(np.ascontiguousarray(ipiv, dtype=np.int32)).cuda()
    if torch.is_tensor(b):
        x = b.to(torch.float64).clone().contiguous()
    else:
        x = torch.from_numpy(np.array(b, dtype=np.float64, copy=True)).cuda()
    if tuple(x.shape) != (nb, M):
        raise ValueError("right-hand sides must be (nbatch, M)")
    _lib.check(_lib.lib().hv_band_solve(d.data_ptr(), ip.data_ptr(), nb, kl, ku, M, x.data_ptr(),
                                        _lib.stream_handle()))
    flops = _solve_flops(M, kl, ku)
    return (x.cpu().numpy() if (host and not torch.is_tensor(b)) else x), flops
