"""Device-resident mesh data and small torch plumbing helpers.

PyTorch is used only for device memory, streams and copies; every numerical
operation on the path runs in ``libhv_b200.so``.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib


def torch_mod():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_2311_11425_b200 needs a CUDA device (B200, sm_100a); there is no CPU fallback")
    return torch


def to_dev(a, dtype=None):
    torch = torch_mod()
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.to("cuda", non_blocking=False)


class DeviceMesh:
    """int32 gid, DSS CSR map (flat order), coordinates, w3 and D on the device."""

    def __init__(self, mesh):
        torch = torch_mod()
        L = _lib.lib()
        self.mesh = mesh
        self.N = mesh.degree
        b = mesh.bases[0]
        self.n = self.N + 1
        self.nn = self.n ** 3
        self.nelem = mesh.nelem
        self.nglobal = mesh.nglobal
        self.nloc = self.nelem * self.nn
        if self.nloc >= 2**31 or self.nglobal >= 2**31:
            raise NotImplementedError("meshes beyond 2^31 local nodes per GPU need the sharded path")
        self.D = np.ascontiguousarray(b.diff_matrix, dtype=np.float64)
        wx, wy, wz = (bb.weights for bb in mesh.bases)
        self.w3_host = wx[:, None, None] * wy[None, :, None] * wz[None, None, :]
        gid = np.ascontiguousarray(mesh.gid.reshape(-1))
        off = np.empty(self.nglobal + 1, dtype=np.int64)
        idx = np.empty(self.nloc, dtype=np.int32)
        _lib.check(L.hv_build_dss_csr(gid.ctypes.data, self.nloc, self.nglobal, off.ctypes.data, idx.ctypes.data))
        self.off_host, self.idx_host = off, idx
        self.gid32 = to_dev(gid.astype(np.int32))
        self.off = to_dev(off)
        self.idx = to_dev(idx)
        self.w3 = to_dev(self.w3_host.reshape(-1))
        self._coords = None
        self.stream = torch.cuda.current_stream()

    @property
    def coords(self):
        if self._coords is None:
            self._coords = to_dev(self.mesh.coords)
        return self._coords

    def last_writer(self, elem_vals):
        """Gridpoint value of the last element copy in flat order (metrics.py:40-46)."""
        torch = torch_mod()
        last = self.idx[self.off[1:] - 1].long()
        return elem_vals.reshape(-1)[last]

    def gather(self, fg):
        """field_g[gid] (assembly.py:12-14) as a device gather."""
        return fg[self.gid32.long()].reshape((self.nelem,) + (self.n,) * 3 + tuple(fg.shape[1:]))
