"""LHEVI time stepping on the device.

Mirrors the reference's ``hevi.LheviState`` / ``solve_stage_lhevi`` /
``step_lhevi`` (hevi.py:225-362) on device tensors: the explicit stage sums of
S = H (+ H_nu) + V, one cached column-system solve per implicit stage
(``linalg.banded_solve_batch`` on the factored ``EulerOps.column_jacobian``
band), all on one CUDA stream with no host round trips.  ``LheviGraph``
captures a whole step in a CUDA graph and replays it (the factorisation is
rebuilt eagerly, in place, when ``LheviState.needs_rebuild`` says so).

The IMEX tableau is any object with the ``ark.ButcherPair`` fields
(A, b, A_im, b_im as arrays); the tableau registry itself stays with the
reference (out of scope).
"""

from __future__ import annotations

import numpy as np

from . import linalg
from .device import torch_mod

__all__ = ["LheviState", "solve_stage_lhevi", "step_lhevi", "LheviGraph", "StageSolveError"]


class StageSolveError(RuntimeError):
    pass


def _gamma(tab):
    return float(np.asarray(tab.A_im)[-1, -1])


class LheviState:
    """Cached factored column Jacobian (hevi.py:225-264): mode "PS" relinearises about
    the newest state every ``update_interval`` steps, "RS" keeps ``reference``."""

    def __init__(self, update_interval=5, mode="PS", reference=None):
        if mode not in ("PS", "RS"):
            raise ValueError("mode must be PS or RS")
        if update_interval < 1:
            raise ValueError("update interval must be >= 1")
        self.K = int(update_interval)
        self.mode = mode
        self.reference = reference
        self.band = None
        self.ipiv = None
        self.lam = None
        self.age = 0

    def needs_rebuild(self, lam):
        if self.band is None or self.lam is None:
            return True
        if abs(lam - self.lam) > 1e-14 * max(abs(lam), 1.0):
            return True
        return self.mode == "PS" and self.age >= self.K

    def rebuild(self, vop, qcol, lam, counters=None):
        ref = self.reference if self.mode == "RS" else qcol
        if ref is None:
            raise StageSolveError("LHEVI-RS needs a reference state")
        band = vop.column_jacobian(ref, lam)
        # factor the fresh band first: on SingularMatrixError the cached factorisation, ipiv and lam stay
        # intact (the reference assigns its cache only after a successful factorisation, hevi.py:254-262)
        ipiv, _ = linalg.banded_lu_factor_batch(band, vop.kl, vop.ku)
        if self.band is not None and tuple(self.band.shape) == tuple(band.shape):
            self.band.copy_(band)          # in place: captured graphs keep pointing at it
        else:
            self.band = band
        if self.ipiv is not None and tuple(self.ipiv.shape) == tuple(ipiv.shape):
            self.ipiv.copy_(ipiv)
        else:
            self.ipiv = ipiv
        self.lam, self.age = lam, 0
        if counters is not None:
            counters.factorizations += vop.ncol


def solve_stage_lhevi(lstate, vop, qhat_col, counters=None):
    """Backsolve the cached (I - lam L) system for one implicit stage (hevi.py:267-276)."""
    if lstate.band is None:
        raise StageSolveError("LHEVI cache empty; rebuild before solving")
    x, _ = linalg.banded_solve_batch(lstate.band, lstate.ipiv, vop.kl, vop.ku, qhat_col.reshape(vop.ncol, -1))
    if counters is not None:
        counters.backsolves += vop.ncol
    return x.reshape(qhat_col.shape)


class _Cols:
    def __init__(self, mesh):
        torch = torch_mod()
        self.idx = torch.from_numpy(np.ascontiguousarray(mesh.col_gid, dtype=np.int64)).cuda()

    def to_cols(self, qg):
        return qg[self.idx]

    def to_global(self, qcol, out):
        out[self.idx] = qcol
        return out


def _cols(ops):
    if "lhevi_cols" not in ops._h:
        ops._h["lhevi_cols"] = _Cols(ops.mesh)
    return ops._h["lhevi_cols"]


def _S(ops, q, with_h, out):
    from .state import StateField

    st = StateField(ops.set_name, q)
    ops.rhs_horizontal(st, with_hyperdiff=with_h, out=out)
    ops.rhs_vertical(st, out=out, accumulate=True)
    return out


def _step_body(ops, tab, qg, dt, lstate, counters=None, hyper_final_only=False):
    torch = torch_mod()
    cols = _cols(ops)
    A, Aim, b = np.asarray(tab.A), np.asarray(tab.A_im), np.asarray(tab.b)
    gam = _gamma(tab)
    s = len(b)

    def S(q, i):
        if counters is not None:
            counters.rhs_horizontal += 1
            counters.rhs_vertical += 1
        return _S(ops, q, (not hyper_final_only) or (i == s - 1), torch.empty_like(q))

    Q = [qg]
    Sv = [S(qg, 0)]
    for i in range(1, s):
        qE = qg.clone()
        for j in range(i):
            if A[i, j] != 0.0:
                qE.add_(Sv[j] * (dt * A[i, j]))
        corr = torch.zeros_like(qg)
        for j in range(i):
            coef = (Aim[i, j] - A[i, j]) / gam
            if coef != 0.0:
                corr.add_(Q[j] * coef)
        qhat = qE + corr
        x = solve_stage_lhevi(lstate, ops, cols.to_cols(qhat), counters=counters)
        qtt = cols.to_global(x, torch.empty_like(qg))
        Qi = qtt - corr
        Q.append(Qi)
        Sv.append(S(Qi, i))
        if counters is not None:
            counters.stages += 1
    q1 = qg.clone()
    for i in range(s):
        if b[i] != 0.0:
            q1.add_(Sv[i] * (dt * b[i]))
    return q1


def step_lhevi(ops, tab, qg, dt, lstate, counters=None, hyper_final_only=False):
    """One LHEVI step (hevi.py:317-362) on the device; qg (nglobal, 5) float64 (numpy in,
    numpy out; CUDA tensor in, CUDA tensor out)."""
    from .hyperdiff import _as_device

    q, host = _as_device(qg)
    lam = _gamma(tab) * dt
    if lstate.needs_rebuild(lam):
        lstate.rebuild(ops, _cols(ops).to_cols(q) if lstate.mode == "PS" else lstate.reference, lam,
                       counters=counters)
    q1 = _step_body(ops, tab, q, dt, lstate, counters, hyper_final_only)
    lstate.age += 1
    return q1.cpu().numpy() if host else q1


class LheviGraph:
    """A whole LHEVI step captured once in a CUDA graph and replayed per call.

    ``step(q)`` copies q into the graph's input buffer, rebuilds the factorisation
    eagerly (in place) when the cache is stale, replays the graph and returns the
    graph's output buffer (overwritten by the next call)."""

    def __init__(self, ops, tab, dt, lstate, q_example, hyper_final_only=False):
        torch = torch_mod()
        self.ops, self.tab, self.dt, self.lstate = ops, tab, dt, lstate
        self.hfo = hyper_final_only
        self.lam = _gamma(tab) * dt
        self.q_in = q_example.detach().clone()
        if lstate.needs_rebuild(self.lam):
            lstate.rebuild(ops, _cols(ops).to_cols(self.q_in), self.lam)
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):      # warm-up (plans, workspaces) outside the capture
            _step_body(ops, tab, self.q_in, dt, lstate, None, self.hfo)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.q_out = _step_body(ops, tab, self.q_in, dt, lstate, None, self.hfo)

    def step(self, q):
        if q.data_ptr() != self.q_in.data_ptr():
            self.q_in.copy_(q)
        if self.lstate.needs_rebuild(self.lam):
            self.lstate.rebuild(self.ops, _cols(self.ops).to_cols(self.q_in), self.lam)
        self.graph.replay()
        self.lstate.age += 1
        return self.q_out
