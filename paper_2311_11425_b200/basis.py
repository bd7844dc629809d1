"""One-dimensional Legendre-Gauss-Lobatto basis (host constants for the kernels).

Mirror of the reference ``basis`` module API (``basis.py:18-145``): the hot
path only consumes ``nodes``, ``weights`` and ``diff_matrix`` (uploaded once
into the kernels' constant tables); the remaining helpers keep the public API
a drop-in.  The construction follows the reference algorithm step for step
(Newton on (1-x^2) P_N' from Chebyshev-Lobatto guesses, barycentric D with a
negative-row-sum diagonal) so the constants are bit-identical to the
reference's, which the metric kernels' bit-exactness relies on.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from functools import lru_cache

import numpy as np

__all__ = ["Basis1D", "lobatto", "differentiate", "integrate", "cardinal_values",
           "interpolate", "flux_difference_check"]


@dataclass(frozen=True)
class Basis1D:
    """Lobatto nodes, weights and differentiation matrix of degree ``order`` (basis.py:18-30)."""

    order: int
    nodes: np.ndarray
    weights: np.ndarray
    diff_matrix: np.ndarray
    bary_weights: np.ndarray = field(repr=False, default=None)

    @property
    def npts(self):
        return self.order + 1


def _pn(n, x):
    """Legendre P_n and P_n' (three-term recurrence, endpoint closed form)."""
    x = np.asarray(x, dtype=float)
    lo = np.ones_like(x)
    if n == 0:
        return lo, np.zeros_like(x)
    hi = x.copy()
    for k in range(1, n):
        lo, hi = hi, ((2 * k + 1) * x * hi - k * lo) / (k + 1)
    edge = np.abs(np.abs(x) - 1.0) < 1e-300
    d = n * (x * hi - lo) / np.where(edge, 1.0, x**2 - 1.0)
    d = np.where(edge, np.sign(x) ** (n - 1) * n * (n + 1) / 2.0, d)
    return hi, d


@lru_cache(maxsize=None)
def _build(N):
    n = N + 1
    x = -np.cos(np.pi * np.arange(n) / N)
    if N > 1:
        inner = x[1:-1].copy()
        for _ in range(100):
            p, dp = _pn(N, inner)
            delta = ((1.0 - inner**2) * dp) / (-N * (N + 1) * p)
            inner -= delta
            if np.max(np.abs(delta)) < 1e-15:
                break
        x[1:-1] = inner
    x[0], x[-1] = -1.0, 1.0
    pN, _ = _pn(N, x)
    w = 2.0 / (N * (N + 1) * pN**2)
    gap = x[:, None] - x[None, :]
    np.fill_diagonal(gap, 1.0)
    bw = 1.0 / np.prod(gap, axis=1)
    D = np.empty((n, n))
    for i in range(n):
        h = x[i] - x
        h[i] = 1.0
        D[i, :] = (bw / bw[i]) / h
        D[i, i] = 0.0
        D[i, i] = -np.sum(D[i, :])
    for a in (x, w, D, bw):
        a.setflags(write=False)
    return x, w, D, bw


def lobatto(N):
    """Degree-N Lobatto basis with N+1 nodes (basis.py:50-88)."""
    if N < 1:
        raise ValueError("Lobatto basis needs degree N >= 1")
    x, w, D, bw = _build(int(N))
    return Basis1D(order=int(N), nodes=x, weights=w, diff_matrix=D, bary_weights=bw)


def differentiate(basis, values):
    """Derivative of the interpolant at the nodes (basis.py:91-101)."""
    values = np.asarray(values, dtype=float)
    if values.shape[-1] != basis.npts:
        raise ValueError(f"expected {basis.npts} nodal values, got {values.shape[-1]}")
    return values @ basis.diff_matrix.T


def integrate(basis, values):
    """Lobatto quadrature over [-1, 1] (basis.py:104-107)."""
    return np.asarray(values, dtype=float) @ basis.weights


def cardinal_values(basis, x):
    """Lagrange cardinal functions at points x, barycentric form (basis.py:110-124)."""
    x = np.atleast_1d(np.asarray(x, dtype=float))
    L = np.zeros((x.size, basis.npts))
    diff = x[:, None] - basis.nodes[None, :]
    exact = np.abs(diff) < 1e-14
    hit = exact.any(axis=1)
    terms = np.where(exact, 1.0, basis.bary_weights / np.where(exact, 1.0, diff))
    L[~hit] = terms[~hit] / terms[~hit].sum(axis=1, keepdims=True)
    L[hit] = exact[hit].astype(float)
    return L


def interpolate(basis, values, x):
    """Interpolant of nodal values at x (basis.py:127-129)."""
    return cardinal_values(basis, x) @ np.asarray(values, dtype=float)


def flux_difference_check(basis, p, q, tol=1e-13):
    """p_i (Dq)_i == sum_j D_ij p_i q_j (basis.py:132-145)."""
    p = np.asarray(p, dtype=float)
    q = np.asarray(q, dtype=float)
    if p.shape != q.shape:
        raise ValueError("p and q must have equal length")
    lhs = p * (basis.diff_matrix @ q)
    rhs = np.einsum("ij,i,j->i", basis.diff_matrix, p, q)
    return bool(np.max(np.abs(lhs - rhs)) <= tol)
