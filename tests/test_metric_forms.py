"""Compact forms of the Laplacian metric (CPU checks of the algebra the plane kernel relies on).

In scaled mode (reference hyperdiff.py:71-80) k_m = nu_m * vals_m = a_m / b up to an ulp, so
G_nu = sum_m k_m e_m e_m^T.  With c_1 == c_2 (every BASELINE config) W = w3 Jg G_nu equals
kh |u|^2 I + kd u u^T with u = sqrt(w3 Jg) e_3 (axis form, 3 doubles per node); with
c_1 == c_2 == c_3 it is kh w3 Jg I (isotropic form, 1 double).  DESIGN.md §4.2.
"""

from __future__ import annotations

import numpy as np
import pytest

from paper_2311_11425_b200 import hyperdiff


def _params(cfg, N, dt):
    """(mode, a, b, nu) exactly as build_viscous_metric forms them (hyperdiff.py:71-72)."""
    if cfg.mode == "scaled":
        a = (np.asarray(cfg.c, dtype=float) ** (1.0 / cfg.alpha)) * 4.0
        return (0, a, N**2 * dt ** (1.0 / cfg.alpha), np.zeros(3))
    nu = np.asarray(cfg.nu, dtype=float) if cfg.mode == "constant" else np.array([cfg.nu_h, cfg.nu_h, cfg.nu_v])
    return (1 if cfg.mode == "constant" else 2, np.zeros(3), 0.0, nu)


@pytest.mark.parametrize("kw,expect", [
    (dict(alpha=2, c=(0.05, 0.05, 0.0)), "axis"),        # configs 2 and 5
    (dict(alpha=2, c=(0.1, 0.1, 0.01)), "axis"),         # config 3
    (dict(alpha=2, c=(0.02, 0.02, 0.02)), "iso"),        # config 4
    (dict(alpha=1, c=(1.0, 1.0, 1.0)), "iso"),           # config 1
    (dict(alpha=2, c=(0.05, 0.04, 0.0)), None),          # c_1 != c_2: 6 components
    (dict(alpha=2, mode="constant", nu=(3e3, 3e3, 1e2)), None),
    (dict(alpha=1, mode="anisotropic", nu_h=5e2, nu_v=3.0), None),
])
def test_axis_form_selection(kw, expect):
    cfg = hyperdiff.HyperDiffConfig(**kw)
    vm = hyperdiff.ViscousMetric(None, None, cfg, _params(cfg, 4, 0.5))
    ax = vm.axis_form()
    if expect is None:
        assert ax is None
        return
    kh, kd = ax
    a, b = vm._params[1], vm._params[2]
    assert kh == a[0] / b and kd == a[2] / b - kh
    assert (kd == 0.0) == (expect == "iso")


@pytest.mark.parametrize("c", [(0.05, 0.05, 0.0), (0.1, 0.1, 0.01), (0.02, 0.02, 0.02)])
def test_compact_forms_reproduce_six_components(c):
    """W d of the compact forms equals the reference-formula W d (G_nu = sum_m (nu_m vals_m) e_m e_m^T with
    the scaled nu_m, reference order) on random thin / curved metrics, to rounding."""
    rng = np.random.default_rng(0)
    alpha, N, dt = 2, 4, 0.5
    a = (np.asarray(c) ** (1.0 / alpha)) * 4.0
    b = N**2 * dt ** (1.0 / alpha)
    kh, kd = a[0] / b, a[2] / b - a[0] / b
    for _ in range(200):
        grad = rng.standard_normal((3, 3)) * np.array([1.0, 1.0, 10.0])[:, None]   # thin element: large grad zeta
        G = grad @ grad.T
        vals, vecs = np.linalg.eigh(G)
        lam = 1.0 / vals
        nu = (np.asarray(c) ** (1.0 / alpha)) * 4.0 * lam / (N**2 * dt ** (1.0 / alpha))   # hyperdiff.py:71-72
        Gnu = (vecs * (nu * vals)) @ vecs.T                                              # hyperdiff.py:80
        s = rng.uniform(0.1, 10.0)                                                        # w3 * Jg
        d = rng.standard_normal(3)
        ref = (s * Gnu) @ d
        u = np.sqrt(s) * vecs[:, 2]
        axis = kh * (u @ u) * d + kd * u * (u @ d)
        assert np.linalg.norm(axis - ref) <= 1e-14 * np.linalg.norm(ref) * 10
        if kd == 0.0:
            iso = (kh * s) * d
            assert np.linalg.norm(iso - ref) <= 1e-14 * np.linalg.norm(ref) * 10
