"""Parity cases shared by the golden generator, the oracle tests and the GPU tests.

Each case describes a mesh (by generator parameters), a hyper-diffusion
configuration and seeded inputs.  ``tests/golden/make_golden.py`` runs the
REFERENCE on these cases; the tests rebuild the same inputs and compare.
"""

from __future__ import annotations

import numpy as np

from paper_2311_11425_b200 import synthetic

CASES = {
    # config-1/2 generator (perturbed lattice box) at reduced size, alpha = 2
    "box_p_n4": dict(kind="lattice", nx=4, ny=3, nv=2, N=4, extents=(8000.0, 6000.0, 2000.0),
                     hd=dict(alpha=2, c=(0.05, 0.05, 0.0)), dt=0.5, state="fourier",
                     sets=("2C", "2NC", "3C"), omega=0.0, lap_fields=(1,)),
    # config 1 at full size: alpha = 1 on all five fields
    "c1": dict(kind="lattice", nx=8, ny=8, nv=4, N=4, extents=(8000.0, 8000.0, 2000.0),
               hd=dict(alpha=1, c=(1.0, 1.0, 1.0)), dt=1.0, state="normal", sets=(), omega=0.0,
               lap_fields=(0, 1, 2, 3, 4)),
    # config-3 generator (cubed sphere) at reduced size, rotation on
    "sphere_n4": dict(kind="sphere", ne=2, nv=2, N=4, radius=6.371e6, z_top=1.0e4,
                      hd=dict(alpha=2, c=(0.1, 0.1, 0.01)), dt=300.0, state="sphere",
                      sets=("2C", "2NC", "3C"), omega=7.292e-5, lap_fields=(1, 4)),
    # config-4 generator (N = 7 box, warm bubble) at reduced size
    "box_n7": dict(kind="box", ne=2, nv=2, N=7, extents=(1.0e4, 1.0e4, 1.0e4),
                   hd=dict(alpha=2, c=(0.02, 0.02, 0.02)), dt=0.1, state="bubble",
                   sets=("2C", "2NC", "3C"), omega=0.0, lap_fields=None),
    # low degrees, constant and anisotropic viscosity modes.  nu_1 == nu_2: on
    # elements with a degenerate horizontal eigenspace the reference's G_nu is
    # only basis-independent when the two horizontal viscosities agree
    # (LAPACK picks an arbitrary basis there)
    "box_p_n2_const": dict(kind="lattice", nx=3, ny=2, nv=2, N=2, extents=(3000.0, 2000.0, 1000.0),
                           hd=dict(alpha=2, mode="constant", nu=(3e3, 3e3, 1e2)), dt=1.0, state="fourier",
                           sets=("2C",), omega=0.0, lap_fields=(2,)),
    "box_p_n3_aniso": dict(kind="lattice", nx=2, ny=2, nv=3, N=3, extents=(2000.0, 2000.0, 600.0),
                           hd=dict(alpha=1, mode="anisotropic", nu_h=5e2, nu_v=3.0), dt=1.0, state="fourier",
                           sets=("2C",), omega=0.0, lap_fields=(3,)),
    # the remaining degrees: N = 1 (plane kernel, 2-node lines), N = 5 and N = 6 (line-tile kernel)
    "box_p_n1": dict(kind="lattice", nx=5, ny=3, nv=3, N=1, extents=(5000.0, 3000.0, 1500.0),
                     hd=dict(alpha=2, c=(0.05, 0.05, 0.0)), dt=0.5, state="fourier",
                     sets=("2C",), omega=0.0, lap_fields=(1,)),
    "box_p_n5": dict(kind="lattice", nx=3, ny=2, nv=2, N=5, extents=(3000.0, 2000.0, 800.0),
                     hd=dict(alpha=1, c=(0.05, 0.05, 0.01)), dt=0.5, state="fourier",
                     sets=("2NC",), omega=0.0, lap_fields=(0, 2)),
    "box_p_n6": dict(kind="lattice", nx=2, ny=3, nv=2, N=6, extents=(2000.0, 3000.0, 800.0),
                     hd=dict(alpha=2, c=(0.05, 0.05, 0.0)), dt=0.5, state="fourier",
                     sets=("3C",), omega=0.0, lap_fields=(4,)),
    # a single layer (bottom and top level in one element: carries, masks, column DSS)
    "box_p_1lay": dict(kind="lattice", nx=3, ny=2, nv=1, N=4, extents=(3000.0, 2000.0, 500.0),
                       hd=dict(alpha=2, c=(0.05, 0.05, 0.0)), dt=0.5, state="fourier",
                       sets=("2C", "3C"), omega=0.0, lap_fields=(1,)),
    # N = 7 with a single layer (Euler column sweep: no carries, both masked levels in one element)
    "box_n7_1lay": dict(kind="box", ne=2, nv=1, N=7, extents=(1.0e4, 1.0e4, 2.0e3),
                        hd=dict(alpha=2, c=(0.02, 0.02, 0.02)), dt=0.1, state="bubble",
                        sets=("2C", "2NC"), omega=0.0, lap_fields=None),
    # ragged 2x2 tiles on the sphere (3 elements per panel edge), N = 3
    "sphere_n3_ragged": dict(kind="sphere", ne=3, nv=2, N=3, radius=6.371e6, z_top=1.0e4,
                             hd=dict(alpha=2, c=(0.1, 0.1, 0.01)), dt=300.0, state="sphere",
                             sets=("2C",), omega=7.292e-5, lap_fields=(2,)),
    # N = 7 on the cubed sphere with rotation (split-plane sweep and Euler column sweep on curved panels)
    "sphere_n7": dict(kind="sphere", ne=1, nv=2, N=7, radius=6.371e6, z_top=1.0e4,
                      hd=dict(alpha=2, c=(0.1, 0.1, 0.01)), dt=300.0, state="sphere",
                      sets=("2C", "3C"), omega=7.292e-5, lap_fields=None),
    # config 4 at its OWN element geometry (156.25 x 156.25 x 625 m elements, N = 7, the c4 bubble,
    # c = 0.02, dt = 0.1): a 4 x 4 x 4 window of the 64 x 64 x 16 box around the bubble centre
    # (5, 5, 2) km, bottom at z = 0; the target quantity is S(q) + H_nu(q) on the bubble state
    "c4_win": dict(kind="window", ne=64, nv_full=16, N=7, extents=(1.0e4, 1.0e4, 1.0e4),
                   ia0=30, nx=4, ib0=30, ny=4, nv=4,
                   hd=dict(alpha=2, c=(0.02, 0.02, 0.02)), dt=0.1, state="bubble",
                   sets=("2C",), omega=0.0, lap_fields=None, c4_target=True),
}


def window_args(c):
    return (c["ne"], c["nv_full"], c["N"], c["extents"], c["ia0"], c["nx"], c["ib0"], c["ny"], c["nv"])


def make_state(case, xg):
    """Regenerate a case's seeded input state on this host (numpy transcendental functions and BLAS
    may round differently on another host: the GPU-side tests use ``case_state``)."""
    c = CASES[case] if isinstance(case, str) else case
    if c["state"] == "normal":
        return np.random.default_rng(synthetic.STATE_SEED).standard_normal((xg.shape[0], 5))
    if c["state"] == "fourier":
        return synthetic.fourier_state(xg, c["extents"])
    if c["state"] == "sphere":
        return synthetic.sphere_state(xg, c["radius"], c["z_top"])
    if c["state"] == "bubble":
        return synthetic.bubble_state_2c(xg)
    raise ValueError(c["state"])


def case_state(name, xg, c=None):
    """The input state of a case: the exact bytes stored in its golden fixture (made in the build
    container, where tests/test_oracle_golden.py checks that regeneration reproduces them bit for bit),
    so the oracle, the reference outputs and the CUDA path see identical inputs on any host.  Cases
    without a fixture (full-size runs compared against the oracle alone) regenerate it."""
    from pathlib import Path

    f = Path(__file__).resolve().parent / "golden" / f"{name}.npz"
    if c is None and f.exists():
        z = np.load(f)
        if "state" in z.files:
            return np.array(z["state"])
    return make_state(CASES[name] if c is None else c, xg)


def random_state(ng, set_name, seed=7):
    """Non-balanced positive random state (test S on such states)."""
    rng = np.random.default_rng(seed)
    q = np.empty((ng, 5))
    q[:, 0] = 1.0 + 0.2 * rng.random(ng)
    if set_name == "2NC":
        q[:, 1:4] = 10.0 * rng.standard_normal((ng, 3))
        q[:, 4] = 300.0 + 5.0 * rng.random(ng)
    elif set_name == "2C":
        q[:, 1:4] = 10.0 * rng.standard_normal((ng, 3)) * q[:, :1]
        q[:, 4] = q[:, 0] * (300.0 + 5.0 * rng.random(ng))
    else:
        q[:, 1:4] = 10.0 * rng.standard_normal((ng, 3)) * q[:, :1]
        q[:, 4] = 2.5e5 + 1e4 * rng.random(ng)
    return q


def rel_l2(a, b):
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (den if den > 0 else 1.0))


# LHEVI step parity case (hevi.step_lhevi, hevi.py:317-362): set 2C on the box_p_n4 mesh,
# warm-bubble state with seeded momenta, two steps sharing one cached factorisation
LHEVI = dict(case="box_p_n4", tabs=("ARK2", "ARS3"), dt=0.05, steps=2, update_interval=5,
             hd=dict(alpha=2, c=(1e-4, 1e-4, 0.0)))   # explicit-stable hyper-diffusion strength


def lhevi_state(xg, seed=5, stored=True):
    """LHEVI initial state: the stored fixture bytes (``stored``), else regenerated."""
    if stored:
        from pathlib import Path

        f = Path(__file__).resolve().parent / "golden" / "lhevi.npz"
        if f.exists():
            z = np.load(f)
            if "q0" in z.files:
                return np.array(z["q0"])
    from paper_2311_11425_b200.synthetic import bubble_state_2c

    q = bubble_state_2c(xg, centre=(4000.0, 3000.0, 1000.0), radius=1500.0)
    rng = np.random.default_rng(seed)
    x, y, z = xg[:, 0] / 8000.0, xg[:, 1] / 6000.0, xg[:, 2] / 2000.0
    s2 = lambda a: np.sin(2.0 * np.pi * a)  # noqa: E731
    q[:, 1] = q[:, 0] * (2.0 * s2(x) * np.cos(np.pi * y) + 0.01 * rng.standard_normal(xg.shape[0]))
    q[:, 2] = q[:, 0] * (1.5 * s2(y) * np.cos(np.pi * x) + 0.01 * rng.standard_normal(xg.shape[0]))
    q[:, 3] = q[:, 0] * (0.5 * np.sin(np.pi * z) * s2(x) + 0.01 * rng.standard_normal(xg.shape[0]))
    return q


def diag_state(m, seed=9):
    """Physical set-2C state on any mesh (box or sphere): stratified density, seeded
    momenta, potential temperature 300 K (diagnostics fixture)."""
    if m.cfg.geometry == "sphere":
        h = np.linalg.norm(m.xg, axis=1) - m.cfg.radius
    else:
        h = m.xg[:, 2]
    rng = np.random.default_rng(seed)
    rho = 1.2 * np.exp(-h / 8000.0)
    q = np.empty((m.xg.shape[0], 5))
    q[:, 0] = rho
    q[:, 1:4] = rho[:, None] * rng.normal(0.0, 3.0, (m.xg.shape[0], 3))
    q[:, 4] = rho * (300.0 + rng.uniform(0.0, 2.0, m.xg.shape[0]))
    return q
