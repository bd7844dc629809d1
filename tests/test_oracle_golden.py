"""Pin the CPU oracle against the reference's own outputs (tests/golden/*.npz).

The oracle restates the reference algorithm operation by operation, so on
this numpy build it must reproduce the fixtures bit for bit: integer maps and
metrics by SHA-256 digest, operator outputs with np.array_equal.
"""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from cases import CASES, random_state
from conftest import golden
from oracle import hevi_oracle as O
from oracle_cases import OracleProblem


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module", params=list(CASES))
def prob(request):
    return OracleProblem(request.param), golden(request.param)


def test_basis_bitwise():
    g = golden("basis")
    for N in range(1, 9):
        x, w, D = O.lgl(N)
        assert np.array_equal(D, g[f"D{N}"]) and np.array_equal(w, g[f"w{N}"]) and np.array_equal(x, g[f"x{N}"])


def test_numbering_and_columns(prob):
    p, g = prob
    assert p.m.ng == int(g["ng"])
    assert sha(p.m.gid) == str(g["sha_gid"])
    assert sha(p.m.xg) == str(g["sha_xg"])
    assert sha(p.m.col_gid) == str(g["sha_col_gid"])
    assert sha(p.m.flux_mask) == str(g["sha_flux_mask"])


def test_metrics_bitwise(prob):
    p, g = prob
    assert sha(p.J) == str(g["sha_J"])
    assert sha(p.grad) == str(g["sha_grad"])
    assert sha(p.dxdxi) == str(g["sha_dxdxi"])
    assert sha(p.Jg0) == str(g["sha_Jg_naive"])
    assert sha(p.gz0) == str(g["sha_gz_naive"])
    assert sha(p.Jg) == str(g["sha_Jg"])
    assert sha(p.gz) == str(g["sha_gz"])
    assert sha(p.M) == str(g["sha_M"])
    _, _, gx = O.cross_metrics(p.m)
    assert sha(gx) == str(g["sha_grad_cross"])


def test_hyperdiffusion_bitwise(prob):
    p, g = prob
    assert np.array_equal(p.hyper(), g["hyper"])


def test_laplacian_bitwise(prob):
    p, g = prob
    if p.c["lap_fields"] is None:
        pytest.skip("no laplacian fixture")
    got = np.stack([p.lap(f) for f in p.c["lap_fields"]], axis=1)
    assert np.array_equal(got, g["lap"])


def test_rhs_bitwise(prob):
    p, g = prob
    for s in p.c["sets"]:
        e = p.euler(s)
        rs = random_state(p.m.ng, s)
        assert np.array_equal(e.rhs_full(rs), g[f"rhs_full_{s}"]), s
        assert np.array_equal(e.rhs_horizontal_nohd(rs), g[f"rhs_h_{s}"]), s
        assert np.array_equal(e.rhs_vertical(rs), g[f"rhs_v_{s}"]), s


def test_c4_target_bitwise(prob):
    """Config 4's quantity rhs_full(q) + hyperdiffusion_apply(q) on the case's own (near-hydrostatic)
    state, at config 4's element geometry (case c4_win)."""
    p, g = prob
    if "c4_target" not in g:
        pytest.skip("no config-4 target fixture")
    e = p.euler("2C")
    S = e.rhs_full(p.state)
    assert np.array_equal(S, g["rhs_full_state"])
    assert np.array_equal(S + p.hyper(), g["c4_target"])


def test_column_system_bitwise(prob):
    """LHEVI column Jacobian band, its pivoted band LU and the back-solve (euler.py:274-417,
    linalg.py:112-194) against the reference on the first golden columns."""
    p, g = prob
    if p.name == "c1":
        pytest.skip("no column-system fixture for c1")
    for s in p.c["sets"]:
        e = p.euler(s)
        rs = random_state(p.m.ng, s)
        band, kl, ku = O.column_jacobian(e, rs[p.m.col_gid], 0.37)
        band = np.ascontiguousarray(band[:24])
        assert sha(band) == str(g[f"jac_sha_{s}"]), s
        ipiv = O.band_lu_factor(band, kl, ku)
        assert sha(band) == str(g[f"lu_sha_{s}"]), s
        assert np.array_equal(ipiv, g[f"ipiv_{s}"]), s
        rhs = np.random.default_rng(11).standard_normal((band.shape[0], band.shape[2]))
        assert np.array_equal(O.band_solve(band, ipiv, kl, ku, rhs), g[f"solve_{s}"]), s


class _Tab:
    def __init__(self, z, name):
        for f in ("A", "b", "c", "A_im", "b_im", "c_im"):
            setattr(self, f, z[f"tab_{name}_{f}"])


def test_lhevi_step_bitwise():
    """Two LHEVI steps (ark tableaux ARK2 / ARS3) with one cached factorisation, against
    hevi.step_lhevi run by the reference (tests/golden/lhevi.npz)."""
    from cases import LHEVI, lhevi_state

    z = golden("lhevi")
    p = OracleProblem(LHEVI["case"])
    e = p.euler("2C", omega=0.0)
    # H_nu of this case at the LHEVI dt (the viscous metric depends on dt)
    hd = dict(LHEVI["hd"])
    alpha = hd.pop("alpha")
    Gnu, _, _ = O.viscous_metric(p.m, p.grad, alpha, dt=LHEVI["dt"], **hd)
    hyper = lambda q: O.hyperdiffusion(p.m, Gnu, p.Jg_e, p.Minv, q, alpha)  # noqa: E731
    q0 = lhevi_state(p.m.xg)
    for name in LHEVI["tabs"]:
        cache = O.LheviCache(LHEVI["update_interval"])
        q = q0.copy()
        for k in range(LHEVI["steps"]):
            q = O.lhevi_step(e, hyper, _Tab(z, name), q, LHEVI["dt"], cache)
            assert np.array_equal(q, z[f"step_{name}_{k}"]), (name, k, np.abs(q - z[f"step_{name}_{k}"]).max())


@pytest.mark.parametrize("cname", ["box_p_n4", "sphere_n4"])
def test_diagnostics_bitwise(cname):
    """EulerOps.diagnostics (euler.py:421-456) restated: bitwise the reference's values."""
    z = golden("diag")
    p = OracleProblem(cname)
    for s in ("2C", "2NC", "3C"):
        d = p.euler(s, omega=0.0).diagnostics(z[f"{cname}_{s}_state"])
        keys = list(z[f"{cname}_{s}_keys"])
        assert sorted(d) == keys
        assert np.array_equal(np.array([d[k] for k in keys]), z[f"{cname}_{s}_vals"]), s


def test_field_dump_bytes(tmp_path):
    """run.dump_fields format (run.py:202-211): our writer is byte-identical to the reference's;
    load_fields reads it back."""
    from product_cases import product_mesh
    from paper_2311_11425_b200 import dumps, state

    z = golden("diag")
    m = product_mesh("box_p_n4")
    q = z["box_p_n4_2C_state"]
    dumps.dump_fields(str(tmp_path / "f"), m, state.StateField("2C", q), 12.5)
    assert (tmp_path / "f.bin").read_bytes() == z["dump_bin"].tobytes()
    assert (tmp_path / "f.hdr").read_text() == str(z["dump_hdr"])
    st, hdr = dumps.load_fields(str(tmp_path / "f"))
    assert np.array_equal(st.data, q) and st.set_name == "2C" and hdr["time"] == 12.5
    assert hdr["n_z"] == m.n_z and hdr["columns"] == m.ncol


def test_state_helpers_match_reference():
    """convert_state / temperature / pressure_derivatives (state.py:104-165): the package's host
    helpers reproduce the reference's converted fixture states bit for bit."""
    from product_cases import product_mesh
    from paper_2311_11425_b200 import state

    z = golden("diag")
    m = product_mesh("box_p_n4")
    k = state.PhysConstants(omega=0.0)
    phi = k.g * m.xg[:, 2]
    q2c = state.StateField("2C", z["box_p_n4_2C_state"])
    for s in ("2NC", "3C"):
        got = state.convert_state(q2c, s, k, phi)
        assert got.set_name == s and np.array_equal(got.data, z[f"box_p_n4_{s}_state"]), s
        back = state.convert_state(got, "2C", k, phi)
        assert np.allclose(back.data, q2c.data, rtol=1e-12, atol=1e-12)
    d = state.pressure_derivatives("3C", z["box_p_n4_3C_state"], k, Phi=phi)
    assert set(d) == {"rho", "U", "V", "W", "E"}
    T = state.temperature("2C", q2c.data, k)
    assert np.allclose(T, state.pressure("2C", q2c.data, k) / (q2c.data[:, 0] * k.R))


@pytest.mark.parametrize("name", list(CASES))
def test_stored_state_is_the_generator_output(name):
    """The input state stored in each fixture is, byte for byte, what the seeded generator produces
    in this container (the fixtures' reference outputs were made from it); the GPU tests read the
    stored bytes, so host-dependent rounding of np.cos / BLAS on another host cannot perturb them."""
    from cases import case_state, make_state

    g = golden(name)
    from oracle_cases import oracle_mesh

    xg = oracle_mesh(name).xg
    regen = make_state(CASES[name], xg)
    assert sha(regen) == str(g["sha_state"]) == sha(g["state"])
    assert np.array_equal(case_state(name, xg), regen)


def test_stored_lhevi_state():
    from cases import LHEVI, lhevi_state
    from oracle_cases import oracle_mesh

    xg = oracle_mesh(LHEVI["case"]).xg
    assert np.array_equal(lhevi_state(xg, stored=False), golden("lhevi")["q0"])
