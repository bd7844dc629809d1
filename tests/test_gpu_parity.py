"""GPU parity: the CUDA path (through the C-ABI) vs the CPU oracle and the reference goldens.

Bars (BASELINE.json north_star): integer maps bit-exact; metric setup
bit-exact (rounding-faithful kernel); H_nu / Laplacian / S within 1e-12
relative L2 in fp64.
"""

from __future__ import annotations

import numpy as np
import pytest

from cases import CASES, rel_l2
from conftest import golden

pytestmark = pytest.mark.gpu


def sha(a):
    import hashlib

    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()

TOL = 1e-12


def xtol(p):
    """Agreement bar between two of OUR kernel paths (different summation orders).  1e-14, except
    for config 4's stratified bubble state (state "bubble", N = 7: the c4 window and box_n7), where
    a reordering of the same sums -- e.g. the plane kernel's even-odd line contractions against the
    element kernel's plain ones -- moves H_nu by 1-5e-14 (kernel-internal re-ordering
    1.2-1.6e-13 on c4-like elements); parity with the reference stays at TOL."""
    return 2e-13 if (p.c["kind"] == "window" or p.c.get("state") == "bubble") else 1e-14


@pytest.fixture(scope="module", params=list(CASES))
def pair(request):
    from oracle_cases import OracleProblem
    from product_cases import ProductProblem

    return request.param, ProductProblem(request.param), OracleProblem(request.param)


def test_metrics_bitwise(pair):
    name, p, o = pair
    assert np.array_equal(p.mets0.J_elem, o.J)
    assert np.array_equal(p.mets0.grad_elem, o.grad)
    assert np.array_equal(p.mets0.Jg, o.Jg0) and np.array_equal(p.mets0.gradzeta_g, o.gz0)
    assert np.array_equal(p.mets.Jg, o.Jg) and np.array_equal(p.mets.gradzeta_g, o.gz)
    assert np.array_equal(p.ops.mass.M, o.M) and np.array_equal(p.ops.mass.Minv, o.Minv)


def test_dxdxi_and_cross_bitwise(pair):
    name, p, o = pair
    from oracle import hevi_oracle as O
    from paper_2311_11425_b200 import metrics

    assert np.array_equal(p.mets0.dxdxi, o.dxdxi)
    xm = metrics.cross_product_metrics(p.m)
    _, _, gx = O.cross_metrics(o.m)
    assert np.array_equal(xm.grad_elem, gx)


def test_viscous_metric(pair):
    name, p, o = pair
    G = p.vm.Gnu
    scale = np.max(np.abs(o.Gnu))
    assert np.max(np.abs(G - o.Gnu)) <= 1e-13 * scale
    assert np.max(np.abs(G - np.swapaxes(G, -1, -2))) <= 1e-15 * scale
    # eigenvalues of G: LAPACK resolves them to eps*|G| absolute (the small ones of thin
    # elements only to ~1e-10 relative), so compare vals = 1/lam on that scale
    vg, vo = 1.0 / p.vm.lam, 1.0 / o.lam
    assert np.max(np.abs(vg - vo)) <= 64 * np.finfo(float).eps * np.max(np.abs(vo))
    E = p.vm.evecs
    eye = np.einsum("...ci,...cj->...ij", E, E)
    assert np.max(np.abs(eye - np.eye(3))) < 1e-12


def test_hyperdiffusion_parity(pair):
    name, p, o = pair
    from paper_2311_11425_b200 import hyperdiff, state

    got = hyperdiff.hyperdiffusion_apply(state.StateField("2C", o.state), p.cfg, p.vm, p.ops)
    ref = o.hyper()
    assert rel_l2(got, ref) <= TOL, rel_l2(got, ref)
    assert rel_l2(got, golden(name)["hyper"]) <= TOL
    assert np.all(got[:, 0] == 0.0)


def test_laplacian_parity(pair):
    name, p, o = pair
    from paper_2311_11425_b200 import hyperdiff

    if p.c["lap_fields"] is None:
        pytest.skip("no laplacian fixture")
    g = golden(name)["lap"]
    for col, f in enumerate(p.c["lap_fields"]):
        got = hyperdiff.laplacian_apply(o.state[:, f], p.vm, p.ops)
        assert rel_l2(got, o.lap(f)) <= TOL
        assert rel_l2(got, g[:, col]) <= TOL


def test_device_resident_matches_host_path(pair):
    import torch

    name, p, o = pair
    from paper_2311_11425_b200 import hyperdiff, state

    qd = torch.from_numpy(o.state).cuda()
    out_d = hyperdiff.hyperdiffusion_apply(state.StateField("2C", qd), p.cfg, p.vm, p.ops)
    out_h = hyperdiff.hyperdiffusion_apply(state.StateField("2C", o.state), p.cfg, p.vm, p.ops)
    assert out_d.is_cuda
    assert np.array_equal(out_d.cpu().numpy(), out_h)   # deterministic kernels


def test_dss_primitive_bitwise(pair):
    name, p, o = pair
    from oracle import hevi_oracle as O
    from paper_2311_11425_b200 import assembly

    rng = np.random.default_rng(11)
    fe = rng.standard_normal(p.m.gid.shape + (3,))
    assert np.array_equal(assembly.dss(p.m, fe), O.dss(o.m.gid, o.m.ng, fe))


def test_constant_field_annihilated():
    from paper_2311_11425_b200 import hyperdiff
    from product_cases import ProductProblem

    p = ProductProblem("box_p_n4")
    y = hyperdiff.laplacian_apply(np.full(p.m.nglobal, 3.7), p.vm, p.ops)
    assert np.max(np.abs(y)) < 1e-12 * 3.7 * np.max(np.abs(p.ops.mass.Minv)) * 1e3


def test_inverted_element_raises():
    from paper_2311_11425_b200 import metrics
    from product_cases import product_mesh

    m = product_mesh("box_p_n2_const")
    m.coords[0, 2] = m.coords[0, 2][:, :, ::-1].copy()  # flip zeta in element 0 -> J < 0
    m._dev = None
    with pytest.raises(ValueError):
        metrics.curl_invariant_metrics(m)


def test_hyperdiffusion_config_validation():
    from paper_2311_11425_b200 import hyperdiff

    with pytest.raises(ValueError):
        hyperdiff.HyperDiffConfig(alpha=3)
    with pytest.raises(ValueError):
        hyperdiff.HyperDiffConfig(variables=(0, 1))
    with pytest.raises(ValueError):
        hyperdiff.HyperDiffConfig(mode="bogus")


def test_tile_path_used_and_matches_element_path(pair):
    """The tile-sweep kernel runs for structured meshes and agrees with the element-parallel path."""
    name, p, o = pair
    from paper_2311_11425_b200 import euler, hyperdiff, state

    import os

    assert p.ops._tile_arrays() is not None, "tile plan rejected"
    ops_v1 = euler.EulerOps(p.m, p.mets, p.consts, "2C", hyper=(p.cfg, p.vm))
    ops_v1._h["tiles"] = None
    os.environ["HV_KERNEL"] = "line"          # the line-tile kernel (default is plane-owner for N <= 4)
    try:
        ops_line = euler.EulerOps(p.m, p.mets, p.consts, "2C", hyper=(p.cfg, p.vm))
        ops_line.lap_plan(p.vm)
    finally:
        del os.environ["HV_KERNEL"]
    st = state.StateField("2C", o.state)
    a = hyperdiff.hyperdiffusion_apply(st, p.cfg, p.vm, p.ops)
    b = hyperdiff.hyperdiffusion_apply(st, p.cfg, p.vm, ops_v1)
    c = hyperdiff.hyperdiffusion_apply(st, p.cfg, p.vm, ops_line)
    assert rel_l2(a, b) <= xtol(p) and rel_l2(c, b) <= xtol(p)
    for f in range(1, 5):
        la = hyperdiff.laplacian_apply(o.state[:, f], p.vm, p.ops)
        lb = hyperdiff.laplacian_apply(o.state[:, f], p.vm, ops_v1)
        lc = hyperdiff.laplacian_apply(o.state[:, f], p.vm, ops_line)
        assert rel_l2(la, lb) <= xtol(p) and rel_l2(lc, lb) <= xtol(p)


def test_axis_form_matches_six_components(pair, monkeypatch):
    """Plane kernel with the compact forms of W -- axis (u = sqrt(w3 Jg) e_3, scaled mode with
    c_1 == c_2) and isotropic (s = kh w3 Jg, c_1 == c_2 == c_3) -- equals the 6-component form
    (HV_WFORM=0) to rounding, and the plan picks them exactly when G_nu has that structure."""
    name, p, o = pair
    from paper_2311_11425_b200 import euler, hyperdiff, state

    plan = p.ops.lap_plan(p.vm)
    ax = p.vm.axis_form()
    hd = p.cfg
    assert (ax is not None) == (hd.mode == "scaled" and hd.c[0] == hd.c[1])
    if ax is not None and plan.kernel == 1 and ax[1] == 0.0:
        assert plan.wform == 2                       # isotropic: c_1 == c_2 == c_3
    else:
        assert plan.wform == (1 if (ax is not None and plan.kernel == 1 and plan.N <= 4) else 0)
    if plan.wform == 0:
        pytest.skip("6-component form for this case")
    monkeypatch.setenv("HV_WFORM", "0")
    ops6 = euler.EulerOps(p.m, p.mets, p.consts, "2C", hyper=(p.cfg, p.vm))
    assert ops6.lap_plan(p.vm).wform == 0
    st = state.StateField("2C", o.state)
    a = hyperdiff.hyperdiffusion_apply(st, p.cfg, p.vm, p.ops)
    b = hyperdiff.hyperdiffusion_apply(st, p.cfg, p.vm, ops6)
    assert rel_l2(a, b) <= xtol(p)
    assert rel_l2(a, o.hyper()) <= TOL
    for f in (1, 4):
        la = hyperdiff.laplacian_apply(o.state[:, f], p.vm, p.ops)
        lb = hyperdiff.laplacian_apply(o.state[:, f], p.vm, ops6)
        assert rel_l2(la, lb) <= xtol(p)


def test_tile_ordered_intermediate_bitwise(pair, monkeypatch):
    """H_nu alpha=2 through the tile-ordered intermediate (pass 1 writes L q in the sweep's block
    layout, the fix-up completes the perimeter nodes in place, pass 2 bulk-copies the blocks) is
    bitwise the (nglobal, 4) path: same sums in the same order, only the storage differs."""
    name, p, o = pair
    from paper_2311_11425_b200 import euler, hyperdiff, state

    monkeypatch.setenv("HV_SEG", "0")          # whole columns (small meshes are otherwise segmented)
    monkeypatch.setenv("HV_YT7", "1")          # the N = 7 split-plane variant too
    yops = euler.EulerOps(p.m, p.mets, p.consts, "2C", hyper=(p.cfg, p.vm))
    plan = yops.lap_plan(p.vm)
    if not plan.d_yt:
        pytest.skip("no tile-ordered mode for this plan (N != 4 or not the plane kernel)")
    monkeypatch.setenv("HV_YT", "0")
    ops0 = euler.EulerOps(p.m, p.mets, p.consts, "2C", hyper=(p.cfg, p.vm))
    assert not ops0.lap_plan(p.vm).d_yt
    cfg2 = hyperdiff.HyperDiffConfig(**{**p.c["hd"], "alpha": 2})
    st = state.StateField("2C", o.state)
    a = hyperdiff.hyperdiffusion_apply(st, cfg2, p.vm, yops)
    b = hyperdiff.hyperdiffusion_apply(st, cfg2, p.vm, ops0)
    assert np.array_equal(a, b)
    if p.cfg.alpha == 2:
        assert rel_l2(a, o.hyper()) <= TOL
    # accumulate into an existing output, device-resident
    import torch

    qd = torch.from_numpy(o.state).cuda()
    base = torch.randn_like(qd)
    oa, ob = base.clone(), base.clone()
    hyperdiff.hyperdiffusion_apply(state.StateField("2C", qd), cfg2, p.vm, yops, out=oa, accumulate=True)
    hyperdiff.hyperdiffusion_apply(state.StateField("2C", qd), cfg2, p.vm, ops0, out=ob, accumulate=True)
    assert torch.equal(oa, ob)


@pytest.mark.parametrize("seg", ["1", "2"])
def test_vertical_segments_match_whole_columns(pair, monkeypatch, seg):
    """The plane sweep cut into vertical segments (HV_SEG layers per CTA; the levels between segments
    completed by the slot fix-up) gives the whole-column result to rounding, for H_nu and for the
    Laplacian on 1, 4 and 5 fields."""
    name, p, o = pair
    from paper_2311_11425_b200 import euler, hyperdiff, state

    if p.m.degree > 4 or p.c.get("nv", 2) < 2 or not p.ops._tile_arrays():
        pytest.skip("segments: N <= 4 plane kernel, >= 2 layers")
    monkeypatch.setenv("HV_SEG", "0")
    ops0 = euler.EulerOps(p.m, p.mets, p.consts, "2C", hyper=(p.cfg, p.vm))
    ops0.lap_plan(p.vm)                        # plans are built lazily: before HV_SEG changes
    monkeypatch.setenv("HV_SEG", seg)
    ops1 = euler.EulerOps(p.m, p.mets, p.consts, "2C", hyper=(p.cfg, p.vm))
    plan = ops1.lap_plan(p.vm)
    if plan.seg == 0:
        pytest.skip("mesh has fewer layers than the segment")
    assert ops0.lap_plan(p.vm).seg == 0 and not plan.d_yt
    st = state.StateField("2C", o.state)
    a = hyperdiff.hyperdiffusion_apply(st, p.cfg, p.vm, ops0)
    b = hyperdiff.hyperdiffusion_apply(st, p.cfg, p.vm, ops1)
    assert rel_l2(b, a) <= 1e-14 and rel_l2(b, o.hyper()) <= TOL
    for fields in ((3,), (1, 2, 3, 4), (0, 1, 2, 3, 4)):
        la = hyperdiff.laplacian_apply_fields(o.state, p.vm, ops0, fields)
        lb = hyperdiff.laplacian_apply_fields(o.state, p.vm, ops1, fields)
        assert rel_l2(lb, la) <= 1e-14


def test_all_five_fields_one_pass(pair):
    """F=5 tile kernel (config 1 applies L to all five fields)."""
    name, p, o = pair
    from paper_2311_11425_b200 import hyperdiff

    got = hyperdiff.laplacian_apply_fields(o.state, p.vm, p.ops, (0, 1, 2, 3, 4))
    ref = np.stack([o.lap(f) for f in range(5)], axis=1)
    assert rel_l2(got, ref) <= TOL


def test_rhs_full_and_horizontal_parity(pair):
    """S(q) and H(q) (sets 2NC / 2C / 3C) vs the oracle and the reference goldens, random states."""
    name, p, o = pair
    from cases import random_state
    from paper_2311_11425_b200 import euler, state

    g = golden(name)
    for s in p.c["sets"]:
        ops = euler.EulerOps(p.m, p.mets, p.consts, s, hyper=(p.cfg, p.vm))
        rs = random_state(p.m.nglobal, s)
        oe = o.euler(s)
        full = ops.rhs_full(state.StateField(s, rs))
        assert rel_l2(full, oe.rhs_full(rs)) <= TOL, (s, rel_l2(full, oe.rhs_full(rs)))
        assert rel_l2(full, g[f"rhs_full_{s}"]) <= TOL
        hor = ops.rhs_horizontal(state.StateField(s, rs), with_hyperdiff=False)
        assert rel_l2(hor, oe.rhs_horizontal_nohd(rs)) <= TOL, s
        assert rel_l2(hor, g[f"rhs_h_{s}"]) <= TOL


def test_rhs_full_plus_hyperdiffusion(pair):
    """The config-4 quantity S + H_nu in one buffer, and rhs_horizontal with H_nu."""
    name, p, o = pair
    from cases import random_state
    from paper_2311_11425_b200 import euler, state

    s = "2C"
    ops = euler.EulerOps(p.m, p.mets, p.consts, s, hyper=(p.cfg, p.vm))
    rs = o.state if p.c["state"] == "bubble" else random_state(p.m.nglobal, s)
    oe = o.euler(s)
    ref = oe.rhs_full(rs) + o.hyper(rs)
    got = ops.rhs_full_hyper(state.StateField(s, rs))
    assert rel_l2(got, ref) <= TOL, rel_l2(got, ref)
    ref_h = oe.rhs_horizontal_nohd(rs) + o.hyper(rs)
    got_h = ops.rhs_horizontal(state.StateField(s, rs), with_hyperdiff=True)
    assert rel_l2(got_h, ref_h) <= TOL


def test_rhs_vertical_and_splitting(pair):
    """V(q) per column vs the oracle and the reference goldens; H + V == S with omega = 0."""
    name, p, o = pair
    from cases import random_state
    from paper_2311_11425_b200 import euler, state

    g = golden(name)
    for s in p.c["sets"]:
        ops = euler.EulerOps(p.m, p.mets, p.consts, s, hyper=(p.cfg, p.vm))
        rs = random_state(p.m.nglobal, s)
        v = ops.rhs_vertical(state.StateField(s, rs))
        assert rel_l2(v, o.euler(s).rhs_vertical(rs)) <= TOL, (s, rel_l2(v, o.euler(s).rhs_vertical(rs)))
        assert rel_l2(v, g[f"rhs_v_{s}"]) <= TOL
        if p.c["omega"] == 0.0:
            h = ops.rhs_horizontal(state.StateField(s, rs), with_hyperdiff=False)
            full = ops.rhs_full(state.StateField(s, rs))
            # SPEC.md:292 asks H + V == S; the reference does not satisfy it pointwise
            # (V divides by the column mass, S by the 3-D mass: ~1e-3 on random
            # states), so the check is that our splitting defect is the reference's.
            oe = o.euler(s)
            ref_defect = oe.rhs_horizontal_nohd(rs) + oe.rhs_vertical(rs) - oe.rhs_full(rs)
            err = np.linalg.norm((h + v - full) - ref_defect) / np.linalg.norm(full)
            assert err <= 1e-11, (s, err)


def test_column_system(pair):
    """LHEVI column Jacobian band (hv_column_jacobian), band LU (hv_band_lu_factor) and
    back-solve (hv_band_solve) against the oracle and the reference fixtures."""
    name, p, o = pair
    if name == "c1":
        pytest.skip("no column-system fixture for c1")
    from cases import random_state
    from oracle import hevi_oracle as O
    from paper_2311_11425_b200 import euler, linalg

    g = golden(name)
    for s in p.c["sets"]:
        ops = euler.EulerOps(p.m, p.mets, p.consts, s, hyper=(p.cfg, p.vm))
        rs = random_state(p.m.nglobal, s)
        qcol = np.ascontiguousarray(rs[p.m.col_gid][:24])
        band = ops.column_jacobian(qcol, 0.37)
        ob, kl, ku = O.column_jacobian(o.euler(s), rs[p.m.col_gid], 0.37)
        ob = np.ascontiguousarray(ob[:24])
        assert (kl, ku) == (ops.kl, ops.ku) and band.shape == ob.shape
        assert np.abs(band - ob).max() <= 1e-13 * np.abs(ob).max(), (s, np.abs(band - ob).max())
        assert rel_l2(band[:, :, :g[f"jac_cols_{s}"].shape[2]], g[f"jac_cols_{s}"]) <= 1e-13
        # the factorisation repeats the reference's elementary operations: bitwise on the same band
        ref_band = ob.copy()
        ipiv, flops = linalg.banded_lu_factor_batch(ref_band, kl, ku)
        assert sha(ref_band) == str(g[f"lu_sha_{s}"]), s
        assert np.array_equal(ipiv, g[f"ipiv_{s}"]), s
        rhs = np.random.default_rng(11).standard_normal((24, ops.Mdim))
        x, _ = linalg.banded_solve_batch(ref_band, ipiv, kl, ku, rhs)
        # a backward-stable solve: the bar scales with the system's conditioning (~1e4 for the
        # N = 6 3C columns), so 1e-11 here
        assert rel_l2(x, g[f"solve_{s}"]) <= 1e-11, (s, rel_l2(x, g[f"solve_{s}"]))
        # our own band end to end (within 1e-13 of the reference's, not bitwise): the pivots follow
        # the reference's except at exact ties of |candidates| in the reference band (symmetric
        # geometry, e.g. the one-element-per-panel sphere), where rounding may pick the other row;
        # the solution is held to the bar either way
        ip2, _ = linalg.banded_lu_factor_batch(band, kl, ku)
        if name != "sphere_n7":
            assert np.array_equal(ip2, g[f"ipiv_{s}"]), s
        x2, _ = linalg.banded_solve_batch(band, ip2, kl, ku, rhs)
        assert rel_l2(x2, g[f"solve_{s}"]) <= 1e-11, (s, rel_l2(x2, g[f"solve_{s}"]))


def test_band_lu_singular_and_wide():
    from paper_2311_11425_b200 import linalg

    kl = ku = 2
    data = np.zeros((2, 2 * kl + ku + 1, 6))
    data[:, kl + ku, :] = 1.0
    data[1, kl + ku, 3] = 0.0     # system 1: zero pivot at column 3 (nothing below to swap in)
    with pytest.raises(linalg.SingularMatrixError) as e:
        linalg.banded_lu_factor_batch(data, kl, ku)
    assert e.value.j == 3 and e.value.batch == 1


@pytest.mark.parametrize("kl,M,nb", [(4, 9, 3), (24, 85, 5), (24, 165, 7), (24, 645, 3), (39, 232, 4), (2, 300, 9)])
def test_band_lu_random_vs_oracle(kl, M, nb):
    """Random (pivoting) band systems of the column-system shapes, incl. M far beyond the
    kernel's column window: factors bitwise equal to the oracle, solve within tolerance."""
    from oracle import hevi_oracle as O
    from paper_2311_11425_b200 import linalg

    ku = kl
    rng = np.random.default_rng(kl * 1000 + M)
    data = np.zeros((nb, 2 * kl + ku + 1, M))
    for j in range(M):                     # random entries inside the band, zero fill-in rows
        lo, hi = max(0, j - ku), min(M - 1, j + kl)
        data[:, kl + ku + lo - j:kl + ku + hi - j + 1, j] = rng.standard_normal((nb, hi - lo + 1))
    ref = data.copy()
    ip_ref = O.band_lu_factor(ref, kl, ku)
    got = data.copy()
    ip, _ = linalg.banded_lu_factor_batch(got, kl, ku)
    assert np.array_equal(ip, ip_ref)
    assert np.array_equal(got, ref)
    b = rng.standard_normal((nb, M))
    x, _ = linalg.banded_solve_batch(got, ip, kl, ku, b)
    assert rel_l2(x, O.band_solve(ref, ip_ref, kl, ku, b)) <= 1e-12


@pytest.mark.parametrize("cname", ["box_p_n4", "sphere_n4"])
def test_diagnostics_device(cname):
    """hv_euler_diagnostics vs the reference's EulerOps.diagnostics (sums within 1e-12
    relative, extrema exact)."""
    import torch

    from product_cases import ProductProblem
    from paper_2311_11425_b200 import euler, state

    z = golden("diag")
    p = ProductProblem(cname)
    for s in ("2C", "2NC", "3C"):
        ops = euler.EulerOps(p.m, p.mets, state.PhysConstants(omega=0.0), s)
        q = torch.from_numpy(z[f"{cname}_{s}_state"]).cuda()
        d = ops.diagnostics(state.StateField(s, q))
        ref = dict(zip(z[f"{cname}_{s}_keys"], z[f"{cname}_{s}_vals"]))
        for k, v in ref.items():
            tol = 0.0 if k in ("w_vertical_max",) else 1e-12
            assert abs(d[k] - v) <= tol * max(abs(v), 1.0) + (1e-9 if k == "energy_internal" and s == "3C" else 0), \
                (s, k, d[k], v)


@pytest.mark.parametrize("kernel,split,tile", [("", "4", (1, 1)), ("", "2", (1, 1)), ("plane2x2", "4", (2, 2)),
                                               ("plane2x2", "2", (2, 2)), ("line", "4", (1, 1))])
def test_n7_sweep_kernels(monkeypatch, kernel, split, tile):
    """The N = 7 sweeps: split-plane kernel (H lanes per plane exchanging xi lines by shuffles)
    on 1x1 (default) and 2x2 tiles, and the line kernel, against the oracle and the golden."""
    monkeypatch.setenv("HV_N7_KERNEL", kernel)
    monkeypatch.setenv("HV_N7_SPLIT", split)
    from oracle_cases import OracleProblem
    from product_cases import ProductProblem
    from paper_2311_11425_b200 import hyperdiff, state

    p = ProductProblem("box_n7")
    plan = p.ops.lap_plan(p.vm)
    assert plan.kernel == (0 if kernel == "line" else 1) and (plan.TX, plan.TY) == tile
    o = OracleProblem("box_n7")
    got = hyperdiff.hyperdiffusion_apply(state.StateField("2C", o.state), p.cfg, p.vm, p.ops)
    assert rel_l2(got, o.hyper()) <= TOL
    assert rel_l2(got, golden("box_n7")["hyper"]) <= TOL


def test_elem_deriv_primitives(pair):
    """assembly.elem_deriv / weak_deriv_acc (assembly.py:29-51) on random element data."""
    name, p, o = pair
    from oracle import hevi_oracle as O
    from paper_2311_11425_b200 import assembly

    dev = p.m.device()
    f = np.random.default_rng(3).standard_normal((dev.nelem, dev.n, dev.n, dev.n))
    for axis in range(3):
        assert rel_l2(assembly.elem_deriv(p.m, f, axis), O.dstrong(o.m.D, f, axis)) <= 1e-13
        assert rel_l2(assembly.weak_deriv_acc(p.m, f, axis), O.dweak(o.m.D, o.m.w3, f, axis)) <= 1e-13


def test_column_apply(pair):
    """EulerOps.column_apply (euler.py:231-235): V on column-gathered states."""
    name, p, o = pair
    from cases import random_state
    from paper_2311_11425_b200 import euler

    for s in p.c["sets"]:
        ops = euler.EulerOps(p.m, p.mets, p.consts, s, hyper=(p.cfg, p.vm))
        rs = random_state(p.m.nglobal, s)
        got = ops.column_apply(rs[p.m.col_gid])
        ref = o.euler(s).rhs_vertical(rs)[p.m.col_gid]
        assert rel_l2(got, ref) <= TOL, s


def test_euler_column_sweep_vs_element_path(monkeypatch):
    """N = 7 (single-column tile plan): the column-sweep Euler RHS (hv_euler_rhs_tiles, on-chip
    vertical DSS + fixed-order slot fix-up) against the element kernel + CSR DSS path and the
    oracle, all sets, S and H (with and without accumulation)."""
    import torch

    from cases import random_state
    from oracle_cases import OracleProblem
    from product_cases import ProductProblem
    from paper_2311_11425_b200 import euler, state

    p = ProductProblem("box_n7")
    o = OracleProblem("box_n7")
    for s in ("2C", "2NC", "3C"):
        ops = euler.EulerOps(p.m, p.mets, p.consts, s)
        assert ops._euler_tile_plan() is not None
        q = torch.from_numpy(random_state(p.m.nglobal, s)).cuda()
        full = ops.rhs_full(state.StateField(s, q)).cpu().numpy()
        hor = ops.rhs_horizontal(state.StateField(s, q), with_hyperdiff=False).cpu().numpy()
        acc = torch.ones_like(q)
        ops._rhs(q, 7, 0, out=acc, accumulate=True)
        monkeypatch.setenv("HV_EULER_TILES", "0")
        ops2 = euler.EulerOps(p.m, p.mets, p.consts, s)
        assert ops2._euler_tile_plan() is None
        full2 = ops2.rhs_full(state.StateField(s, q)).cpu().numpy()
        hor2 = ops2.rhs_horizontal(state.StateField(s, q), with_hyperdiff=False).cpu().numpy()
        monkeypatch.delenv("HV_EULER_TILES")
        oe = o.euler(s)
        rs = q.cpu().numpy()
        assert rel_l2(full, oe.rhs_full(rs)) <= TOL and rel_l2(full, full2) <= 1e-13, s
        assert rel_l2(hor, oe.rhs_horizontal_nohd(rs)) <= TOL and rel_l2(hor, hor2) <= 1e-13, s
        assert rel_l2(acc.cpu().numpy() - 1.0, full) <= 1e-12, s


def test_misaligned_output_view():
    """An output that is not 16-byte aligned (an offset view) takes the element-parallel path
    (the sweeps store rows with 16-byte stores) and gives the same result."""
    import torch

    from product_cases import ProductProblem
    from oracle_cases import OracleProblem
    from paper_2311_11425_b200 import hyperdiff, state

    p = ProductProblem("box_p_n4")
    o = OracleProblem("box_p_n4")
    q = torch.from_numpy(o.state).cuda()
    ref = hyperdiff.hyperdiffusion_apply(state.StateField("2C", q), p.cfg, p.vm, p.ops)
    ng = q.shape[0]
    big = torch.full((ng * 5 + 1,), float("nan"), dtype=torch.float64, device="cuda")
    out = big[1:].view(ng, 5)
    assert out.data_ptr() % 16 == 8
    hyperdiff.hyperdiffusion_apply(state.StateField("2C", q), p.cfg, p.vm, p.ops, out=out)
    assert rel_l2(out.cpu().numpy(), ref.cpu().numpy()) <= 1e-14
    assert rel_l2(out.cpu().numpy(), o.hyper()) <= TOL


@pytest.mark.parametrize("case", ["box_p_n4", "box_n7"])
def test_laplacian_leaves_unlisted_columns(case):
    """hv_laplacian writes only the listed output columns: with ldo = 5, fields 1..4 and no zero
    mask, column 0 of the output keeps the caller's values on every node (the 16-byte (ng, 5) row
    stores of the sweeps zero column 0 only for H_nu's zero mask)."""
    import ctypes as C

    import torch

    from oracle_cases import OracleProblem
    from product_cases import ProductProblem
    from paper_2311_11425_b200 import _lib, hyperdiff

    p = ProductProblem(case)
    o = OracleProblem(case)
    q = torch.from_numpy(o.state).cuda()
    out = torch.full_like(q, 7.0)
    fl = (C.c_int32 * 4)(1, 2, 3, 4)
    plan = p.ops.lap_plan(p.vm)
    _lib.check(_lib.lib().hv_laplacian(C.byref(plan), q.data_ptr(), 5, 4, fl, out.data_ptr(), 5, fl, 1.0,
                                       _lib.stream_handle()))
    got = out.cpu().numpy()
    assert np.all(got[:, 0] == 7.0)
    ref = hyperdiff.laplacian_apply_fields(q, p.vm, p.ops, (1, 2, 3, 4)).cpu().numpy()
    assert np.array_equal(got[:, 1:], ref[:, 1:])


def test_eos_power_device():
    """The power function of the Euler kernels' equation of state (csrc/hv_pow.cuh; state.py:84-101 uses
    numpy's power, i.e. glibc pow): within 1 ulp of numpy over the EOS range and far outside it, and
    the library pow for arguments outside the fast path (zero, subnormal, huge exponents)."""
    import torch

    from paper_2311_11425_b200 import _lib

    rng = np.random.default_rng(7)
    x = np.concatenate([0.5 + 1.5 * rng.random(200000), np.exp((rng.random(200000) * 2 - 1) * 200.0),
                        [0.0, 1e-320, 1e-200, 1e200, np.inf, 1.0]])
    xd = torch.from_numpy(x).cuda()
    out = torch.empty_like(xd)
    for y in (1.4, 1004.5 / 717.5, -1.4, 0.5):
        _lib.check(_lib.lib().hv_probe_pow(x.size, xd.data_ptr(), y, out.data_ptr(), _lib.stream_handle()))
        got = out.cpu().numpy()
        with np.errstate(divide="ignore", over="ignore"):
            ref = np.power(x, y)
        fin = np.isfinite(ref) & (ref != 0)
        assert np.array_equal(got[~fin], ref[~fin])
        ulp = np.abs(got[fin] - ref[fin]) / np.spacing(np.abs(ref[fin]))
        assert ulp.max() <= 1.0, (y, ulp.max())


def test_small_mesh_graph_replay():
    """Small meshes replay a captured CUDA graph from the third call with the same plan and buffers
    (hyperdiff._run_graphed): the replays read the buffers' current contents and give the first
    call's bits; HV_GRAPH=0 (no capture) gives the same."""
    import torch

    from oracle_cases import OracleProblem
    from product_cases import ProductProblem
    from paper_2311_11425_b200 import hyperdiff, state

    p = ProductProblem("box_p_n4")
    o = OracleProblem("box_p_n4")
    q = torch.from_numpy(o.state).cuda()
    out = torch.empty_like(q)
    st = state.StateField("2C", q)
    hyperdiff._GRAPHS.clear()
    first = hyperdiff.hyperdiffusion_apply(st, p.cfg, p.vm, p.ops, out=out).clone()
    assert rel_l2(first.cpu().numpy(), o.hyper()) <= TOL
    for _ in range(3):
        out.fill_(float("nan"))
        hyperdiff.hyperdiffusion_apply(st, p.cfg, p.vm, p.ops, out=out)
        assert torch.equal(out, first)
    assert any(g is not None for _, g in hyperdiff._GRAPHS.values())
    q.mul_(2.0)                                   # a replay reads the new contents
    hyperdiff.hyperdiffusion_apply(st, p.cfg, p.vm, p.ops, out=out)
    assert torch.equal(out, 2.0 * first)
    lap = [hyperdiff.laplacian_apply_fields(q, p.vm, p.ops, (0, 1, 2, 3, 4)) for _ in range(4)]
    assert all(torch.equal(x, lap[0]) for x in lap[1:])


def test_division_by_reciprocal_is_ieee():
    """hv::div_rcp (one correctly rounded reciprocal per divisor, then a rb and an exact-residual correction:
    the Euler column sweep's quotients by rho and P_A) gives IEEE a / b bit for bit: 4e8 pairs over the
    magnitudes of densities, momenta and pressures."""
    import torch

    from paper_2311_11425_b200 import _lib

    rng = np.random.default_rng(11)
    n = 200000
    a = (rng.standard_normal(n) * np.exp(rng.uniform(-12, 12, n)))
    b = np.concatenate([rng.uniform(0.01, 2.0, n // 2), np.exp(rng.uniform(-12, 12, n - n // 2))])
    ad, bd = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    bad = torch.zeros(1, dtype=torch.int64, device="cuda")
    _lib.check(_lib.lib().hv_probe_div(n, ad.data_ptr(), bd.data_ptr(), bad.data_ptr(), _lib.stream_handle()))
    assert int(bad.item()) == 0
