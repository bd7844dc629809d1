"""Generate golden fixtures by running the REFERENCE implementation (hevicore).

Run in the build container, where the reference is mounted read-only:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Every fixture is produced by the reference's own public API on seeded inputs
from ``paper_2311_11425_b200.synthetic`` (geometry seed 0, state seed 1);
the GPU box has no /root/reference, so the committed .npz files plus the
oracle (oracle/hevi_oracle.py, pinned against these fixtures by
tests/test_oracle_golden.py) are the parity anchors there.

Each case stores the reference arrays that are small, and SHA-256 digests of
the exact bytes of the bit-exact integer/metric arrays.
"""

from __future__ import annotations

import hashlib
import os
import sys
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))
sys.path.insert(0, REF)
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")

from hevicore import basis as rbasis  # noqa: E402
from hevicore import euler as reuler  # noqa: E402
from hevicore import hyperdiff as rhd  # noqa: E402
from hevicore import linalg as rlinalg  # noqa: E402
from hevicore import ark as rark  # noqa: E402
from hevicore import hevi as rhevi  # noqa: E402
from hevicore import mesh as rmesh  # noqa: E402
from hevicore import metrics as rmet  # noqa: E402
from hevicore import state as rstate  # noqa: E402

from paper_2311_11425_b200 import synthetic  # noqa: E402

sys.path.insert(0, str(HERE.parent))
from cases import CASES, LHEVI, window_args, diag_state, lhevi_state, make_state, random_state  # noqa: E402


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def ref_mesh_lattice(nx, ny, nv, N, extents, perturb):
    coords, layer, hcol = synthetic.perturbed_box_coords(nx, ny, nv, N, extents, perturb=perturb)
    cfg = rmesh.MeshConfig("box", panels_per_edge=max(nx, ny), n_elem_vertical=nv, degree=N,
                           box_extents=tuple(float(e) for e in extents))
    b = rbasis.lobatto(N)
    return rmesh.Mesh(cfg, coords, (b, b, b), layer, hcol)


JAC_COLS = 24
JAC_LAM = 0.37


def case(name, m, hd_cfg, dt, state, sets=("2C",), omega=0.0, store_full=True, lap_fields=None, jac=False,
         c4_target=False):
    """Reference outputs for one mesh; inputs are regenerated from the seeds by the tests."""
    out = {}
    mets0 = rmet.curl_invariant_metrics(m)
    mets = rmet.project_metrics_to_columns(mets0, m)
    consts = rstate.PhysConstants(omega=omega)
    out["ng"] = np.array(m.nglobal)
    out["state"] = state                       # the exact input bytes (tests use these on any host)
    out["sha_state"] = np.array(sha(state))
    out["sha_gid"] = np.array(sha(m.gid))
    out["sha_xg"] = np.array(sha(m.xg))
    out["sha_col_gid"] = np.array(sha(m.col_gid))
    out["sha_flux_mask"] = np.array(sha(m.flux_mask))
    out["sha_J"] = np.array(sha(mets0.J_elem))
    out["sha_grad"] = np.array(sha(mets0.grad_elem))
    out["sha_dxdxi"] = np.array(sha(mets0.dxdxi))
    out["sha_Jg_naive"] = np.array(sha(mets0.Jg))
    out["sha_gz_naive"] = np.array(sha(mets0.gradzeta_g))
    out["sha_Jg"] = np.array(sha(mets.Jg))
    out["sha_gz"] = np.array(sha(mets.gradzeta_g))
    xm = rmet.cross_product_metrics(m)
    out["sha_grad_cross"] = np.array(sha(xm.grad_elem))
    vm = rhd.build_viscous_metric(m, mets, hd_cfg, dt=dt)
    ops = reuler.EulerOps(m, mets, consts, (sets or ("2C",))[0], hyper=(hd_cfg, vm))
    out["sha_M"] = np.array(sha(ops.mass.M))
    st = rstate.StateField((sets or ("2C",))[0], state)
    if lap_fields is not None:
        out["lap"] = np.stack([rhd.laplacian_apply(state[:, f], vm, ops) for f in lap_fields], axis=1)
    out["hyper"] = rhd.hyperdiffusion_apply(st, hd_cfg, vm, ops)
    if c4_target:
        # config 4's quantity on the case state itself: rhs_full + hyperdiffusion_apply
        # (euler.py:111-118 + hyperdiff.py:97-106); near-hydrostatic, so S alone is ill-conditioned
        out["c4_target"] = ops.rhs_full(st) + out["hyper"]
        out["rhs_full_state"] = ops.rhs_full(st)
    for s in sets:
        o = reuler.EulerOps(m, mets, consts, s, hyper=(hd_cfg, vm))
        rs = random_state(m.nglobal, s, seed=7)
        out[f"rhs_full_{s}"] = o.rhs_full(rstate.StateField(s, rs))
        out[f"rhs_h_{s}"] = o.rhs_horizontal(rstate.StateField(s, rs), with_hyperdiff=False)
        out[f"rhs_v_{s}"] = o.rhs_vertical(rstate.StateField(s, rs))
        if jac:
            # LHEVI column system (euler.py:274-306, linalg.py:112-194) on a column subset
            band = np.ascontiguousarray(o.column_jacobian(rs[m.col_gid], JAC_LAM)[:JAC_COLS])
            out[f"jac_sha_{s}"] = np.array(sha(band))
            out[f"jac_cols_{s}"] = band[:, :, :2 * o.nvar * o.nzl].copy()
            bf = band.copy()
            ipiv, _ = rlinalg.banded_lu_factor_batch(bf, o.kl, o.ku)
            out[f"lu_sha_{s}"] = np.array(sha(bf))
            out[f"ipiv_{s}"] = ipiv.astype(np.int32)
            rhs = np.random.default_rng(11).standard_normal((band.shape[0], o.Mdim))
            x, _ = rlinalg.banded_solve_batch(bf, ipiv, o.kl, o.ku, rhs)
            out[f"solve_{s}"] = x
    if store_full:
        out["gid"] = m.gid.astype(np.int32)
        out["Jg"] = mets.Jg
        out["gz"] = mets.gradzeta_g
        out["M"] = ops.mass.M
        out["Gnu_sample"] = vm.Gnu.reshape(-1, 3, 3)[:: max(1, vm.Gnu.size // 9 // 512)]
    np.savez_compressed(HERE / f"{name}.npz", **out)
    print(name, "ng", m.nglobal, "nelem", m.nelem, "bytes", (HERE / f"{name}.npz").stat().st_size)


def ref_mesh(c):
    if c["kind"] == "window":
        coords, layer, hcol = synthetic.box_window_coords(*window_args(c))
        cfg = rmesh.MeshConfig("box", panels_per_edge=max(c["nx"], c["ny"]), n_elem_vertical=c["nv"],
                               degree=c["N"], box_extents=tuple(float(e) for e in c["extents"]))
        b = rbasis.lobatto(c["N"])
        return rmesh.Mesh(cfg, coords, (b, b, b), layer, hcol)
    if c["kind"] == "lattice":
        return ref_mesh_lattice(c["nx"], c["ny"], c["nv"], c["N"], c["extents"], perturb=True)
    if c["kind"] == "sphere":
        cfg = rmesh.MeshConfig("sphere", panels_per_edge=c["ne"], n_elem_vertical=c["nv"], degree=c["N"],
                               radius=c["radius"], z_top=c["z_top"])
        return rmesh.build_cubed_sphere(cfg)
    cfg = rmesh.MeshConfig("box", panels_per_edge=c["ne"], n_elem_vertical=c["nv"], degree=c["N"],
                           box_extents=c["extents"])
    return rmesh.build_box(cfg)


def lhevi_fixture():
    """IMEX tableaux (ark.py) and reference LHEVI steps (hevi.step_lhevi) for the device driver."""
    out = {}
    for name in rark.tableau_names():
        t = rark.tableau(name)
        for f in ("A", "b", "c", "A_im", "b_im", "c_im"):
            out[f"tab_{name}_{f}"] = np.asarray(getattr(t, f), dtype=np.float64)
        out[f"tab_{name}_order"] = np.array(t.order)
    c = CASES[LHEVI["case"]]
    m = ref_mesh(c)
    mets = rmet.project_metrics_to_columns(rmet.curl_invariant_metrics(m), m)
    hd = rhd.HyperDiffConfig(**LHEVI["hd"])
    vm = rhd.build_viscous_metric(m, mets, hd, dt=LHEVI["dt"])
    ops = reuler.EulerOps(m, mets, rstate.PhysConstants(omega=0.0), "2C", hyper=(hd, vm))
    q0 = lhevi_state(m.xg, stored=False)
    out["q0"] = q0
    for name in LHEVI["tabs"]:
        ls = rhevi.LheviState(update_interval=LHEVI["update_interval"], mode="PS")
        q = q0.copy()
        for k in range(LHEVI["steps"]):
            q = rhevi.step_lhevi(ops, rark.tableau(name), q, LHEVI["dt"], ls)
            out[f"step_{name}_{k}"] = q
    np.savez_compressed(HERE / "lhevi.npz", **out)
    print("lhevi", "bytes", (HERE / "lhevi.npz").stat().st_size)


def diag_fixture():
    """EulerOps.diagnostics (euler.py:421-456) for all sets on a box and the sphere, and a
    run.dump_fields dump (run.py:202-211), from the reference."""
    import tempfile

    from hevicore import run as rrun

    out = {}
    for cname in ("box_p_n4", "sphere_n4"):
        c = CASES[cname]
        m = ref_mesh(c)
        mets = rmet.project_metrics_to_columns(rmet.curl_invariant_metrics(m), m)
        consts = rstate.PhysConstants(omega=0.0)
        q2c = diag_state(m)
        for s in ("2C", "2NC", "3C"):
            ops = reuler.EulerOps(m, mets, consts, s)
            st = rstate.convert_state(rstate.StateField("2C", q2c), s, consts, ops.Phi_g)
            out[f"{cname}_{s}_state"] = st.data
            d = ops.diagnostics(st)
            out[f"{cname}_{s}_keys"] = np.array(sorted(d))
            out[f"{cname}_{s}_vals"] = np.array([d[k] for k in sorted(d)])
        if cname == "box_p_n4":
            with tempfile.TemporaryDirectory() as td:
                rrun.dump_fields(td + "/f", m, rstate.StateField("2C", q2c), 12.5)
                out["dump_bin"] = np.frombuffer(open(td + "/f.bin", "rb").read(), dtype=np.uint8)
                out["dump_hdr"] = np.array(open(td + "/f.hdr").read())
    np.savez_compressed(HERE / "diag.npz", **out)
    print("diag", "bytes", (HERE / "diag.npz").stat().st_size)


def add_states():
    """Add the regenerated input states to existing fixtures without re-running the reference
    (``--states-only``; tests/test_oracle_golden.py proves they are the bytes the fixtures were
    made from: the oracle reproduces every stored output bit for bit from them)."""
    for name, c in CASES.items():
        f = HERE / f"{name}.npz"
        z = dict(np.load(f))
        coords_mesh = ref_mesh(c)
        st = make_state(c, coords_mesh.xg)
        z["state"], z["sha_state"] = st, np.array(sha(st))
        np.savez_compressed(f, **z)
        print(name, "state", st.shape, f.stat().st_size)
    f = HERE / "lhevi.npz"
    z = dict(np.load(f))
    z["q0"] = lhevi_state(ref_mesh(CASES[LHEVI["case"]]).xg, stored=False)
    np.savez_compressed(f, **z)


def main():
    if "--states-only" in sys.argv:
        add_states()
        return
    only = [a for a in sys.argv[1:] if not a.startswith("-")]
    if only:   # regenerate the named cases only
        for name in only:
            c = CASES[name]
            m = ref_mesh(c)
            case(name, m, rhd.HyperDiffConfig(**c["hd"]), c["dt"], make_state(c, m.xg), sets=c["sets"],
                 omega=c["omega"], store_full=(name != "c1"), lap_fields=c["lap_fields"], jac=(name != "c1"),
                 c4_target=c.get("c4_target", False))
        return
    diag_fixture()
    lhevi_fixture()
    for name, c in CASES.items():
        m = ref_mesh(c)
        case(name, m, rhd.HyperDiffConfig(**c["hd"]), c["dt"], make_state(c, m.xg), sets=c["sets"],
             omega=c["omega"], store_full=(name != "c1"), lap_fields=c["lap_fields"], jac=(name != "c1"),
             c4_target=c.get("c4_target", False))
    # basis constants
    np.savez_compressed(HERE / "basis.npz", **{f"D{N}": rbasis.lobatto(N).diff_matrix for N in range(1, 9)},
                        **{f"w{N}": rbasis.lobatto(N).weights for N in range(1, 9)},
                        **{f"x{N}": rbasis.lobatto(N).nodes for N in range(1, 9)})


if __name__ == "__main__":
    main()
