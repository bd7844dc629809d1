"""Config 4 at full size (64 x 64 x 16 elements, N = 7): S + H_nu on the GPU vs the CPU oracle.

    python tools/c4_fullsize_parity.py [--out profiles/r02_c4_fullsize_parity.txt]

The oracle (oracle/hevi_oracle.py, pinned bit for bit to the reference's outputs) needs
~27 GB of host RAM and several minutes for the mesh, metrics and G_nu of 33.5 M element
nodes; this is a one-off check run on the GPU box (not part of pytest), its output is
committed under profiles/.  Target quantity: rhs_full(q) + hyperdiffusion_apply(q)
(euler.py:111-118 + hyperdiff.py:97-106) on the c4 bubble state, <= 1e-12 relative L2.
"""

from __future__ import annotations

import argparse
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--ne", type=int, default=64)
    ap.add_argument("--nv", type=int, default=16)
    args = ap.parse_args()
    import torch

    from cases import rel_l2
    from oracle_cases import OracleProblem
    from product_cases import ProductProblem
    from paper_2311_11425_b200 import euler, state

    case = dict(kind="box", ne=args.ne, nv=args.nv, N=7, extents=(1.0e4, 1.0e4, 1.0e4),
                hd=dict(alpha=2, c=(0.02, 0.02, 0.02)), dt=0.1, state="bubble", sets=("2C",), omega=0.0,
                lap_fields=None)
    lines = []

    def log(s):
        print(s, flush=True)
        lines.append(s)

    log(f"c4 full-size parity: box {args.ne}x{args.ne}x{args.nv}, N=7, set 2C, c=(0.02,0.02,0.02), dt=0.1; "
        f"host {os.cpu_count()} cpus")
    t0 = time.time()
    p = ProductProblem("c4_full", case=case)
    log(f"product setup {time.time() - t0:.1f} s: nelem {p.m.nelem}, nglobal {p.m.nglobal}")
    t0 = time.time()
    o = OracleProblem("c4_full", case=case)
    log(f"oracle setup {time.time() - t0:.1f} s: ng {o.m.ng}")
    assert np.array_equal(p.m.gid, o.m.gid), "gid differs"
    log("gid bit-equal: True")
    for name, a, b in (("J_elem", p.mets0.J_elem, o.J), ("grad_elem", p.mets0.grad_elem, o.grad),
                       ("Jg", p.mets.Jg, o.Jg), ("gradzeta_g", p.mets.gradzeta_g, o.gz), ("M", p.ops.mass.M, o.M)):
        log(f"{name} bit-equal: {bool(np.array_equal(a, b))}")
    t0 = time.time()
    ref_S = o.euler("2C").rhs_full(o.state)
    ref_H = o.hyper()
    ref = ref_S + ref_H
    log(f"oracle S + H_nu {time.time() - t0:.1f} s")
    for wf in ("", "0"):
        if wf:
            os.environ["HV_WFORM"] = wf
        ops = euler.EulerOps(p.m, p.mets, p.consts, "2C", hyper=(p.cfg, p.vm))
        plan = ops.lap_plan(p.vm)
        got = ops.rhs_full_hyper(state.StateField("2C", torch.from_numpy(o.state).cuda())).cpu().numpy()
        den = np.linalg.norm(ref)
        per = " ".join(f"{np.linalg.norm(got[:, f] - ref[:, f]) / den:.2e}" for f in range(5))
        err = rel_l2(got, ref)
        log(f"wform={plan.wform}: S+H_nu rel L2 vs oracle {err:.3e} (per field |diff_f|/|ref|: {per}) "
            f"-> {'PASS' if err <= 1e-12 else 'FAIL'} at 1e-12")
        S = ops.rhs_full(state.StateField("2C", torch.from_numpy(o.state).cuda())).cpu().numpy()
        log(f"wform={plan.wform}: S alone rel L2 {rel_l2(S, ref_S):.3e} (SURVEY A.3: conditioned at ~1e-10 on "
            f"this near-hydrostatic state)")
        os.environ.pop("HV_WFORM", None)
        del ops
        torch.cuda.empty_cache()
    if args.out:
        Path(args.out).write_text("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
