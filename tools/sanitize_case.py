"""Small end-to-end run of every device kernel for compute-sanitizer (dev helper)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import sys

import numpy as np
import torch

sys.path.insert(0, "tests")
from cases import random_state  # noqa: E402
from product_cases import ProductProblem  # noqa: E402
from paper_2311_11425_b200 import euler, hyperdiff, parallel, state  # noqa: E402

for name in ("box_p_n4", "sphere_n4", "box_n7"):
    p = ProductProblem(name)
    st = state.StateField("2C", random_state(p.m.nglobal, "2C"))
    hyperdiff.hyperdiffusion_apply(st, p.cfg, p.vm, p.ops)
    hyperdiff.laplacian_apply(st.data[:, 1], p.vm, p.ops)
    hyperdiff.laplacian_apply_fields(st.data, p.vm, p.ops, (0, 1, 2, 3, 4))
    for s in ("2NC", "2C", "3C"):
        o = euler.EulerOps(p.m, p.mets, p.consts, s, hyper=(p.cfg, p.vm))
        o.rhs_full(state.StateField(s, random_state(p.m.nglobal, s)))
        o.rhs_horizontal(state.StateField(s, random_state(p.m.nglobal, s)))
        o.rhs_vertical(state.StateField(s, random_state(p.m.nglobal, s)))
        o.diagnostics(state.StateField(s, random_state(p.m.nglobal, s)))
    # LHEVI column systems: Jacobian band, block band LU, solve
    from paper_2311_11425_b200 import linalg
    q = torch.from_numpy(random_state(p.m.nglobal, "2C")).cuda()
    cg = torch.from_numpy(p.m.col_gid.astype(np.int64)).cuda()
    band = p.ops.column_jacobian(q[cg].contiguous(), 0.37)
    ipiv, _ = linalg.banded_lu_factor_batch(band, p.ops.kl, p.ops.ku)
    rhs = torch.randn((p.m.ncol, p.ops.Mdim), dtype=torch.float64, device="cuda")
    linalg.banded_solve_batch(band, ipiv, p.ops.kl, p.ops.ku, rhs)
layouts = [parallel.SlabLayout(r, 2, 2, 2, 2, 4, elem_size=(100.0, 120.0, 50.0)) for r in range(2)]
ops = parallel.setup_loopback(layouts, hyperdiff.HyperDiffConfig(alpha=2, c=(0.05, 0.05, 0.0)), 0.5)
qs = [torch.randn((op.mesh.nglobal, 5), dtype=torch.float64, device="cuda") for op in ops]
parallel.run_loopback(ops, qs, [torch.empty_like(q) for q in qs])
torch.cuda.synchronize()
print("sanitize case done")
