"""Time the LHEVI column-system path (Jacobian band + band LU + one solve) on a BASELINE mesh (dev helper).

python tools/time_column.py c2 [ncol]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import sys
import time

import numpy as np
import torch

import bench
from paper_2311_11425_b200 import linalg

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
W = bench.build_workload(name, 0, 1)
ops, m = W["ops"], W["m"]
# physical column state (the H_nu benchmark state is not a valid 2C state): stratified
# density, small random momenta, potential temperature 300 K
z = m.xg[:, 2]
rng = np.random.default_rng(3)
rho = 1.2 * np.exp(-z / 8000.0)
qh = np.stack([rho, 0.5 * rng.standard_normal(m.nglobal), 0.5 * rng.standard_normal(m.nglobal),
               0.1 * rng.standard_normal(m.nglobal), rho * 300.0], axis=1)
q = torch.from_numpy(qh).cuda()
ncol = min(int(sys.argv[2]) if len(sys.argv) > 2 else m.ncol, m.ncol)
cg = torch.from_numpy(m.col_gid[:ncol].astype(np.int64)).cuda()
qcol = q[cg].contiguous()
lam = 0.37
rhs = torch.randn((ncol, ops.Mdim), dtype=torch.float64, device="cuda")
for _ in range(2):
    band = ops.column_jacobian(qcol, lam)
    ipiv, _ = linalg.banded_lu_factor_batch(band, ops.kl, ops.ku)
    x, _ = linalg.banded_solve_batch(band, ipiv, ops.kl, ops.ku, rhs)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
ev[0].record()
band = ops.column_jacobian(qcol, lam)
ev[1].record()
ipiv, _ = linalg.banded_lu_factor_batch(band, ops.kl, ops.ku)
ev[2].record()
x, _ = linalg.banded_solve_batch(band, ipiv, ops.kl, ops.ku, rhs)
ev[3].record()
torch.cuda.synchronize()
t = [ev[i].elapsed_time(ev[i + 1]) for i in range(3)]
gb = band.numel() * 8 / 1e9
print(f"{name}: ncol={ncol} M={ops.Mdim} kl={ops.kl} band {gb:.2f} GB | jacobian {t[0]:.3f} ms "
      f"({gb / t[0] * 1e3:.0f} GB/s write) | LU {t[1]:.3f} ms ({2 * gb / t[1] * 1e3:.0f} GB/s r+w) | "
      f"solve {t[2]:.3f} ms ({gb / t[2] * 1e3:.0f} GB/s read)")
