"""Time one LHEVI step (eager vs CUDA-graph replay) on a BASELINE mesh (dev helper).

python tools/time_lhevi.py c2 [ARK2]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import sys
from pathlib import Path

import numpy as np
import torch

import bench
from paper_2311_11425_b200 import euler, hyperdiff, state
from paper_2311_11425_b200.hevi import LheviGraph, LheviState, step_lhevi

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
tname = sys.argv[2] if len(sys.argv) > 2 else "ARK2"
z = np.load(Path(__file__).resolve().parents[1] / "tests" / "golden" / "lhevi.npz")


class Tab:
    pass


tab = Tab()
for f in ("A", "b", "c", "A_im", "b_im", "c_im"):
    setattr(tab, f, z[f"tab_{tname}_{f}"])
W = bench.build_workload(name, 0, 1)
m, mets = W["m"], W["mets"]
dt = 0.05
cfg = hyperdiff.HyperDiffConfig(alpha=2, c=(1e-4, 1e-4, 0.0))
vm = hyperdiff.build_viscous_metric(m, mets, cfg, dt=dt)
ops = euler.EulerOps(m, mets, state.PhysConstants(omega=0.0), "2C", hyper=(cfg, vm))
zc = m.xg[:, 2]
rho = 1.2 * np.exp(-zc / 8000.0)
rng = np.random.default_rng(3)
q0 = np.stack([rho, rho * 0.5 * rng.standard_normal(m.nglobal), rho * 0.5 * rng.standard_normal(m.nglobal),
               rho * 0.1 * rng.standard_normal(m.nglobal), rho * 300.0], axis=1)
q = torch.from_numpy(q0).cuda()
ls = LheviState(update_interval=1000)
for _ in range(2):
    step_lhevi(ops, tab, q, dt, ls)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
K = 5
e0.record()
for _ in range(K):
    step_lhevi(ops, tab, q, dt, ls)
e1.record()
torch.cuda.synchronize()
eager = e0.elapsed_time(e1) / K
g = LheviGraph(ops, tab, dt, ls, q)
for _ in range(2):
    g.step(q)
torch.cuda.synchronize()
e0.record()
for _ in range(K):
    g.step(q)
e1.record()
torch.cuda.synchronize()
graph = e0.elapsed_time(e1) / K
print(f"{name} {tname}: nglobal={m.nglobal} ncol={m.ncol} M={ops.Mdim} | LHEVI step eager {eager:.3f} ms, "
      f"graph replay {graph:.3f} ms (factorisation cached)")
