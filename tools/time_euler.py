"""Time the c4 Euler column sweep alone (rhs_full on the c4 state; dev helper): python tools/time_euler.py [steps]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import bench
from paper_2311_11425_b200 import state

K = int(sys.argv[1]) if len(sys.argv) > 1 else 10
P = bench.build_workload("c4", 0, 1)
ops = P["ops"]
qd = torch.from_numpy(P["q"]).cuda()
st = state.StateField("2C", qd)
out = torch.empty_like(qd)
for _ in range(3):
    ops.rhs_full(st, out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(K):
    ops.rhs_full(st, out=out)
e1.record()
torch.cuda.synchronize()
print(f"c4 rhs_full: {e0.elapsed_time(e1) / K:.4f} ms/op", flush=True)
