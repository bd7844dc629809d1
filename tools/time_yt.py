"""Time H_nu (alpha=2) per op with the tile-ordered intermediate (HV_YT=1, default) against the
(nglobal, 4) intermediate (HV_YT=0), same workload and state; checks bitwise equality (dev helper).

python tools/time_yt.py [c5|c2|c3]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import os

import torch

import bench
from paper_2311_11425_b200 import euler, hyperdiff, state

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 20
WU = 3 if K >= 5 else 1
P = bench.build_workload(name, 0, 1)
m, mets, cfg, vm, ops = P["m"], P["mets"], P["cfg"], P["vm"], P["ops"]
qd = torch.from_numpy(P["q"]).cuda()
os.environ["HV_YT"] = "0"
ops0 = euler.EulerOps(m, mets, ops.c, "2C", hyper=(cfg, vm))
ops0.lap_plan(vm)
del os.environ["HV_YT"]
st = state.StateField("2C", qd)
res = {}
for tag, o in ((("yt", ops), ("rows", ops0)) * (2 if K >= 5 else 1)):
    out = torch.empty_like(qd)
    for _ in range(WU):
        hyperdiff.hyperdiffusion_apply(st, cfg, vm, o, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(K):
        hyperdiff.hyperdiffusion_apply(st, cfg, vm, o, out=out)
    e1.record()
    torch.cuda.synchronize()
    print(f"{name} {tag}: {e0.elapsed_time(e1) / K:.4f} ms/op (plan d_yt={bool(o.lap_plan(vm).d_yt)})", flush=True)
    res[tag] = out.clone()
print("bitwise equal:", bool(torch.equal(res["yt"], res["rows"])))
