"""Time the c5 sweep kernel (one Laplacian pass, hv_lap_local) per HV_PLANE_VARIANT (dev helper).

python tools/time_plane.py 0 1 2 3 4   -> ms per launch for each variant and max |diff| vs the first
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import ctypes as C
import os
import sys

import torch

import bench
from paper_2311_11425_b200 import _lib

W = bench.build_workload(os.environ.get("HV_WORKLOAD", "c5"), 0, 1)
ops, vm, cfg, q = W["ops"], W["vm"], W["cfg"], W["q"]
if not torch.is_tensor(q):
    q = q.data if hasattr(q, "data") and torch.is_tensor(getattr(q, "data")) else q
if not torch.is_tensor(q):
    import numpy as np
    q = torch.from_numpy(np.ascontiguousarray(q))
q = q.cuda()
plan = ops.lap_plan(vm)
ng = W["m"].nglobal
nv = len(cfg.variables)
qa = (C.c_int32 * nv)(*cfg.variables)
oa = (C.c_int32 * nv)(*range(nv))
L = _lib.lib()
st = _lib.stream_handle()
ref = None
# HV_PASS=2: the second pass of H_nu (y (ng, 4) in, (ng, 5) rows out with column 0 zeroed, scale -1)
pass2 = os.environ.get("HV_PASS", "1") == "2"
if pass2:
    q = q[:, 1:5].contiguous()
    qa = (C.c_int32 * nv)(*range(nv))
    oa = (C.c_int32 * nv)(*cfg.variables)
for v in sys.argv[1:]:
    os.environ["HV_PLANE_VARIANT"] = v
    y = torch.zeros((ng, 5 if pass2 else nv), dtype=torch.float64, device="cuda")

    def one():
        if pass2:
            _lib.check(L.hv_lap_local(C.byref(plan), q.data_ptr(), nv, nv, qa, y.data_ptr(), 5, oa, -1.0, 1, 0, st))
        else:
            _lib.check(L.hv_lap_local(C.byref(plan), q.data_ptr(), 5, nv, qa, y.data_ptr(), nv, oa, 1.0, 0, 0, st))

    for _ in range(3):
        one()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        one()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    d = None if ref is None else float((y - ref).abs().max() / ref.abs().max())
    if ref is None:
        ref = y.clone()
    alg = bench.algorithmic_bytes_hnu(ng, W["m"].nelem * (W["m"].cfg.degree + 1) ** 3) / 2
    print(f"variant {v}: {ms:.4f} ms  {alg / ms / 1e6:.0f} GB/s  ({alg / ms / 1e6 / 6540.2 * 100:.1f}% of 6540)  diff {d}",
          flush=True)
