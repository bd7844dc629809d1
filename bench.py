#!/usr/bin/env python
"""Benchmark of the B200 H_nu (alpha=2) hot path -- BASELINE.json metric, one JSON line.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload c5|c2|c3]

Default workload (N=1): configuration 5 of BASELINE.json, the weak-scaled
config-2-style hyper-diffusion (alpha=2, N=4, fp64) with 128x128x32 elements
per GPU (x-slabs of the global (128*N)x128x32 perturbed box), the only
configuration BASELINE.json quotes at 1/2/4/8 GPUs; it fits one GPU and its
inputs (11.7 GB per op) exceed the 126 MB L2, so no flush is needed between
steps.  A "step" is one hyperdiffusion_apply over the full per-GPU state.

`value` = DOF-updates/s (4 diffused fields x global nodes / device time per
step, inputs resident in HBM); `e2e` = the same metric through the public API
with the state copied from pinned host memory and the result copied back
every step.  `roofline` relates the algorithmic bytes of the op (SURVEY.md
§8(d)) to its device time and the measured HBM copy bandwidth.
`--impl reference` times the reference algorithm's CPU port (oracle/, numpy,
single-threaded like the reference) on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured", d
    return 6650.0, "fallback", {}


def _dist():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled while the timed region runs."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.f = None

    def __enter__(self):
        try:
            self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=self.f, stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if self.proc is None or self.f is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.f.flush()
        rows = []
        for line in Path(self.f.name).read_text().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) != 7:
                continue
            try:
                rows.append((float(parts[0]), float(parts[1]), float(parts[2]), parts[3:]))
            except ValueError:
                continue
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i, v in enumerate(r[3]) if v.lower() == "active"})
        loaded = [r for r in rows if r[2] > 250.0] or rows
        return {"sm_mhz": statistics.median(r[0] for r in loaded), "sm_max_mhz": max(r[1] for r in rows),
                "power_w_max": max(r[2] for r in rows), "samples": len(rows), "reasons": reasons}


# ----------------------------------------------------------------- workloads
def algorithmic_bytes_hnu(ng, nloc, F=4, alpha=2, ncomp=6):
    """per pass 2*F*ng*8 (read q / write) + 6*nloc*8 (G_nu J w) + ng*8 (Minv) + nloc*4 (map).

    ncomp=3: the same count with the axis form of the metric the plane kernel reads instead of the
    6 components (u = sqrt(w3 Jg) e_3) -- the bytes this kernel actually needs."""
    return alpha * (2 * F * ng * 8 + ncomp * nloc * 8 + ng * 8 + nloc * 4)


def algorithmic_bytes_c4(ng, nloc):
    """SURVEY §8(d) Euler+H_nu: fused pass A (S and L pass 1) + pass B (L pass 2, accumulate)."""
    A = 5 * ng * 8 + 19 * nloc * 8 + ng * 8 + nloc * 4 + 5 * ng * 8 + 4 * ng * 8
    B = 4 * ng * 8 + 6 * nloc * 8 + ng * 8 + nloc * 4 + 2 * 4 * ng * 8
    return A + B


def flops_hnu(nelem, N, F=4, alpha=2):
    """per element per field per pass 2*(6 n^4 + 9 n^3) + n^3 FP64 operations."""
    n = N + 1
    return alpha * F * nelem * (2 * (6 * n ** 4 + 9 * n ** 3) + n ** 3)


def fp64_peak_tflops(reps=3):
    """Measured FP64 FMA throughput (hv_probe_dfma: 8 independent DFMA chains per thread, 148 x 8 CTAs
    of 256 threads), best of ``reps`` CUDA-event timings, TFLOP/s."""
    import torch

    from paper_2311_11425_b200 import _lib

    blocks, threads, iters = 148 * 8, 256, 4096
    out = torch.empty(blocks * threads, dtype=torch.float64, device="cuda")
    L = _lib.lib()
    run = lambda: _lib.check(L.hv_probe_dfma(out.data_ptr(), iters, blocks, threads,  # noqa: E731
                                             _lib.stream_handle()))
    run()
    torch.cuda.synchronize()
    best = None
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        best = ms if best is None else min(best, ms)
    return 2.0 * 8 * iters * blocks * threads / (best * 1e-3) / 1e12


def build_workload(name, rank, world, scale=1):
    from paper_2311_11425_b200 import euler, hyperdiff, metrics, state, synthetic

    w = synthetic.workload(name, scale=scale, slabs=1)
    t0 = time.time()
    m = synthetic.make_mesh(w)
    t_mesh = time.time() - t0
    mets = metrics.project_metrics_to_columns(metrics.curl_invariant_metrics(m), m)
    cfg = hyperdiff.HyperDiffConfig(alpha=w.alpha, c=w.c)
    vm = hyperdiff.build_viscous_metric(m, mets, cfg, dt=w.dt)
    ops = euler.EulerOps(m, mets, state.PhysConstants(omega=0.0), w.set_name, hyper=(cfg, vm))
    if w.operator == "euler+hyperdiff":
        ops.rhs_full_hyper(state.StateField(w.set_name, torch_zeros_state(m.nglobal)))
    import torch

    q = synthetic.make_state(w, m, device=torch.device("cuda"))
    return dict(w=w, m=m, mets=mets, cfg=cfg, vm=vm, ops=ops, q=q, t_mesh=t_mesh)


def torch_zeros_state(ng):
    import torch

    z = torch.zeros((ng, 5), dtype=torch.float64, device="cuda")
    z[:, 0] = 1.0
    z[:, 4] = 300.0
    return z


def time_secondary(name, steps=5, warmup=3):
    """Device time of one op of a secondary BASELINE config (same process, inputs resident)."""
    import torch

    from paper_2311_11425_b200 import hyperdiff, state

    P = build_workload(name, 0, 1)
    w, m, ops, vm, cfg = P["w"], P["m"], P["ops"], P["vm"], P["cfg"]
    n3 = (w.N + 1) ** 3
    qd = torch.from_numpy(P["q"]).cuda()
    out = torch.empty_like(qd)
    st = state.StateField(w.set_name, qd)
    if w.operator == "euler+hyperdiff":
        step = lambda: ops.rhs_full_hyper(st, out=out)  # noqa: E731
        alg = algorithmic_bytes_c4(m.nglobal, m.nelem * n3)
    elif w.operator == "laplacian":
        step = lambda: hyperdiff.laplacian_apply_fields(qd, vm, ops, (0, 1, 2, 3, 4))  # noqa: E731
        alg = algorithmic_bytes_hnu(m.nglobal, m.nelem * n3, F=5, alpha=1)
    else:
        step = lambda: hyperdiff.hyperdiffusion_apply(st, cfg, vm, ops, out=out)  # noqa: E731
        alg = algorithmic_bytes_hnu(m.nglobal, m.nelem * n3)
    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    peak, _, _ = _peaks()
    res = {"workload": f"{name}: {w.operator}, N={w.N}, nelem={m.nelem}, nglobal={m.nglobal}",
           "ms_per_op": ms, "dof_updates_per_s": w.fields_out * m.nglobal / (ms * 1e-3),
           "roofline_frac": alg / (ms * 1e-3) / 1e9 / peak, "algorithmic_bytes_per_op": alg}
    del P, ops, vm, qd, out
    torch.cuda.empty_cache()
    return res


def _cpu_problem(name, sx=16, sy=16):
    """The oracle problem of the CPU sample: an sx x sy column block (all layers, the same element
    size, geometry generator and state generator) of the workload's per-GPU mesh, set up with the
    ORACLE alone (KD-tree numbering, metrics, G_nu, mass: oracle/hevi_oracle.py restating
    mesh.py:86-145, metrics.py:79-142, hyperdiff.py:54-81, assembly.py:54-64); no product code or
    library is loaded on this path.  Returns (run, ng, description)."""
    from oracle import hevi_oracle as O
    from paper_2311_11425_b200 import synthetic   # input generators only (pure numpy)

    w = synthetic.workload(name)
    sx, sy = min(sx, w.nx or w.ne), min(sy, w.ny or w.ne)
    ext = (w.extents[0] * sx / w.nx, w.extents[1] * sy / w.ny, w.extents[2])
    coords, layer, hcol = synthetic.perturbed_box_coords(sx, sy, w.nv, w.N, ext, perturb=w.perturb)
    om = O.OracleMesh.from_coords("box", w.N, coords, layer, hcol, O.dedupe_tol("box", max(sx, sy), extents=ext))
    _, J, grad = O.curl_metrics(om)
    Jg, _ = O.project_columns(om, J, grad)
    _, Minv = O.lumped_mass(om, J)
    Gnu, _, _ = O.viscous_metric(om, grad, w.alpha, c=w.c, dt=w.dt)
    Jg_e = O.gather(om.gid, Jg)
    q = synthetic.fourier_state(om.xg, ext)
    run = lambda: O.hyperdiffusion(om, Gnu, Jg_e, Minv, q, w.alpha)  # noqa: E731
    return run, om.ng, f"{sx}x{sy}x{w.nv} element column block of {name} (N={w.N}, ng={om.ng})"


def _cpu_worker(name, warmup, steps, barrier, out):
    os.environ["OMP_NUM_THREADS"] = os.environ["OPENBLAS_NUM_THREADS"] = "1"
    sys.path.insert(0, str(ROOT))
    run, ng, desc = _cpu_problem(name)
    for _ in range(warmup):
        run()
    barrier.wait()
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        run()
        times.append(time.perf_counter() - t0)
    out.put((times, ng, desc))


def cpu_sample(name, warmup=1, steps=3, procs=None):
    """The reference algorithm (oracle port, numpy) on a bounded sample of the workload.

    The reference is serial (numpy einsum / add.at, GIL-bound); to use every host core, ``procs``
    worker processes each run one copy of the sample concurrently (independent problems, like an
    ensemble).  A step = one H_nu op on the sample in every worker; the step time is the slowest
    worker's.  Returns dict(value DOF-updates/s, ms_per_step, step_times, ng, cores, sample)."""
    import multiprocessing as mp

    procs = procs or max(1, len(os.sched_getaffinity(0)))
    ctx = mp.get_context("spawn")
    barrier = ctx.Barrier(procs)
    out = ctx.Queue()
    ps = [ctx.Process(target=_cpu_worker, args=(name, warmup, steps, barrier, out)) for _ in range(procs)]
    for p in ps:
        p.start()
    res = [out.get(timeout=1800) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    ng, desc = res[0][1], res[0][2]
    step_s = [max(r[0][k] for r in res) for k in range(steps)]      # slowest worker per step
    total = sum(step_s)
    value = 4 * ng * procs * steps / total
    desc = (f"{desc}: one H_nu op per step in each of {procs} concurrent single-thread worker processes "
            f"(oracle port of the reference, numpy); {warmup} warm-up + {steps} timed ops; setup untimed")
    return dict(value=value, ms_per_step=1e3 * total / steps, step_times=step_s, ng=ng, cores=procs, sample=desc)


# ---------------------------------------------------------------------- arms
def bench_config(w, world):
    """The `config` object of both arms (identical: the same workload; sample sizes and per-GPU
    node counts live outside it)."""
    return {"workload": f"{w.name}: H_nu alpha=2, {w.nx}x{w.ny}x{w.nv} elem/GPU, N={w.N}, "
                        f"perturbed box, c={w.c}, dt={w.dt}",
            "fields": 4, "l2": "inputs (11.7 GB/op) exceed L2; no flush",
            "parallelism": (f"x-slabs x{world} of a ({w.nx}*{world})x{w.ny}x{w.nv} box, slab-face "
                            "DSS over NCCL p2p" if world > 1 else "single GPU")}


def run_reference(args, rank, world):
    """The reference's CPU algorithm on the host cores (oracle port; the reference package itself
    does not exist on the GPU box).  Rank 0 only; a step = one H_nu op on a bounded column-block
    sample of the workload in each worker process."""
    if rank != 0:
        return
    from paper_2311_11425_b200 import synthetic

    w = synthetic.workload(args.workload)
    one = cpu_sample(args.workload, warmup=1, steps=2, procs=1)          # the single-core rate
    r = cpu_sample(args.workload, warmup=max(1, args.warmup), steps=args.steps)
    line = {
        "impl": "reference",
        "metric": "fp64 DOF-updates/s of H_nu (alpha=2)",
        "value": r["value"],
        "unit": "DOF-updates/s",
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": max(1, args.warmup),
        "ms_per_step": r["ms_per_step"],
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded, host-generated geometry; Fourier state)",
        "config": bench_config(w, world),
        "cpu_baseline": {"value": r["value"], "unit": "DOF-updates/s", "cores": r["cores"], "kind": "port",
                         "sample": r["sample"], "value_1core": one["value"],
                         "host_cpu": _host_cpu()},
        "e2e": {"value": r["value"], "unit": "DOF-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _host_cpu():
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def run_ours(args, rank, world, local):
    import torch

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2311_11425_b200 import _lib, hyperdiff, state

    stream = torch.cuda.current_stream()
    if world > 1:
        # config 5 proper: x-slab of the global (128*world) x 128 x 32 box per rank, slab-face
        # DSS exchanged with the neighbours over NCCL (parallel.py)
        from paper_2311_11425_b200 import parallel, synthetic

        w = synthetic.workload(args.workload)
        if args.workload != "c5":
            raise SystemExit("multi-GPU runs are defined for the weak-scaled config 5")
        t0 = time.time()
        layout = parallel.SlabLayout(rank, world, w.nx, w.ny, w.nv, w.N)
        cfg = hyperdiff.HyperDiffConfig(alpha=w.alpha, c=w.c)
        transport = parallel.DistTransport(rank, world)
        sop = parallel.setup_distributed(layout, cfg, w.dt, transport)
        m, vm, ops = sop.mesh, sop.vm, sop.ops
        # white noise keyed on the global lattice node, so the slab-face nodes two ranks share hold
        # the same state on both (the smooth part depends on the bitwise-shared coordinates only)
        q_host = synthetic.fourier_state(m.xg, layout.extents, device=torch.device("cuda"),
                                         noise_keys=layout.lattice_keys(m))
        P = dict(w=w, m=m, q=q_host, t_mesh=time.time() - t0)

        def hyperdiffusion_apply(st_, cfg_, vm_, ops_, out=None):
            return sop.apply(st_.data, out, transport)
    else:
        P = build_workload(args.workload, rank, world)
        hyperdiffusion_apply = hyperdiff.hyperdiffusion_apply
    w, m = P["w"], P["m"]
    ops, vm, cfg = (P["ops"], P["vm"], P["cfg"]) if world == 1 else (ops, vm, cfg)
    ng, nloc = m.nglobal, m.nelem * (w.N + 1) ** 3
    qd = torch.from_numpy(P["q"]).cuda()
    out = torch.empty_like(qd)
    st = state.StateField("2C", qd)

    def step():
        hyperdiffusion_apply(st, cfg, vm, ops, out=out)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    L = _lib.lib()
    n0 = L.hv_launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
    launches = L.hv_launch_count() - n0
    ms = ev0.elapsed_time(ev1) / args.steps
    if dist:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    if world > 1:
        import torch.distributed as dist_

        t = torch.tensor([ng], dtype=torch.float64, device="cuda")
        dist_.all_reduce(t)
        # interface column nodes are counted once: subtract the duplicated slab faces
        dup = (world - 1) * (w.ny * w.N + 1) * m.n_z
        dof = 4 * (int(t.item()) - dup)
    else:
        dof = 4 * ng
    value = dof / (ms * 1e-3)

    # end to end through the public API: every step copies its input state from pinned host
    # memory and reads its result back to pinned host memory.  Steps are software-pipelined on
    # three streams (H2D of step k+1 and D2H of step k-1 overlap the operator of step k; PCIe
    # is full duplex), with double-buffered device inputs / outputs.
    h_in = torch.empty((ng, 5), dtype=torch.float64, pin_memory=True)
    h_in.copy_(torch.from_numpy(P["q"]))
    h_out = [torch.empty_like(h_in, pin_memory=True) for _ in range(2)]
    d_in = [torch.empty_like(qd) for _ in range(2)]
    d_out = [out, torch.empty_like(qd)]
    s_in, s_cmp, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_cmp = [torch.cuda.Event() for _ in range(2)]
    ev_out = [torch.cuda.Event() for _ in range(2)]

    def e2e_run(k_steps, e_start, e_end):
        s_in.wait_stream(stream)
        e_start.record(s_in)
        for k in range(k_steps):
            b = k % 2
            with torch.cuda.stream(s_in):
                if k >= 2:
                    s_in.wait_event(ev_cmp[b])            # d_in[b] consumed by step k-2
                d_in[b].copy_(h_in, non_blocking=True)
                ev_in[b].record(s_in)
            with torch.cuda.stream(s_cmp):
                s_cmp.wait_event(ev_in[b])
                if k >= 2:
                    s_cmp.wait_event(ev_out[b])           # d_out[b] read back by step k-2
                hyperdiffusion_apply(state.StateField("2C", d_in[b]), cfg, vm, ops, out=d_out[b])
                ev_cmp[b].record(s_cmp)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_cmp[b])
                h_out[b].copy_(d_out[b], non_blocking=True)
                ev_out[b].record(s_out)
        s_out.wait_stream(s_in)
        s_out.wait_stream(s_cmp)
        e_end.record(s_out)

    e2e_run(2, torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    torch.cuda.synchronize()
    ke = max(3, min(args.steps, 10))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2e_run(ke, e0, e1)
    torch.cuda.synchronize()
    ms_e2e = e0.elapsed_time(e1) / ke
    if dist:
        t = torch.tensor([ms_e2e], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_e2e = float(t.item())

    peak, peak_kind, _ = _peaks()
    alg = algorithmic_bytes_hnu(ng, nloc)
    achieved_op = alg / (ms * 1e-3) / 1e9
    # dominant kernel alone: the tile sweep of one pass (pass 1, q -> L q), CUDA events on its stream
    kern_ms, kern_name, traffic, wform, pass_ms, traffic_src = None, None, None, 0, {}, None
    fix_ms, yt_mode = {}, False
    if world == 1 and getattr(ops, "_plans", None):
        import ctypes as C

        plan = ops.lap_plan(vm)
        if plan.d_gt:
            nv_ = len(cfg.variables)
            va = (C.c_int32 * nv_)(*cfg.variables)
            L = _lib.lib()
            out5 = torch.empty((ng, 5), dtype=torch.float64, device="cuda")

            # one kernel of the op at a time through hv_hyperdiffusion_stage (the op's own launches, the
            # op's own buffers): stage 1 = pass-1 sweep, 3 = pass-2 sweep, 2 / 4 = their fix-ups
            def one_stage(k):
                _lib.check(L.hv_hyperdiffusion_stage(C.byref(plan), qd.data_ptr(), 5, nv_, va, out5.data_ptr(), 5, k,
                                                     _lib.stream_handle()))

            nk = max(5, args.steps)
            pass_ms = {}
            for k in (1, 2, 3, 4):
                for _ in range(3):
                    for kk in (1, 2, 3, 4):   # keep the intermediate of a whole op in place
                        one_stage(kk)
                torch.cuda.synchronize()
                k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                k0.record(stream)
                for _ in range(nk):
                    one_stage(k)
                k1.record(stream)
                torch.cuda.synchronize()
                pass_ms[k] = k0.elapsed_time(k1) / nk
            fix_ms = {1: pass_ms.pop(2), 2: pass_ms.pop(4)}
            pass_ms = {1: pass_ms[1], 2: pass_ms[3]}
            kern_ms = 0.5 * (pass_ms[1] + pass_ms[2])      # average launch of the dominant kernel
            kern_name = "lap_plane_kernel" if plan.kernel == 1 else "lap_tile_kernel"
            wform = int(plan.wform)
            prof = ROOT / "profiles" / "r02_dominant_kernel.json"
            if not prof.exists():
                prof = ROOT / "profiles" / "r01_dominant_kernel.json"
            if prof.exists():
                traffic = json.loads(prof.read_text()).get("dram_bytes_per_launch")
                traffic_src = str(prof.relative_to(ROOT))
            yt_mode = bool(plan.d_yt)
            del out5
    alg_launch = alg / 2                       # one pass = one sweep launch
    achieved = alg_launch / (kern_ms * 1e-3) / 1e9 if kern_ms else achieved_op
    # what the kernel must move with its metric form (axis form: 3 of the 6 metric doubles)
    own_launch = algorithmic_bytes_hnu(ng, nloc, ncomp=3 if wform == 1 else 6) / 2
    own_achieved = own_launch / (kern_ms * 1e-3) / 1e9 if kern_ms else None
    fp64 = None
    if world == 1:
        pk = fp64_peak_tflops()
        fl_launch = flops_hnu(m.nelem, w.N) / 2
        ach = fl_launch / (kern_ms * 1e-3) / 1e12 if kern_ms else None
        fp64 = {"peak_tflops": pk, "peak_kind": "measured (hv_probe_dfma, DFMA chains, best of 3)",
                "flops_per_op": flops_hnu(m.nelem, w.N), "flops_per_launch": fl_launch,
                "kernel_achieved_tflops": ach, "kernel_frac": (ach / pk) if ach else None,
                "op_achieved_tflops": flops_hnu(m.nelem, w.N) / (ms * 1e-3) / 1e12,
                "arithmetic_intensity_flop_per_byte": flops_hnu(m.nelem, w.N) / alg,
                "ridge_flop_per_byte": pk * 1e3 / peak}
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu:
            r = cpu_sample(args.workload, warmup=1, steps=4)
            cpu = {"value": r["value"], "unit": "DOF-updates/s", "cores": r["cores"], "kind": "port",
                   "sample": r["sample"], "host_cpu": _host_cpu()}
        line = {
            "metric": "fp64 DOF-updates/s of H_nu (alpha=2)",
            "value": value,
            "unit": "DOF-updates/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": max(3, args.warmup),
            "ms_per_step": ms,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (seeded, host-generated geometry; Fourier state)",
            "config": bench_config(w, world),
            "workload_size": {"nglobal_per_gpu": ng, "nelem_per_gpu": m.nelem},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "peak_kind": peak_kind, "traffic": traffic,
                         "kernel": kern_name, "kernel_ms_per_launch": kern_ms,
                         "kernel_ms_pass1": pass_ms.get(1), "kernel_ms_pass2": pass_ms.get(2),
                         "fixup_ms_pass1": fix_ms.get(1), "fixup_ms_pass2": fix_ms.get(2),
                         "intermediate": ("tile-ordered blocks (pass 1 writes L q in the sweep's block layout, "
                                          "pass 2 bulk-copies it)") if yt_mode else "(nglobal, 4) rows",
                         "algorithmic_bytes_per_launch": alg_launch, "algorithmic_bytes_per_op": alg,
                         "op_achieved": achieved_op, "op_frac": achieved_op / peak,
                         "kernel_share_of_step": (2 * kern_ms / ms) if kern_ms else None,
                         "metric_form": "axis (3 doubles per element node)" if wform == 1 else "6 components",
                         "kernel_form_bytes_per_launch": own_launch,
                         "kernel_form_achieved": own_achieved,
                         "kernel_form_frac": (own_achieved / peak) if own_achieved else None,
                         "scope": "dominant kernel = tile sweep of one Laplacian pass (2 per H_nu op), "
                                  "kernel_ms_per_launch = mean of the pass-1 and pass-2 launches, each timed alone "
                                  "through hv_hyperdiffusion_stage (CUDA events on the launching stream, the op's "
                                  "own buffers); achieved/frac use SURVEY 8(d)'s bytes (6 metric doubles "
                                  "per element node); kernel_form_* the bytes of the metric form the kernel reads; "
                                  "op_* = whole op incl. perimeter fix-ups; traffic = ncu dram bytes per launch "
                                  f"from one ncu --set full capture ({traffic_src})"},
            "fp64": fp64,
            "cpu_baseline": cpu,
            "e2e": {"value": dof / (ms_e2e * 1e-3), "unit": "DOF-updates/s",
                    "h2d_bytes_per_step": ng * 5 * 8, "d2h_bytes_per_step": ng * 5 * 8,
                    "ms_per_step": ms_e2e, "steps": ke,
                    "how": "public API hyperdiffusion_apply; pinned H2D of the (ng,5) state and D2H of the "
                           "(ng,5) result every step, 3-stream software pipeline across steps"},
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
            "setup_s": {"mesh": round(P["t_mesh"], 2)},
        }
        if world == 1 and not args.no_extras:
            line["secondary"] = {}
            del P, ops, vm, qd, out, st, d_in, d_out, h_in, h_out
            torch.cuda.empty_cache()
            for name in ("c1", "c2", "c3", "c4"):
                try:
                    line["secondary"][name] = time_secondary(name)
                except Exception as exc:  # a failing secondary config must not hide the headline
                    line["secondary"][name] = {"error": repr(exc)[:300]}
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    # the headline line is config 5 (the only config quoted at 1/2/4/8 GPUs); configs 1-4 are timed
    # into the line's "secondary" object (tools/time_secondary.py runs one of them alone)
    ap.add_argument("--workload", default="c5", choices=["c5"])
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the secondary configs c1-c4")
    args = ap.parse_args()
    rank, world, local = _dist()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
