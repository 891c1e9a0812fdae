"""Benchmark: BASELINE config 5 -- the mode-scaling sweep on the 8 M-tet jittered pipe, 128 modes.

Workload (BASELINE.json configs[4], the largest config that fits one GPU): 8 004 150 tets,
n = 32 937 682 reduced DOFs, nnz = 1 405 049 508, rho = 1.06, mu = 0.04, parabolic Dirichlet inlet
x Q_n with q_n ~ (N + iN)/(1 + n^2) (seed 5), modes 0..127, complex128.  At restart 200 one mode's
Krylov basis is 106 GB, so one mode at a time runs per GPU.

A step is one pass of the hot path for one mode on every GPU: the mode's right-hand side is
assembled on the device and one full restarted-GMRES cycle runs (restart 200: 200 inner iterations
of SpMV + CGS2 + Givens, then the triangular solve, x update and true residual), from x0 = 0.
Rank r walks its LPT shard of the 128 modes (plan by expected iterations); config 5 cannot be
converged at 1e-10 inside a benchmark, so the rate is GMRES mode-iterations per
second.  Measured 3D modes solved/s come from the down-scaled pipes solved to 1e-10 in the same run
(`c3d_converged`) and the 2D config 1 (`c1_converged`).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--workload c5|c4|c3|c2]

Multi-GPU (torchrun, one rank per GPU): weak scaling -- every rank runs one mode-cycle per step
from its shard, no data-path collective; in the end-to-end leg the solved modal fields of every
step are gathered to rank 0 with the library's NCCL communicator (ss_comm_gather_modes).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

os.environ.setdefault("OMP_NUM_THREADS", "1")
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("MKL_NUM_THREADS", "1")

import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Fourier modes solved/sec (3D mesh); batched complex SpMV HBM GB/s vs peak"
UNIT = "GMRES mode-iterations/s"
RESTART = 200
BUDGET = 200           # inner iterations per mode per step (one restart cycle)
TOL = 1e-10
STRATA = (0, 50, 100, 150, 199)

# The workloads' identity (checked against the built operator in the B200 arm, so both arms print
# the same config dict).
WORKLOADS = {
    "c5": dict(workload="c5_pipe_8004150tets", n_dofs=32937682, nnz=1405049508, total_modes=128,
               modes_per_gpu_per_step=1, slab_layers=9),
    "c2": dict(workload="c2_pipe_199800tets", n_dofs=796978, nnz=32911596, total_modes=17,
               modes_per_gpu_per_step=17, slab_layers=None),
    "c3": dict(workload="c3_bend_2059200tets", n_dofs=8394503, nnz=354820086, total_modes=64,
               modes_per_gpu_per_step=6, slab_layers=None),
    "c4": dict(workload="c4_yjunction_4960116tets", n_dofs=20208154, nnz=854029473, total_modes=32,
               modes_per_gpu_per_step=2, slab_layers=None),
}


def config_dict(key):
    w = WORKLOADS[key]
    return {"workload": w["workload"], "total_modes": w["total_modes"],
            "modes_per_gpu_per_step": w["modes_per_gpu_per_step"], "n_dofs": w["n_dofs"], "nnz": w["nnz"],
            "restart": RESTART, "iterations_per_mode_per_step": BUDGET, "tol": TOL, "x0": "zero",
            "mode_plan": "LPT over expected iterations (distributed.expected_iterations, 3D model); "
                         "rank r runs plan[r][step % len(plan[r])]",
            "l2": "inputs larger than L2 (Krylov basis 201 x n x 16 B per mode >> 126 MB)"}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region (B200_PROFILING.md)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int, rank: int = None):
        self.gpu = gpu_index
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_rank{gpu_index if rank is None else rank}.csv")

    def __enter__(self):
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.fh.close()

    def summary(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as fh:
            for line in fh:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sm.append(float(parts[1]))
                    smax.append(float(parts[2]))
                except ValueError:
                    continue
                for nm, val in zip(names, parts[5:9]):
                    if val.lower() == "active":
                        reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------------------------------------
# CPU legs: the oracle port of the reference (test infrastructure, never the product path)
# ------------------------------------------------------------------------------------------------

def _oracle_case(key):
    """The CPU sample of a workload: config 2 itself; a 9-layer slab of config 5; for configs 3 and 4
    a down-scaled instance of the same generator (per-DOF work scaled by n, like the slab)."""
    from paper_2009_06725_b200.workloads import c2_case, c3_case, c4_case, c5_slab

    if key == "c5":
        return c5_slab(WORKLOADS[key]["slab_layers"])
    if key == "c3":
        return c3_case(6)
    if key == "c4":
        return c4_case(6)
    return c2_case()


_CACHE = {}


def _oracle_cycle_seconds(key, mode, seed=0):
    """Seconds of one 200-iteration restart cycle of the oracle port (krylov.py:63-164): the exact
    inner-iteration code path timed at basis indices STRATA (cycle-average), times 200, plus the
    cycle-end/next-start path (triangular solve, x += yQ, true residual, restart residual), scaled
    from the sample to the workload's n.  The sample system is assembled once per process and mode.
    Returns (seconds per cycle at the workload's size, detail)."""
    import oracle

    t_asm = 0.0
    if (key, mode) not in _CACHE:
        case = _oracle_case(key)
        t0 = time.perf_counter()
        s = oracle.assemble_mode_system(case.qmesh, case.density, case.viscosity, case.omegas[mode],
                                        g_mode=case.coefficients[mode] * case.profile)
        t_asm = time.perf_counter() - t0
        _CACHE[(key, mode)] = (s, oracle.jacobi_scale(s.matrix), case.name)
    s, sc, name = _CACHE[(key, mode)]
    n_sample = s.matrix.shape[0]
    scale = WORKLOADS[key]["n_dofs"] / n_sample
    rng = np.random.default_rng(1000 * seed + mode)
    costs = [oracle.gmres_inner_step_cost(s.matrix, sc, k, RESTART, rng) for k in STRATA]
    t_end = oracle.gmres_cycle_end_cost(s.matrix, s.rhs, sc, RESTART, rng)
    cycle = (float(np.mean(costs)) * BUDGET + t_end) * scale
    return cycle, dict(n_sample=n_sample, nnz_sample=int(s.matrix.nnz), scale=scale, costs=costs, t_end=t_end,
                       t_assembly=t_asm, sample=name)


def _cpu_sample_text(key, det, procs):
    base = (f"oracle port of krylov.py:63-164 (numpy/scipy, 1 BLAS thread per process): the exact inner-"
            f"iteration code path timed at basis indices {list(STRATA)} of a restart-200 cycle (x200) plus the "
            f"cycle-end path, on {det['sample']} (n = {det['n_sample']}")
    if key == "c5":
        base += (f", a 9-layer slab of config 5 with its cross-section, spacing and jitter), scaled by "
                 f"n_c5/n_slab = {det['scale']:.2f} (per-iteration work is linear in n)")
    elif key in ("c3", "c4"):
        base += (f", a down-scaled instance of the config-{key[1]} generator), scaled by n/n_sample = "
                 f"{det['scale']:.2f} (per-iteration work is linear in n)")
    else:
        base += ")"
    return base + f"; {procs} process(es); per-mode oracle assembly ({det['t_assembly']:.1f} s on the sample) " \
                  f"is once per mode, not per cycle, and is excluded"


def _ref_worker(args):
    os.environ["OMP_NUM_THREADS"] = "1"
    key, mode, steps = args
    out = []
    for st in range(steps):
        t0 = time.perf_counter()
        cyc, det = _oracle_cycle_seconds(key, mode, seed=st)
        out.append((cyc, time.perf_counter() - t0, det))
    return out


def run_reference(args):
    """--impl reference: the reference's CPU path (the oracle port: the reference is pure Python and
    cannot travel to the box) on all usable host cores, one process per mode."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import multiprocessing as mp

    try:
        import psutil
        avail_gb = psutil.virtual_memory().available / 2 ** 30
    except Exception:
        avail_gb = 64.0
    cores = len(os.sched_getaffinity(0))
    # one process needs ~6 GB at the c5 slab / c2 size (basis sample + matrix + assembly peak)
    procs = max(1, min(cores, WORKLOADS[args.workload]["total_modes"], int(avail_gb // 6)))
    steps = args.steps + args.warmup
    t0 = time.perf_counter()
    ctx = mp.get_context("spawn")
    with ctx.Pool(procs) as pool:
        res = pool.map(_ref_worker, [(args.workload, 1 + (m % (WORKLOADS[args.workload]["total_modes"] - 1)), steps)
                                     for m in range(procs)])
    wall = time.perf_counter() - t0
    timed = [r[args.warmup:] for r in res]
    # every process runs cycles of its own mode concurrently: throughput = sum over processes
    per_step = [sum(BUDGET / timed[p][s][0] for p in range(procs)) for s in range(args.steps)]
    value = float(np.mean(per_step))
    ms_step = 1e3 * float(np.mean([max(timed[p][s][1] for p in range(procs)) for s in range(args.steps)]))
    det = res[0][0][2]
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "c128",
        "data": f"synthetic (seeded, BASELINE config {args.workload[1]})",
        "config": config_dict(args.workload),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": procs, "kind": "port",
                         "sample": _cpu_sample_text(args.workload, det, procs) + "; value = sum over processes of "
                                   "200 / (seconds per cycle)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "host_cores": cores, "wall_s": wall, "sample_s_per_step": ms_step / 1e3,
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------------
# B200 arm
# ------------------------------------------------------------------------------------------------

def _setup_workload(key, world, rank):
    from paper_2009_06725_b200 import FluidProps
    from paper_2009_06725_b200.assembly import get_operator
    from paper_2009_06725_b200.distributed import expected_iterations, lpt_shard
    from paper_2009_06725_b200.workloads import c2_case, c3_case, c4_case, c5_case

    case = {"c2": c2_case, "c3": c3_case, "c4": c4_case, "c5": c5_case}[key]()
    q = case.qmesh
    props = FluidProps(case.density, case.viscosity)
    op = get_operator(q, props)
    w = WORKLOADS[key]
    if (op.n, op.nnz, case.name) != (w["n_dofs"], w["nnz"], w["workload"]):
        raise RuntimeError(f"workload mismatch: {(op.n, op.nnz, case.name)} != {w}")
    n_total = w["total_modes"]
    plan = lpt_shard(expected_iterations(np.arange(n_total), 3), world)
    return case, q, props, op, plan


def run_b200(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # Code-path check on a one-GPU box only (never a measurement): SS_BENCH_PG=gloo runs every rank
    # on cuda:0 with gloo plumbing and the host-staged gather instead of NCCL, which refuses two
    # ranks on one device.  The ranks' kernels never wait on each other (independent mode solves).
    smoke_pg = os.environ.get("SS_BENCH_PG") == "gloo" and world > 1
    if smoke_pg:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if smoke_pg:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def reduce_(t, op):
        if world == 1:
            return t
        if smoke_pg:
            h = t.cpu()
            dist.all_reduce(h, op=op)
            return h.to(t.device)
        dist.all_reduce(t, op=op)
        return t
    from paper_2009_06725_b200 import SolverSettings, _lib
    from paper_2009_06725_b200.assembly import assemble_mode_systems
    from paper_2009_06725_b200.comm import ModeComm
    from paper_2009_06725_b200.krylov import gmres_batched

    key = args.workload
    per_step = WORKLOADS[key]["modes_per_gpu_per_step"]
    hbm_peak, peak_kind = peaks()
    t_setup = time.perf_counter()
    case, q, props, op, plan = _setup_workload(key, world, rank)
    mine = plan[rank]
    dev = op.device
    coeffs = case.coefficients
    omegas_all = case.omegas
    profile_dev = torch.from_numpy(np.ascontiguousarray(case.profile, dtype=complex)).to(dev)
    ws = op.krylov(RESTART, per_step, BUDGET)
    comm = ModeComm.from_process_group(local) if world > 1 and not smoke_pg else None
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t_setup
    stream = torch.cuda.current_stream()

    def modes_of_step(s):
        return [mine[(s * per_step + j) % len(mine)] for j in range(per_step)]

    def step(s):
        ms = modes_of_step(s)
        cf = torch.tensor([coeffs[m] for m in ms], dtype=torch.complex128, device=dev)
        g = profile_dev[None] * cf[:, None, None]
        rhs = op.rhs(omegas_all[ms], None, g)
        return ws.solve(omegas_all[ms], rhs, None, TOL, BUDGET, jacobi=True)

    for s in range(args.warmup):
        step(s)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    # ---- timed region: inputs resident in HBM ----
    l0 = _lib.launch_count()
    with ClockSampler(local, rank) as clk:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        iters = 0
        for s in range(args.steps):
            out = step(args.warmup + s)
            iters += int(out["iterations"].sum())
        e1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    launches = _lib.launch_count() - l0
    t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    it_t = torch.tensor([iters], dtype=torch.float64, device=dev)
    t = reduce_(t, dist.ReduceOp.MAX)
    it_t = reduce_(it_t, dist.ReduceOp.SUM)
    ms_total = float(t.item())
    total_iters = float(it_t.item())
    value = total_iters / (ms_total * 1e-3)
    ms_per_step = ms_total / args.steps

    # ---- end to end through the public API: pinned host Dirichlet data in, nodal fields out and
    #      gathered to rank 0 over the library's NCCL communicator, every step.  Pipelined like a
    #      production driver: step s+1's host data is written by a helper thread while step s
    #      solves, and the host<->device copies run on a copy stream (each step's copies are still
    #      inside the timed region) ----
    from concurrent.futures import ThreadPoolExecutor

    nvn, dim = q.n_velocity_nodes, q.dim
    nf = nvn * dim + q.n_vertices
    g_pins = [torch.empty((per_step, nvn, dim), dtype=torch.complex128).pin_memory() for _ in range(2)]
    g_devs = [torch.empty((per_step, nvn, dim), dtype=torch.complex128, device=dev) for _ in range(2)]
    f_pins = [torch.empty((per_step, nf), dtype=torch.complex128).pin_memory() for _ in range(2)]
    f_devs = [torch.empty((per_step, nf), dtype=torch.complex128, device=dev) for _ in range(2)]
    prof_np = np.ascontiguousarray(case.profile, dtype=complex)
    gather_out = torch.empty((world * per_step, nf), dtype=torch.complex128, device=dev) if rank == 0 and world > 1 \
        else None
    settings = SolverSettings(tolerance=TOL, restart=RESTART, max_iterations=BUDGET)
    h2d = g_pins[0].numel() * 16
    d2h = f_pins[0].numel() * 16
    copy_stream = torch.cuda.Stream(dev)
    h2d_done = [torch.cuda.Event() for _ in range(2)]
    d2h_done = [torch.cuda.Event() for _ in range(2)]
    for ev in d2h_done:
        ev.record(copy_stream)
    filler = ThreadPoolExecutor(max_workers=1)

    def fill(s):   # the user's nodal BC data of step s, written into pinned host memory
        buf = g_pins[s % 2].numpy()
        for j, m in enumerate(modes_of_step(s)):
            np.multiply(prof_np, coeffs[m], out=buf[j])

    def e2e_step(s, pending):
        i = s % 2
        ms = modes_of_step(s)
        pending.result()                                  # step s's host data is ready
        with torch.cuda.stream(copy_stream):
            g_devs[i].copy_(g_pins[i], non_blocking=True)
            h2d_done[i].record(copy_stream)
        nxt = filler.submit(fill, s + 1)                  # overlaps this step's solve
        stream.wait_event(h2d_done[i])
        b = assemble_mode_systems(q, props, omegas_all[ms], None, None, operator=op, g_device=g_devs[i])
        X, reps = gmres_batched(b, settings, keep_history=False)
        U, P = op.expand(X, b.g)
        stream.wait_event(d2h_done[i])                    # step s-2's read of this buffer is done
        f = f_devs[i]
        f[:, : nvn * dim] = U.reshape(per_step, -1)
        f[:, nvn * dim:] = P
        if world > 1:   # every rank's fields of this step -> rank 0 (slots rank*per_step + j)
            step_plan = [list(range(r * per_step, (r + 1) * per_step)) for r in range(world)]
            if comm is not None:
                comm.gather_modes(f, step_plan, root=0, out=gather_out)
            else:
                from paper_2009_06725_b200.distributed import gather_mode_fields

                gather_mode_fields(f, step_plan, rank, world, comm=None, dst=0)
        ready = torch.cuda.Event()
        ready.record(stream)
        with torch.cuda.stream(copy_stream):
            copy_stream.wait_event(ready)
            f_pins[i].copy_(f, non_blocking=True)         # the step's result, read back to the host
            d2h_done[i].record(copy_stream)
        return sum(r.iterations for r in reps), nxt

    fill(0)
    _, pending = e2e_step(0, filler.submit(lambda: None))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0.record(stream)
    w0 = time.perf_counter()
    e_iters = 0
    for s in range(args.steps):
        it, pending = e2e_step(s + 1, pending)
        e_iters += it
    stream.wait_stream(copy_stream)                       # the last read-back is inside the timing
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_wall = time.perf_counter() - w0
    pending.result()
    filler.shutdown()
    t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    ei = torch.tensor([e_iters], dtype=torch.float64, device=dev)
    t = reduce_(t, dist.ReduceOp.MAX)
    ei = reduce_(ei, dist.ReduceOp.SUM)
    e2e_value = float(ei.item()) / (float(t.item()) * 1e-3)
    del g_pins, g_devs, f_pins, f_devs, gather_out

    # ---- roofline: one instrumented (event-timed, un-graphed) cycle on the same stream ----
    ms0 = modes_of_step(0)
    cf = torch.tensor([coeffs[m] for m in ms0], dtype=torch.complex128, device=dev)
    ws.load_rhs(op.rhs(omegas_all[ms0], None, profile_dev[None] * cf[:, None, None]))
    prof = ws.profile(omegas_all[ms0], TOL, BUDGET, jacobi=True)
    dom_name = max((k for k in prof if k != "spmv"), key=lambda k: prof[k]["ms"])
    dom = prof[dom_name]
    traffic = _traffic_from_profile(key, dom_name, dom)
    achieved = dom["bytes"] / (dom["ms"] * 1e-3) / 1e9
    total_ms = sum(v["ms"] for v in prof.values())
    passes_bytes = sum(prof[k]["bytes"] for k in prof if k != "spmv")
    passes_ms = sum(prof[k]["ms"] for k in prof if k != "spmv")

    # ---- the tick SpMV standalone (second half of the metric) ----
    spmv = _spmv_numbers(op, omegas_all[ms0], ws, e0, e1, stream, hbm_peak, torch)
    # headline SpMV figure: the tick's SpMV inside the instrumented cycle (CUDA events around each
    # launch on the solve stream); the standalone call is kept beside it
    in_cycle_ms = prof["spmv"]["ms"] / max(1, prof["spmv"]["launches"])
    in_gbs = op.spmv_bytes(per_step) / (in_cycle_ms * 1e-3) / 1e9
    spmv.update({"standalone_ms": spmv["ms"], "standalone_gbs": spmv["achieved_gbs"], "ms": in_cycle_ms,
                 "achieved_gbs": in_gbs, "frac": in_gbs / hbm_peak, "share_of_cycle": prof["spmv"]["ms"] / total_ms,
                 "measured": "in-cycle (instrumented cycle, per launch); standalone_* = one isolated call"})

    extras = {}
    if rank == 0 and world == 1 and not args.quick:
        op.release_workspaces()
        extras.update(_converged_extras(torch))
        if key == "c5":
            extras["c2_secondary"] = _c2_secondary(torch, hbm_peak)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        c0 = time.perf_counter()
        cyc, det = _oracle_cycle_seconds(key, 1)
        cpu = {"value": BUDGET / cyc, "unit": UNIT, "cores": 1, "kind": "port",
               "sample": _cpu_sample_text(key, det, 1) + f"; per-index seconds on the sample "
                         f"{[round(c, 3) for c in det['costs']]}, cycle end {det['t_end']:.3f} s; "
                         f"{time.perf_counter() - c0:.1f} s of CPU work"}

    if rank == 0:
        clocks = clk.summary()
        cfg = config_dict(key)
        w = WORKLOADS[key]
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "c128",
            "data": f"synthetic (seeded, BASELINE config {key[1]})",
            "config": cfg,
            "setup_s": setup_s,
            "projected_modes_per_s": _projection(key, value),
            "sweep": {"modes": w["total_modes"], "max_modes_per_gpu": max(len(p) for p in plan),
                      "one_cycle_of_every_mode_s": max(len(p) for p in plan) / per_step * ms_per_step / 1e3,
                      "note": "derived: makespan of one restart cycle of all modes on n_gpus (LPT plan)"},
            "roofline": {"bound": "hbm", "kernel": f"k_pass<{dom_name}>", "achieved": achieved, "peak": hbm_peak,
                         "unit": "GB/s", "frac": achieved / hbm_peak,
                         "traffic": None if traffic is None else traffic["ratio"] * dom["bytes"] / dom["launches"],
                         "algorithmic_bytes_per_launch": dom["bytes"] / dom["launches"],
                         "traffic_detail": traffic, "peak_kind": peak_kind, "share_of_step": dom["ms"] / total_ms,
                         "all_basis_passes_gbs": passes_bytes / (passes_ms * 1e-3) / 1e9,
                         "per_kernel": prof},
            "spmv": spmv,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "pipelined": "step s+1's host data written by a helper thread and all host<->device copies on a "
                                 "copy stream while step s solves; every step's copies inside the timed region",
                    "gather": None if world == 1 else ("ss_comm_gather_modes (NCCL) to rank 0 every step" if comm
                                                       else "gloo host-staged gather (SS_BENCH_PG=gloo code-path check)"),
                    "wall_s": e2e_wall},
            "gpu_launches": int(launches),
            "clocks": clocks,
        }
        line.update(extras)
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()


def _projection(key, value):
    """Modes/s projected from the measured rate and iteration counts measured to convergence at
    config 2 (profiles/r2_c2_converge.json: modes 1 and 16 to 1e-10 on the GPU), scaled to the
    workload's n by the growth measured on the reference's down-scaled pipes (iterations ~ n^0.92,
    SURVEY.md §8d).  A projection, labelled as such."""
    from paper_2009_06725_b200.distributed import C2_MEASURED_ITERATIONS, expected_iterations

    w = WORKLOADS[key]
    growth = (w["n_dofs"] / WORKLOADS["c2"]["n_dofs"]) ** 0.92
    idx = np.arange(w["total_modes"])
    per_mode = C2_MEASURED_ITERATIONS[1] * expected_iterations(idx, 3) * growth
    mean_iters = float(per_mode[1:].mean())
    return {"value": value / mean_iters, "mean_iterations_per_mode": mean_iters,
            "basis": "PROJECTION: measured mode-iterations/s / mean iterations per mode; iterations from modes 1 and "
                     "16 solved to 1e-10 at config 2 (336 974 and 886 922, profiles/r2_c2_converge.json), linear in "
                     f"the mode index, scaled by (n/n_c2)^0.92 = {growth:.2f}"}


def _traffic_from_profile(key, dom_name, dom):
    """DRAM traffic / algorithmic bytes of the dominant kernel from the committed `ncu --set full`
    capture of this workload (profiles/), or None."""
    path = os.path.join(ROOT, "profiles", f"r2_ncu_full_{key}.json")
    try:
        with open(path) as fh:
            cap = json.load(fh)
        want = {"passA_dot": "k_pass<1>", "passB_update_dot": "k_pass<2>", "passC_update_norm": "k_pass<3>"}[dom_name]
        rec = next(r for r in cap["launches"] if want in r["kernel"])
        return {"bytes_per_launch": rec["dram_read_bytes"] + rec["dram_write_bytes"],
                "algorithmic_bytes_same_launch": rec["algorithmic_bytes"],
                "ratio": (rec["dram_read_bytes"] + rec["dram_write_bytes"]) / rec["algorithmic_bytes"],
                "source": os.path.relpath(path, ROOT)}
    except Exception:
        return None


def _spmv_numbers(op, omegas, ws, e0, e1, stream, hbm_peak, torch):
    nb = len(omegas)
    xr = torch.randn((nb, op.ld), dtype=torch.complex128, device=op.device)
    ys = torch.zeros((nb, op.ld), dtype=torch.complex128, device=op.device)

    def time_it(fn, reps=10):
        for _ in range(2):
            fn()
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    row = ws.options()["row_spmv"]
    if row:
        ms = time_it(lambda: op.spmv(omegas, xr, jacobi=True, out=ys))
        kern = "row-layout tick SpMV (saddle_block: 4 lanes per node row, 8 per pressure row)"
    else:
        xi = torch.randn((op.ld, nb), dtype=torch.complex128, device=op.device)
        ms = time_it(lambda: op.spmv_interleaved(omegas, xi, jacobi=True, out=ys))
        kern = "k_spmv_interleaved (tick SpMV)"
    by = op.spmv_bytes(nb)
    gbs = by / (ms * 1e-3) / 1e9
    return {"kernel": kern, "modes": nb, "ms": ms, "bytes": by, "achieved_gbs": gbs, "frac": gbs / hbm_peak,
            "peak": hbm_peak,
            "note": "algorithmic bytes (ss_spmv_bytes) = matrix stream once + x read + y write per mode"}


def _converged_extras(torch):
    """Measured modes solved/s: config 1 (2D) and the down-scaled 3D pipes, every mode to 1e-10,
    through the public batched API (gmres_batched: small systems run as concurrent sub-batches)."""
    from paper_2009_06725_b200 import FluidProps, SolverSettings
    from paper_2009_06725_b200.assembly import assemble_mode_systems, get_operator
    from paper_2009_06725_b200.krylov import concurrent_groups, gmres_batched
    from paper_2009_06725_b200.workloads import c1_case, c5_small, pipe3d_case

    out = {}
    settings = SolverSettings(tolerance=TOL, restart=RESTART, max_iterations=400_000)
    for tag, case in (("c1_converged", c1_case()), ("c3d_converged_pipe3d", pipe3d_case()),
                      ("c3d_converged_c5small", c5_small())):
        props = FluidProps(case.density, case.viscosity)
        op = get_operator(case.qmesh, props)
        nm = case.n_modes + 1
        b = assemble_mode_systems(case.qmesh, props, case.omegas, case.g_modes(), case.h_modes(), operator=op)
        gmres_batched(b, settings, keep_history=False)   # warm-up (workspaces, graph capture)
        torch.cuda.synchronize()
        secs = []
        for _ in range(1 if tag == "c3d_converged_c5small" else 3):   # sub-second solves: median of 3
            w0 = time.perf_counter()
            X, reps = gmres_batched(b, settings, keep_history=False)
            torch.cuda.synchronize()
            secs.append(time.perf_counter() - w0)
        sec = sorted(secs)[len(secs) // 2]
        out[tag] = {"workload": case.name, "n_dofs": op.n, "modes": int(nm), "tol": TOL, "restart": RESTART,
                    "seconds": sec, "repeat_seconds": secs, "modes_per_s": nm / sec,
                    "all_converged": all(r.converged for r in reps),
                    "iterations": [int(r.iterations) for r in reps],
                    "concurrent_sub_batches": concurrent_groups(op.n, nm),
                    "measured": "every mode solved to the reference's stopping rule (true residual re-checked)"}
        op.release_workspaces()
    return out


def _c2_secondary(torch, hbm_peak):
    """Config 2 (17 modes in one batch per GPU): one graphed cycle per step, device-resident."""
    from paper_2009_06725_b200 import FluidProps
    from paper_2009_06725_b200.assembly import assemble_mode_systems, get_operator
    from paper_2009_06725_b200.workloads import c2_case

    case = c2_case()
    props = FluidProps(case.density, case.viscosity)
    op = get_operator(case.qmesh, props)
    b = assemble_mode_systems(case.qmesh, props, case.omegas, case.g_modes(), None, operator=op)
    ws = op.krylov(RESTART, 17, BUDGET)
    ws.solve(case.omegas, b.rhs, None, TOL, BUDGET)
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    it = 0
    for _ in range(3):
        it += int(ws.solve(case.omegas, b.rhs, None, TOL, BUDGET)["iterations"].sum())
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    xi = torch.randn((op.ld, 17), dtype=torch.complex128, device=op.device)
    ys = torch.zeros((17, op.ld), dtype=torch.complex128, device=op.device)
    for _ in range(3):
        op.spmv_interleaved(case.omegas, xi, jacobi=True, out=ys)
    e0.record(stream)
    for _ in range(20):
        op.spmv_interleaved(case.omegas, xi, jacobi=True, out=ys)
    e1.record(stream)
    torch.cuda.synchronize()
    sms = e0.elapsed_time(e1) / 20
    by = op.spmv_bytes(17)
    op.release_workspaces()
    return {"workload": case.name, "modes_per_step": 17, "value": it / (ms * 1e-3), "unit": UNIT,
            "ms_per_step": ms / 3, "spmv_ms": sms, "spmv_gbs": by / (sms * 1e-3) / 1e9,
            "spmv_frac": by / (sms * 1e-3) / 1e9 / hbm_peak}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="c5", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--quick", action="store_true", help="skip the converged-mode and config-2 extras")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
