"""Benchmark: BASELINE config 2 (3D pipe, 199 800 jittered tets, 17 Fourier modes, complex128).

A step is one pass of the hot path over the config's mode batch: one full restarted-GMRES cycle
(restart 200, i.e. 200 inner iterations per mode: SpMV + CGS2 + Givens, then the cycle-end
solve, x update and true residual) for every mode, from x0 = 0 on the assembled right-hand
sides.  Config 2 cannot be converged at 1e-10 inside a benchmark (~10^5+
iterations per mode), so the rate is reported as GMRES mode-iterations per second at that fixed
budget, with the projected modes/s labelled as a projection; config 1 (2D channel, which does
converge) is also solved to 1e-10 and reported as measured modes/s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Multi-GPU (torchrun, one rank per GPU): weak scaling, each rank owns a 17-mode batch of a
17*N-mode set (modes are independent; LPT shard, no data-path collective; the solved modal
fields are all-gathered once per step over NCCL).
"""

from __future__ import annotations

import argparse
import json
import math
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

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_rank{gpu_index}.csv")

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
# CPU baselines (oracle port of the reference; test infrastructure, never the product path)
# ------------------------------------------------------------------------------------------------

STRATA = (0, 50, 100, 150, 199)


def _oracle_cycle_cost(seed_mode: int = 1):
    """Seconds per inner GMRES iteration of the oracle port on config 2, averaged over a restart
    cycle by timing the exact inner-iteration code path at basis indices STRATA."""
    import oracle
    from paper_2009_06725_b200.workloads import c2_case

    case = c2_case()
    s = oracle.assemble_mode_system(case.qmesh, case.density, case.viscosity, case.omegas[seed_mode],
                                    g_mode=case.coefficients[seed_mode] * case.profile)
    sc = oracle.jacobi_scale(s.matrix)
    costs = [oracle.gmres_inner_step_cost(s.matrix, sc, k, RESTART, np.random.default_rng(k)) for k in STRATA]
    return float(np.mean(costs)), costs


def _ref_worker(args):
    os.environ["OMP_NUM_THREADS"] = "1"
    mode, steps = args
    import oracle
    from paper_2009_06725_b200.workloads import c2_case

    case = c2_case()
    s = oracle.assemble_mode_system(case.qmesh, case.density, case.viscosity, case.omegas[mode],
                                    g_mode=case.coefficients[mode] * case.profile)
    sc = oracle.jacobi_scale(s.matrix)
    out = []
    for st in range(steps):
        t0 = time.perf_counter()
        costs = [oracle.gmres_inner_step_cost(s.matrix, sc, k, RESTART, np.random.default_rng(k + 7 * st)) for k in STRATA]
        out.append((float(np.mean(costs)), time.perf_counter() - t0, int(s.matrix.shape[0]), int(s.matrix.nnz),
                    case.name))
    return out


def run_reference(args):
    """--impl reference: the reference's CPU path (oracle port; the reference is pure Python and
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
    procs = max(1, min(cores, 17, int(avail_gb // 4)))
    steps = args.steps + args.warmup
    t0 = time.perf_counter()
    ctx = mp.get_context("spawn")
    with ctx.Pool(procs) as pool:
        res = pool.map(_ref_worker, [(1 + (m % 16), steps) for m in range(procs)])
    wall = time.perf_counter() - t0
    timed = [r[args.warmup:] for r in res]
    per_step = [sum(1.0 / timed[p][s][0] for p in range(procs)) for s in range(args.steps)]
    value = float(np.mean(per_step))
    ms_step = 1e3 * float(np.mean([max(timed[p][s][1] for p in range(procs)) for s in range(args.steps)]))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic (seeded, BASELINE config 2)",
        "config": {"workload": res[0][0][4], "modes_per_gpu": 17, "total_modes": 17, "n_dofs": res[0][0][2],
                   "nnz": res[0][0][3], "restart": RESTART, "iterations_per_mode_per_step": BUDGET, "tol": TOL,
                   "processes": procs},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": procs, "kind": "port",
                         "sample": (f"oracle port of krylov.py:63-164 (numpy/scipy, 1 BLAS thread per process), "
                                    f"{procs} processes each timing the exact inner-iteration code path at basis "
                                    f"indices {list(STRATA)} of a 200-cycle on config 2 (cycle-average cost); "
                                    f"value = sum over processes of 1/cost")},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "host_cores": cores, "wall_s": wall,
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------------
# B200 arm
# ------------------------------------------------------------------------------------------------

def run_b200(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2009_06725_b200 import FluidProps, SolverSettings, _lib
    from paper_2009_06725_b200.assembly import assemble_mode_systems, get_operator
    from paper_2009_06725_b200.distributed import expected_iterations, gather_mode_fields, lpt_shard
    from paper_2009_06725_b200.krylov import gmres_batched
    from paper_2009_06725_b200.workloads import _coefficients, c1_case, c2_case

    hbm_peak, peak_kind = peaks()
    case = c2_case()
    q = case.qmesh
    props = FluidProps(case.density, case.viscosity)
    n_modes_total = 17 * world
    coeffs = case.coefficients if world == 1 else _coefficients(2, n_modes_total - 1, lambda n: 1.0 + n ** 1.5)
    omegas_all = 2.0 * np.pi * np.arange(n_modes_total) / case.period
    plan = lpt_shard(expected_iterations(np.arange(n_modes_total), 3), world)
    mine = plan[rank]
    nb = len(mine)
    omegas = omegas_all[mine]
    g_host = np.stack([coeffs[i] * case.profile for i in mine]).astype(complex)

    t_setup = time.perf_counter()
    op = get_operator(q, props)
    batch = assemble_mode_systems(q, props, omegas, list(g_host), None, operator=op)
    ws = op.krylov(RESTART, nb, BUDGET)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t_setup
    stream = torch.cuda.current_stream()

    def step():
        return ws.solve(omegas, batch.rhs, None, TOL, BUDGET, jacobi=True)

    for _ in range(args.warmup):
        out = step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    # ---- timed region: inputs resident in HBM (basis 200+1 vectors x 17 modes >> 126 MB L2) ----
    l0 = _lib.launch_count()
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        iters = 0
        for _ in range(args.steps):
            out = step()
            iters += int(out["iterations"].sum())
        e1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    launches = _lib.launch_count() - l0
    ms_total = e0.elapsed_time(e1)
    t = torch.tensor([ms_total], dtype=torch.float64, device="cuda")
    it_t = torch.tensor([iters], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(it_t, op=dist.ReduceOp.SUM)
    ms_total = float(t.item())
    total_iters = float(it_t.item())
    value = total_iters / (ms_total * 1e-3)
    ms_per_step = ms_total / args.steps

    # ---- end to end through the public API: pinned host BCs in, nodal fields out, every step ----
    g_pin = torch.from_numpy(g_host.reshape(nb, q.n_velocity_nodes, q.dim)).pin_memory()
    u_pin = torch.empty((nb, q.n_velocity_nodes, q.dim), dtype=torch.complex128).pin_memory()
    p_pin = torch.empty((nb, q.n_vertices), dtype=torch.complex128).pin_memory()
    settings = SolverSettings(tolerance=TOL, restart=RESTART, max_iterations=BUDGET)
    h2d = g_pin.numel() * 16
    d2h = (u_pin.numel() + p_pin.numel()) * 16

    def e2e_step():
        g_dev = g_pin.to(op.device, non_blocking=True)
        b = assemble_mode_systems(q, props, omegas, None, None, operator=op, g_device=g_dev)
        X, reps = gmres_batched(b, settings)
        U, P = op.expand(X, b.g)
        if world > 1:
            nu = q.n_velocity_nodes * q.dim
            gather_mode_fields(torch.cat([U.reshape(nb, -1), P], dim=1), plan, rank, world)
        u_pin.copy_(U, non_blocking=True)
        p_pin.copy_(P, non_blocking=True)
        return sum(r.iterations for r in reps)

    e2e_step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0.record(stream)
    w0 = time.perf_counter()
    e_iters = 0
    for _ in range(args.steps):
        e_iters += e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_wall = time.perf_counter() - w0
    t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
    ei = torch.tensor([e_iters], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(ei, op=dist.ReduceOp.SUM)
    e2e_value = float(ei.item()) / (float(t.item()) * 1e-3)

    # ---- roofline: one instrumented (event-timed, un-graphed) cycle on the same stream ----
    ws.load_rhs(batch.rhs)
    prof = ws.profile(omegas, TOL, BUDGET, jacobi=True)
    dom_name = max((k for k in prof if k != "spmv"), key=lambda k: prof[k]["ms"])
    dom = prof[dom_name]
    traffic = None
    try:   # DRAM traffic of the same kernel from the committed `ncu --set full` capture (J = 100 launch)
        with open(os.path.join(ROOT, "profiles", "r1_ncu_full.json")) as fh:
            cap = json.load(fh)
        rec = next(r for r in cap["launches"] if r["kernel"].startswith("void k_pass<2>"))
        alg = nb * (100 + 2) * 16 * op.n
        traffic = {"bytes_per_launch": rec["dram_read_bytes"] + rec["dram_write_bytes"],
                   "algorithmic_bytes_same_launch": alg,
                   "ratio": (rec["dram_read_bytes"] + rec["dram_write_bytes"]) / alg,
                   "source": "profiles/r1_ncu_full.json (k_pass<2>, tick 100: J = 100)"}
    except Exception:
        traffic = None
    achieved = dom["bytes"] / (dom["ms"] * 1e-3) / 1e9
    share = dom["ms"] / sum(v["ms"] for v in prof.values())
    passes_bytes = sum(prof[k]["bytes"] for k in prof if k != "spmv")
    passes_ms = sum(prof[k]["ms"] for k in prof if k != "spmv")

    # ---- standalone mode-batched SpMV over the 17 modes (second half of the metric): the
    #      mode-interleaved kernel the GMRES tick runs, and the row-layout variant for reference ----
    xi = torch.randn((op.ld, nb), dtype=torch.complex128, device=op.device)
    ys = torch.zeros((nb, op.ld), dtype=torch.complex128, device=op.device)
    xr = torch.randn((nb, op.ld), dtype=torch.complex128, device=op.device)

    def time_spmv(fn, reps=20):
        for _ in range(3):
            fn()
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    spmv_ms = time_spmv(lambda: op.spmv_interleaved(omegas, xi, jacobi=True, out=ys))
    spmv_row_ms = time_spmv(lambda: op.spmv(omegas, xr, jacobi=True, out=ys))
    spmv_bytes = op.spmv_bytes(nb)
    spmv_gbs = spmv_bytes / (spmv_ms * 1e-3) / 1e9
    info = op.info
    spmv_gather = int((q.dim * int(info[4]) + int(info[5]) + q.dim * int(info[6])) * nb * 16)

    extras = {}
    if rank == 0 and world == 1 and not args.quick:
        # config 1 (2D channel, 9 modes) solved to convergence at 1e-10: measured modes/s
        c1 = c1_case()
        p1 = FluidProps(c1.density, c1.viscosity)
        op1 = get_operator(c1.qmesh, p1)
        b1 = assemble_mode_systems(c1.qmesh, p1, c1.omegas, None, c1.h_modes(), operator=op1)
        ws1 = op1.krylov(RESTART, c1.n_modes + 1, 200_000)
        ws1.solve(c1.omegas, b1.rhs, None, TOL, 200_000)
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        o1 = ws1.solve(c1.omegas, b1.rhs, None, TOL, 200_000)
        c1_s = time.perf_counter() - w0
        extras["c1_converged"] = {
            "workload": c1.name, "modes": int(c1.n_modes + 1), "tol": TOL, "seconds": c1_s,
            "modes_per_s": (c1.n_modes + 1) / c1_s, "all_converged": bool(o1["converged"].all()),
            "iterations": [int(v) for v in o1["iterations"]],
            "ticks": ws1.last_stats()[0],
        }

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        c0 = time.perf_counter()
        cost, costs = _oracle_cycle_cost()
        cpu = {"value": 1.0 / cost, "unit": UNIT, "cores": 1, "kind": "port",
               "sample": (f"oracle port of krylov.py:63-164 (numpy/scipy, 1 thread) on config 2 mode 1: exact "
                          f"inner-iteration code path timed at basis indices {list(STRATA)} of a 200-cycle, "
                          f"mean = {cost:.3f} s/iteration (per-index {[round(c, 3) for c in costs]}); "
                          f"{time.perf_counter() - c0:.1f} s of CPU work incl. oracle assembly")}

    if rank == 0:
        clocks = clk.summary()
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "c128", "data": "synthetic (seeded, BASELINE config 2)",
            "config": {"workload": case.name, "modes_per_gpu": nb, "total_modes": n_modes_total,
                       "n_dofs": op.n, "nnz": op.nnz, "restart": RESTART, "iterations_per_mode_per_step": BUDGET,
                       "tol": TOL, "l2": "inputs larger than L2 (basis 17 x 201 x n x 16 B >> 126 MB)",
                       "setup_s": setup_s,
                       "projected_modes_per_s": {
                           "value": value / 2.0e5,
                           "basis": "PROJECTION ONLY: value / 2e5 iterations per mode (krylov.py maxiter default; "
                                    "c2 needs >= 1e5 at 1e-10, SURVEY.md 8d)"}},
            "roofline": {"bound": "hbm", "kernel": f"k_pass<{dom_name}>", "achieved": achieved, "peak": hbm_peak,
                         "unit": "GB/s", "frac": achieved / hbm_peak,
                         "traffic": None if traffic is None else traffic["ratio"] * dom["bytes"] / dom["launches"],
                         "algorithmic_bytes_per_launch": dom["bytes"] / dom["launches"],
                         "traffic_detail": traffic,
                         "peak_kind": peak_kind, "share_of_step": share,
                         "all_basis_passes_gbs": passes_bytes / (passes_ms * 1e-3) / 1e9,
                         "per_kernel": prof},
            "spmv": {"kernel": "k_spmv_interleaved (tick SpMV)", "modes": nb, "ms": spmv_ms, "bytes": spmv_bytes,
                     "achieved_gbs": spmv_gbs, "frac": spmv_gbs / hbm_peak, "peak": hbm_peak,
                     "row_layout_ms": spmv_row_ms,
                     "gathered_bytes": spmv_gather, "gather_tbs": spmv_gather / (spmv_ms * 1e-3) / 1e12,
                     "note": ("algorithmic bytes = matrix once + x read + y write per mode; the kernel gathers "
                              "x once per stored entry and mode (gathered_bytes, served by L1/L2 at "
                              "gather_tbs); ncu: L1 hit 55 %, L2 hit 52 %, long-scoreboard stalls -> "
                              "gather-latency bound")},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "wall_s": e2e_wall},
            "gpu_launches": int(launches),
            "clocks": clocks,
        }
        line.update(extras)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--quick", action="store_true", help="skip the config-1 convergence extra")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
