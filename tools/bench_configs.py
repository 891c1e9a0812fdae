"""BASELINE configs 3-5 at full size on one B200 (evidence line, not the driver's bench):
host setup time (mesh generation + promotion, pattern, assembly, rhs), the modes that fit one GPU
at restart 200, one graphed 200-iteration cycle after a warm-up cycle (GMRES mode-iterations/s),
and the per-kernel split of an instrumented cycle.

    python tools/bench_configs.py [c3 c4 c5] > profiles/r2_configs.jsonl
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2009_06725_b200 import FluidProps  # noqa: E402
from paper_2009_06725_b200.assembly import assemble_mode_systems, get_operator  # noqa: E402
from paper_2009_06725_b200.workloads import c3_case, c4_case, c5_case  # noqa: E402

RESTART, BUDGET, TOL = 200, 200, 1e-10
for name in sys.argv[1:] or ["c3", "c4", "c5"]:
    import gc

    ws = op = b = case = q = None   # release the previous config's workspace and operator
    gc.collect()
    torch.cuda.empty_cache()
    t0 = time.perf_counter()
    case = {"c3": c3_case, "c4": c4_case, "c5": c5_case}[name]()
    q = case.qmesh
    t_mesh = time.perf_counter() - t0
    props = FluidProps(case.density, case.viscosity)
    t1 = time.perf_counter()
    op = get_operator(q, props)
    torch.cuda.synchronize()
    t_op = time.perf_counter() - t1
    nb = min(case.n_modes + 1, op.max_batch(RESTART))
    idx = list(range(1, nb + 1)) if nb <= case.n_modes else list(range(nb))
    t2 = time.perf_counter()
    b = assemble_mode_systems(q, props, case.omegas[idx], [case.coefficients[i] * case.profile for i in idx], None,
                              operator=op)
    ws = op.krylov(RESTART, nb, BUDGET)
    torch.cuda.synchronize()
    t_rhs = time.perf_counter() - t2
    ws.solve(case.omegas[idx], b.rhs, None, TOL, BUDGET)   # warm-up cycle (graph capture)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = ws.solve(case.omegas[idx], b.rhs, None, TOL, BUDGET)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    iters = int(np.asarray(out["iterations"]).sum())
    ws.load_rhs(b.rhs)
    prof = ws.profile(case.omegas[idx], TOL, BUDGET)
    line = {
        "config": name, "workload": case.name, "n_dofs": op.n, "nnz": op.nnz, "modes_in_batch": nb,
        "mode_indices": [idx[0], idx[-1]], "restart": RESTART, "cycle_ms": ms, "iterations": iters,
        "mode_iterations_per_s": iters / (ms * 1e-3),
        "setup_s": {"mesh_and_promotion": t_mesh, "pattern_and_assembly": t_op, "rhs_and_workspace": t_rhs},
        "kernels_ms": {k: v["ms"] for k, v in prof.items()},
        "passes_gbs": {k: v["bytes"] / (v["ms"] * 1e-3) / 1e9 for k, v in prof.items() if v["bytes"] and v["ms"] > 1},
    }
    print(json.dumps(line), flush=True)
    del ws, b, op
    torch.cuda.empty_cache()
