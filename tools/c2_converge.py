"""Solve config-2 modes to the reference's stopping rule (tol 1e-10, restart 200) on the GPU with a
raised maxiter, to measure the real 3D iteration count (SURVEY.md §8d projects ~6e5 for c2).

    python tools/c2_converge.py [modes=1,16] [maxiter=1500000] [out.json]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2009_06725_b200 import FluidProps, SolverSettings  # noqa: E402
from paper_2009_06725_b200.assembly import assemble_mode_systems, get_operator  # noqa: E402
from paper_2009_06725_b200.krylov import gmres_batched  # noqa: E402
from paper_2009_06725_b200.workloads import c2_case  # noqa: E402

modes = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "1,16").split(",")]
maxiter = int(sys.argv[2]) if len(sys.argv) > 2 else 1_500_000
out = sys.argv[3] if len(sys.argv) > 3 else "gpurun_out/c2_converge.json"
case = c2_case()
props = FluidProps(case.density, case.viscosity)
op = get_operator(case.qmesh, props)
batch = assemble_mode_systems(case.qmesh, props, case.omegas[modes], [case.coefficients[i] * case.profile for i in modes],
                              None, operator=op)
torch.cuda.synchronize()
t0 = time.perf_counter()
X, reps = gmres_batched(batch, SolverSettings(tolerance=1e-10, restart=200, max_iterations=maxiter))
torch.cuda.synchronize()
wall = time.perf_counter() - t0
rec = {"workload": case.name, "n_dofs": op.n, "modes": modes, "tol": 1e-10, "restart": 200, "maxiter": maxiter,
       "seconds": wall, "iterations": [r.iterations for r in reps], "converged": [r.converged for r in reps],
       "true_residual": [r.residual for r in reps],
       "history_every_10k": [[float(h) for h in r.residual_history[::10000]] for r in reps]}
print(json.dumps(rec))
with open(out, "w") as fh:
    json.dump(rec, fh, indent=1)
