"""Config 1 (9 modes) solved to 1e-10 through the public batched path (gmres_batched: concurrent
sub-batches), timed twice in one process; environment knobs are set by the caller."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2009_06725_b200 import FluidProps, SolverSettings  # noqa: E402
from paper_2009_06725_b200.assembly import assemble_mode_systems, get_operator  # noqa: E402
from paper_2009_06725_b200.krylov import gmres_batched  # noqa: E402
from paper_2009_06725_b200.workloads import c1_case, pipe3d_case  # noqa: E402

from paper_2009_06725_b200.workloads import c5_small  # noqa: E402
case = {"c1": c1_case, "pipe3d": pipe3d_case, "c5_small": c5_small}[os.environ.get("CASE", "c1")]()
props = FluidProps(case.density, case.viscosity)
op = get_operator(case.qmesh, props)
b = assemble_mode_systems(case.qmesh, props, case.omegas, case.g_modes(), case.h_modes(), operator=op)
st = SolverSettings(tolerance=1e-10, restart=200, max_iterations=400000)
for rep in range(int(os.environ.get("REPS", "3"))):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    X, reps = gmres_batched(b, st, keep_history=False)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
print(f"{os.environ.get('TAG', '')}: {len(reps) / dt:.2f} modes/s  ({dt:.3f} s, iters {sum(r.iterations for r in reps)}, "
      f"converged {all(r.converged for r in reps)})", flush=True)
