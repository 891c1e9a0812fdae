"""A/B workspace configurations (env read per workspace) on config 2, one full cycle each, in one process."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2009_06725_b200 import FluidProps  # noqa: E402
from paper_2009_06725_b200.assembly import assemble_mode_systems, get_operator  # noqa: E402
from paper_2009_06725_b200.krylov import KrylovWorkspace  # noqa: E402
from paper_2009_06725_b200.workloads import c2_case  # noqa: E402

configs = json.loads(sys.argv[1])
case = c2_case()
props = FluidProps(case.density, case.viscosity)
op = get_operator(case.qmesh, props)
idx = list(range(17))
b = assemble_mode_systems(case.qmesh, props, case.omegas[idx], [case.coefficients[i] * case.profile for i in idx],
                          None, operator=op)
for rep in range(2):
    for name, env in configs.items():
        os.environ.update(env)
        ws = KrylovWorkspace.for_operator(op, 200, 17, 200)
        for k in env:
            os.environ.pop(k)
        ws.solve(case.omegas[idx], b.rhs, None, 1e-10, 200)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = ws.solve(case.omegas[idx], b.rhs, None, 1e-10, 200)
        dt = time.perf_counter() - t0
        print(f"{name:24s} cycle {dt:.4f}s  {17 * 200 / dt:7.1f} mode-it/s  ticks={ws.last_stats()[0]}")
        ws.close()
        del ws
        torch.cuda.empty_cache()
