"""Profiling driver: config-2 (17 modes) instrumented solve of `iters` inner iterations
(un-graphed kernels, so ncu can address individual launches).

    python tools/profile_c2.py [iters] [modes]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2009_06725_b200 import FluidProps  # noqa: E402
from paper_2009_06725_b200.assembly import assemble_mode_systems, get_operator  # noqa: E402
from paper_2009_06725_b200.workloads import c2_case  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 110
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 17
case = c2_case()
q = case.qmesh
props = FluidProps(case.density, case.viscosity)
op = get_operator(q, props)
idx = list(range(nb))
batch = assemble_mode_systems(q, props, case.omegas[idx], [case.coefficients[i] * case.profile for i in idx], None,
                              operator=op)
ws = op.krylov(200, nb, iters)
ws.load_rhs(batch.rhs)
torch.cuda.synchronize()
t0 = time.perf_counter()
prof = ws.profile(case.omegas[idx], 1e-10, iters)
torch.cuda.synchronize()
print("wall", time.perf_counter() - t0)
for k, v in prof.items():
    gbs = v["bytes"] / (v["ms"] * 1e-3) / 1e9 if v["bytes"] else 0.0
    print(f"{k:22s} ms={v['ms']:9.2f} launches={v['launches']:5d} GB/s={gbs:8.1f}")
