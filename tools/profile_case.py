"""Instrumented (un-graphed, event-timed) solve of a BASELINE config for per-kernel timing.

    python tools/profile_case.py c1|c2|pipe3d|c3|c4|c5 [iters] [modes]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2009_06725_b200 import FluidProps  # noqa: E402
from paper_2009_06725_b200.assembly import assemble_mode_systems, get_operator  # noqa: E402
from paper_2009_06725_b200.workloads import c1_case, c2_case, c3_case, c4_case, c5_case, pipe3d_case  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 110
case = {"c1": c1_case, "c2": c2_case, "pipe3d": pipe3d_case, "c3": c3_case, "c4": c4_case, "c5": c5_case}[name]()
nb = int(sys.argv[3]) if len(sys.argv) > 3 else case.n_modes + 1
q = case.qmesh
props = FluidProps(case.density, case.viscosity)
op = get_operator(q, props)
idx = list(range(nb))
g = None if case.kind != "dirichlet" else [case.coefficients[i] * case.profile for i in idx]
h = None if case.kind != "neumann" else [case.h_modes()[i] for i in idx]
batch = assemble_mode_systems(q, props, case.omegas[idx], g, h, operator=op)
ws = op.krylov(200, nb, iters)
ws.load_rhs(batch.rhs)
torch.cuda.synchronize()
t0 = time.perf_counter()
prof = ws.profile(case.omegas[idx], 1e-10, iters)
torch.cuda.synchronize()
wall = time.perf_counter() - t0
print(f"{name}: n={op.n} nb={nb} iters={iters} wall={wall:.4f}s info={ws.info.tolist()}")
tot = sum(v["ms"] for v in prof.values())
for k, v in prof.items():
    gbs = v["bytes"] / (v["ms"] * 1e-3) / 1e9 if v["bytes"] else 0.0
    print(f"{k:22s} ms={v['ms']:9.2f} share={v['ms'] / tot:5.2f} launches={v['launches']:5d} "
          f"us/launch={1e3 * v['ms'] / max(1, v['launches']):8.1f} GB/s={gbs:8.1f}")
# graphed solve for comparison
t0 = time.perf_counter()
out = ws.solve(case.omegas[idx], batch.rhs, None, 1e-10, iters)
torch.cuda.synchronize()
t1 = time.perf_counter() - t0
ticks, launches = ws.last_stats()
print(f"graphed solve: {t1:.4f}s ticks={ticks} us/tick={1e6 * t1 / ticks:.1f} launches={launches}")
