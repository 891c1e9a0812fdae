"""Bisect the first difference between the fused and the graphed tick: config 1 with maxiter =
m for several m, comparing x, histories and the per-mode cycle residuals bitwise."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2009_06725_b200 import FluidProps, workloads  # noqa: E402
from paper_2009_06725_b200.assembly import assemble_mode_systems, get_operator  # noqa: E402
from paper_2009_06725_b200.krylov import KrylovWorkspace  # noqa: E402

case = workloads.c1_case()
props = FluidProps(case.density, case.viscosity)
op = get_operator(case.qmesh, props)
nm = len(case.omegas)
b = assemble_mode_systems(case.qmesh, props, case.omegas, case.g_modes(), case.h_modes(), operator=op)
wss = {}
for f in (0, 1):
    wss[f] = KrylovWorkspace.for_operator(op, 200, nm, 400000)
    wss[f].set_option("fused", f)
    wss[f].set_option("ticks_per_graph", int(os.environ.get("TPG", "16")))
for m in [int(v) for v in (sys.argv[1:] or ["199", "200", "201", "202", "205", "400"])]:
    outs = {}
    for f, ws in wss.items():
        o = ws.solve(case.omegas, b.rhs, None, 1e-10, m)
        torch.cuda.synchronize()
        outs[f] = (o["x"].cpu().numpy(), [np.asarray(ws.history(q, int(o["hist_len"][q]))) for q in range(nm)],
                   o["cycle_residual"].copy(), o["iterations"].copy())
    x0, h0, r0, i0 = outs[0]
    x1, h1, r1, i1 = outs[1]
    dx = [float(np.abs(x0[q] - x1[q]).max()) for q in range(nm)]
    hd = [bool(np.array_equal(a, c)) for a, c in zip(h0, h1)]
    print(f"maxiter={m}: x equal {[bool(np.array_equal(x0[q], x1[q])) for q in range(nm)]} max|dx| "
          f"{['%.1e' % v for v in dx]} hist equal {hd} cycle res equal {(r0 == r1).tolist()} iters {i0.tolist()} {i1.tolist()}",
          flush=True)
