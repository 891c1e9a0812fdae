"""Persistent fused tick vs the four-kernel graphed tick, solved to 1e-10 in one process.

    python tools/fused_ab.py [c1|pipe3d|c5_small|c3_small ...]

Per case: one workspace per driver (option "fused" 0/1), the same batch solved twice by each
(second run timed), bitwise comparison of the solutions, iteration counts and residual histories.
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2009_06725_b200 import FluidProps, workloads  # noqa: E402
from paper_2009_06725_b200.assembly import assemble_mode_systems, get_operator  # noqa: E402
from paper_2009_06725_b200.krylov import KrylovWorkspace  # noqa: E402

for name in sys.argv[1:] or ["c1"]:
    case = getattr(workloads, name + "_case" if not name.endswith("_small") else name)()
    props = FluidProps(case.density, case.viscosity)
    op = get_operator(case.qmesh, props)
    nm = len(case.omegas)
    b = assemble_mode_systems(case.qmesh, props, case.omegas, case.g_modes(), case.h_modes(), operator=op)
    res = {}
    runs = [int(v) for v in os.environ.get("FUSED_RUNS", "0,1").split(",")]
    for ri, fused in enumerate(runs):
        ws = KrylovWorkspace.for_operator(op, 200, nm, 400000)
        ws.set_option("fused", fused)
        for rep in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            out = ws.solve(case.omegas, b.rhs, None, 1e-10, 400000)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
        ticks, launches = ws.last_stats()
        x = out["x"].cpu().numpy()
        hist = [np.asarray(ws.history(m, int(out["hist_len"][m]))) for m in range(nm)]
        res[ri] = (x, out["iterations"].copy(), hist)
        print(f"{name:9s} fused={fused} n={op.n} modes={nm} {dt:.3f}s {nm / dt:7.2f} modes/s "
              f"{1e6 * dt / max(1, ticks):7.1f} us/tick ticks={ticks} launches={launches} "
              f"conv={bool(out['converged'].all())}", flush=True)
        prof = os.environ.get("SS_FUSED_PROF")
        if fused and prof and os.path.exists(prof):
            d = np.loadtxt(prof, delimiter=",", ndmin=2)
            if d.size:
                print(f"          phases (us/tick, mean over {len(d)} ticks): spmv {d[:, 0].mean():.1f}  A {d[:, 1].mean():.1f}"
                      f"  B {d[:, 2].mean():.1f}  C {d[:, 3].mean():.1f}  (median tick {np.median(d.sum(1)):.1f})", flush=True)
        ws.close()
    for ri in range(1, len(runs)):
        x0, i0, h0 = res[0]
        x1, i1, h1 = res[ri]
        same_x = np.array_equal(x0.view(np.uint8), x1.view(np.uint8))
        same_h = all(np.array_equal(a, c) for a, c in zip(h0, h1))
        first = []
        for a, c in zip(h0, h1):
            m = min(len(a), len(c))
            d = np.nonzero(a[:m] != c[:m])[0]
            first.append(int(d[0]) if d.size else (-1 if len(a) == len(c) else m))
        print(f"{name:9s} run0(fused={runs[0]}) vs run{ri}(fused={runs[ri]}): bitwise x {same_x}  iterations "
              f"{np.array_equal(i0, i1)}  histories {same_h}  max|dx| {np.abs(x0 - x1).max():.3e}  "
              f"first differing history index per mode {first}", flush=True)
