"""Config 1 solved to 1e-10 with the mode batch split over k concurrent workspaces/streams/threads.

    python tools/c1_streams.py [k ...]

Per-mode results are batch-invariant, so every split gives bitwise-identical solutions; the
question is whether concurrent sub-batches fill the SMs the single batch leaves idle during its
kernels' latency tails (small n).
"""
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2009_06725_b200 import FluidProps  # noqa: E402
from paper_2009_06725_b200.assembly import assemble_mode_systems, get_operator  # noqa: E402
from paper_2009_06725_b200.krylov import KrylovWorkspace  # noqa: E402
from paper_2009_06725_b200.workloads import c1_case, pipe3d_case  # noqa: E402

name = os.environ.get("CASE", "c1")
case = c1_case() if name == "c1" else pipe3d_case()
props = FluidProps(case.density, case.viscosity)
op = get_operator(case.qmesh, props)
nm = case.n_modes + 1
b = assemble_mode_systems(case.qmesh, props, case.omegas, case.g_modes(), case.h_modes(), operator=op)
ref = None
for k in [int(v) for v in (sys.argv[1:] or ["1", "2", "3"])]:
    groups = [list(range(g, nm, k)) for g in range(k)]
    wss = [KrylovWorkspace.for_operator(op, 200, len(g), 400000) for g in groups]
    streams = [torch.cuda.Stream() for _ in groups]
    rhs = [b.rhs[g].contiguous() for g in groups]
    outs = [None] * k

    def run(i):
        with torch.cuda.stream(streams[i]):
            outs[i] = wss[i].solve(case.omegas[groups[i]], rhs[i], None, 1e-10, 400000)

    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        th = [threading.Thread(target=run, args=(i,)) for i in range(k)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    X = np.zeros((nm, op.ld), complex)
    for i, g in enumerate(groups):
        X[g] = outs[i]["x"].cpu().numpy()
    same = ref is None or np.array_equal(X, ref)
    ref = X if ref is None else ref
    print(f"{name} k={k}: {dt:.3f}s {nm / dt:6.2f} modes/s  bitwise-equal-to-k1={same}  "
          f"ticks={[w.last_stats()[0] for w in wss]}", flush=True)
    for w in wss:
        w.close()
