"""A/B the solve-loop drivers (device-side conditional graph vs host-polled graphs) in one process."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2009_06725_b200 import FluidProps  # noqa: E402
from paper_2009_06725_b200.assembly import assemble_mode_systems, get_operator  # noqa: E402
from paper_2009_06725_b200.krylov import KrylovWorkspace  # noqa: E402
from paper_2009_06725_b200.workloads import c1_case  # noqa: E402

case = c1_case()
props = FluidProps(case.density, case.viscosity)
op = get_operator(case.qmesh, props)
b = assemble_mode_systems(case.qmesh, props, case.omegas, None, case.h_modes(), operator=op)
import json
configs = json.loads(sys.argv[1]) if len(sys.argv) > 1 else {
    "device loop, 16 ticks/body": {"SS_DEVICE_LOOP": "1", "SS_TICKS_PER_GRAPH": "16"},
    "host polled, 16 ticks/graph": {"SS_DEVICE_LOOP": "0", "SS_TICKS_PER_GRAPH": "16"}}
wss = {}
for name, env in configs.items():
    os.environ.update(env)
    wss[name] = KrylovWorkspace.for_operator(op, 200, case.n_modes + 1, 200000)
for env in configs.values():
    for k in env:
        os.environ.pop(k, None)
for rep in range(2):
    for name, ws in wss.items():
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = ws.solve(case.omegas, b.rhs, None, 1e-10, 200000)
        dt = time.perf_counter() - t0
        ticks, launches = ws.last_stats()
        print(f"{name:30s} {dt:.3f}s {(case.n_modes + 1) / dt:6.2f} modes/s {1e6 * dt / ticks:6.1f} us/tick "
              f"ticks={ticks} conv={bool(out['converged'].all())} iters={out['iterations'].tolist()}")
