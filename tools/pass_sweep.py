"""Isolated basis-pass throughput (GB/s) vs basis index k on a workload's operator.

usage: python tools/pass_sweep.py [c1|c2] [nb] [json-env-configs]
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2009_06725_b200 import FluidProps  # noqa: E402
from paper_2009_06725_b200.assembly import get_operator  # noqa: E402
from paper_2009_06725_b200.krylov import KrylovWorkspace  # noqa: E402
from paper_2009_06725_b200.workloads import c1_case, c2_case  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "c2"
case = c2_case() if which == "c2" else c1_case()
nb = int(sys.argv[2]) if len(sys.argv) > 2 else len(case.omegas)
configs = json.loads(sys.argv[3]) if len(sys.argv) > 3 else {"default": {}}
op = get_operator(case.qmesh, FluidProps(case.density, case.viscosity))
ks = [0, 4, 8, 12, 16, 20, 25, 32, 40, 50, 64, 75, 100, 125, 150, 175, 199]
for name, env in configs.items():
    os.environ.update(env)
    ws = KrylovWorkspace.for_operator(op, 200, nb, 16)
    for key in env:
        os.environ.pop(key)
    tot = {1: [0.0, 0], 2: [0.0, 0], 3: [0.0, 0]}
    curve = {1: [], 2: [], 3: []}
    print(f"== {name}  n={op.n} nb={nb}")
    for k in ks:
        row = []
        for p in (1, 2, 3):
            ms, by = ws.bench_pass(nb, k, p, reps=5)
            row.append(f"{'ABC'[p - 1]} {ms * 1e3:8.1f}us {by / ms / 1e6:7.0f}GB/s")
            tot[p][0] += ms
            tot[p][1] += by
            curve[p].append(ms)
        print(f"k={k:3d}  " + "  ".join(row))
    print("avg   " + "  ".join(f"{'ABC'[p - 1]} {tot[p][1] / tot[p][0] / 1e6:7.0f}GB/s" for p in (1, 2, 3)))
    cyc = {p: float(np.interp(np.arange(200), ks, curve[p]).sum()) for p in (1, 2, 3)}
    print("cycle (k=0..199, interpolated): " + "  ".join(f"{'ABC'[p - 1]} {cyc[p]:7.1f}ms" for p in (1, 2, 3))
          + f"  total {sum(cyc.values()):7.1f}ms")
    ws.close()
