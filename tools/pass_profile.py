"""Launch isolated basis passes for ncu: python tools/pass_profile.py c2 "2:64,2:150,1:150,3:150"
(pass:k pairs; each bench_pass call launches a warm-up pass plus one timed pass)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2009_06725_b200 import FluidProps  # noqa: E402
from paper_2009_06725_b200.assembly import get_operator  # noqa: E402
from paper_2009_06725_b200.krylov import KrylovWorkspace  # noqa: E402
from paper_2009_06725_b200.workloads import c1_case, c2_case  # noqa: E402

case = c2_case() if sys.argv[1] == "c2" else c1_case()
nb = len(case.omegas)
op = get_operator(case.qmesh, FluidProps(case.density, case.viscosity))
ws = KrylovWorkspace.for_operator(op, 200, nb, 16)
for item in sys.argv[2].split(","):
    p, k = (int(v) for v in item.split(":"))
    ms, by = ws.bench_pass(nb, k, p, reps=1)
    print(f"pass {p} k={k}: {ms * 1e3:.1f} us  {by / ms / 1e6:.0f} GB/s")
ws.close()
