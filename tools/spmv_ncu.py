"""Standalone batched SpMV launches of one config, for ncu captures of the row-layout kernels.

    SS_SPMV_STREAM=0|1 python tools/spmv_ncu.py c5|c2 [nb] [reps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2009_06725_b200 import FluidProps  # noqa: E402
from paper_2009_06725_b200.assembly import get_operator  # noqa: E402
from paper_2009_06725_b200.workloads import c2_case, c5_case  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 1
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
case = {"c2": c2_case, "c5": c5_case}[name]()
op = get_operator(case.qmesh, FluidProps(case.density, case.viscosity))
x = torch.randn((nb, op.ld), dtype=torch.complex128, device=op.device)
y = torch.zeros_like(x)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
op.spmv(case.omegas[:nb], x, jacobi=True, out=y)
e0.record()
for _ in range(reps):
    op.spmv(case.omegas[:nb], x, jacobi=True, out=y)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
print(f"{name} nb={nb} stream={os.environ.get('SS_SPMV_STREAM', '0')}: {ms:.3f} ms "
      f"{op.spmv_bytes(nb) / (ms * 1e-3) / 1e9:.1f} GB/s (bytes {op.spmv_bytes(nb)})")
