"""Standalone mode-batched SpMV timing on config 2 (python tools/spmv_probe.py [nb ...])."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2009_06725_b200 import FluidProps  # noqa: E402
from paper_2009_06725_b200.assembly import get_operator  # noqa: E402
from paper_2009_06725_b200.workloads import c2_case  # noqa: E402

c = c2_case()
op = get_operator(c.qmesh, FluidProps(c.density, c.viscosity))
for nb in [int(v) for v in (sys.argv[1:] or ["1", "17"])]:
    x = torch.randn((nb, op.ld), dtype=torch.complex128, device="cuda")
    y = torch.empty_like(x)
    om = c.omegas[:nb]
    for _ in range(3):
        op.spmv(om, x, True, y)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        op.spmv(om, x, True, y)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"nb={nb} ms={ms:.4f} GB/s={op.spmv_bytes(nb) / ms / 1e6:.1f}")
