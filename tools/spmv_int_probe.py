"""Standalone mode-interleaved SpMV (the GMRES tick's kernel) on config 2: timing + operator stats.
usage: python tools/spmv_int_probe.py [nb] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2009_06725_b200 import FluidProps  # noqa: E402
from paper_2009_06725_b200.assembly import get_operator  # noqa: E402
from paper_2009_06725_b200.workloads import c2_case  # noqa: E402

nb = int(sys.argv[1]) if len(sys.argv) > 1 else 17
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
c = c2_case()
op = get_operator(c.qmesh, FluidProps(c.density, c.viscosity))
info = op.info
print(f"n={op.n} nfree={info[2]} npf={info[3]} nnz_n={info[4]} nnz_p={info[5]} nnz_t={info[6]} nnz={op.nnz}")
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn((op.ld, nb), dtype=torch.complex128, device="cuda", generator=g)
om = c.omegas[:nb]
y = None
for _ in range(3):
    y = op.spmv_interleaved(om, x, True, y)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    op.spmv_interleaved(om, x, True, y)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
gather = (3 * info[4] + info[5] + 3 * info[6]) * nb * 16
print(f"nb={nb} ms={ms:.4f} algorithmic GB/s={op.spmv_bytes(nb) / ms / 1e6:.1f} gathered GB={gather / 1e9:.2f}"
      f" ({gather / ms / 1e9:.1f} TB/s)")
