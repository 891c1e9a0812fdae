"""A/B of the tick SpMV layouts inside one GMRES cycle and of the standalone SpMV.

    python tools/spmv_stream_ab.py c2|c5|c3|pipe3d [modes] [iters]

Prints, per layout (mode-interleaved / TMA-staged row layout), the instrumented per-kernel cycle
times (ws.profile) and the standalone row-layout SpMV (op.spmv, TMA-staged) GB/s.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2009_06725_b200 import FluidProps  # noqa: E402
from paper_2009_06725_b200.assembly import assemble_mode_systems, get_operator  # noqa: E402
from paper_2009_06725_b200.workloads import c2_case, c3_case, c4_case, c5_case, pipe3d_case  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
case = {"c2": c2_case, "c3": c3_case, "c4": c4_case, "c5": c5_case, "pipe3d": pipe3d_case}[name]()
nb = int(sys.argv[2]) if len(sys.argv) > 2 else (1 if name == "c5" else case.n_modes + 1)
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 200
q = case.qmesh
props = FluidProps(case.density, case.viscosity)
op = get_operator(q, props)
idx = list(range(1, nb + 1))
batch = assemble_mode_systems(q, props, case.omegas[idx], [case.coefficients[i] * case.profile for i in idx], None,
                              operator=op)
ws = op.krylov(200, nb, iters)
print(f"{name}: n={op.n} nnz={op.nnz} nb={nb} spmv_bytes={op.spmv_bytes(nb)}", flush=True)
for row in (0, 1):
    ws.set_option("row_spmv", row)
    ws.load_rhs(batch.rhs)
    prof = ws.profile(case.omegas[idx], 1e-10, iters)
    tot = sum(v["ms"] for v in prof.values())
    sp = prof["spmv"]
    gbs = op.spmv_bytes(nb) * sp["launches"] / (sp["ms"] * 1e-3) / 1e9
    print(f"row_spmv={row}: cycle {tot:9.2f} ms  spmv {sp['ms']:8.2f} ms ({sp['ms'] / max(1, sp['launches']):.3f} "
          f"ms/launch, {gbs:7.1f} GB/s)  " + "  ".join(f"{k}={v['ms']:.1f}" for k, v in prof.items()), flush=True)
    out = ws.solve(case.omegas[idx], batch.rhs, None, 1e-10, iters)
    print(f"   graphed: hist0 {ws.history(0, 3)}  iters {out['iterations'].tolist()[:4]}", flush=True)
x = torch.randn((nb, op.ld), dtype=torch.complex128, device=op.device)
y = torch.zeros_like(x)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(3):
    op.spmv(case.omegas[idx], x, jacobi=True, out=y)
e0.record()
for _ in range(10):
    op.spmv(case.omegas[idx], x, jacobi=True, out=y)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"standalone op.spmv (staged) nb={nb}: {ms:.3f} ms, {op.spmv_bytes(nb) / (ms * 1e-3) / 1e9:.1f} GB/s")
