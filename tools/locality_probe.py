"""How much does vertex numbering locality matter to the row-layout SpMV?  Renumber the mesh's
vertices (edges follow: they are sorted by vertex ids), rebuild the operator and time the
standalone one-mode SpMV: native order, reverse Cuthill-McKee over the vertex graph, random.

    python tools/locality_probe.py c2|c5 [reps]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import scipy.sparse as sp  # noqa: E402
import scipy.sparse.csgraph as csg  # noqa: E402
import torch  # noqa: E402

from paper_2009_06725_b200 import FluidProps  # noqa: E402
from paper_2009_06725_b200.assembly import SaddleOperator  # noqa: E402
from paper_2009_06725_b200.mesh import BoundaryPatch, Mesh, promote_to_quadratic  # noqa: E402
from paper_2009_06725_b200.workloads import c2_case, c5_case  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
case = {"c2": c2_case, "c5": c5_case}[name]()
m = case.mesh
nv = m.nodes.shape[0]


def renumber(order):
    inv = np.empty(nv, dtype=np.int64)
    inv[order] = np.arange(nv)
    patches = {k: BoundaryPatch(kind=p.kind, faces=inv[np.asarray(p.faces)]) for k, p in m.boundary_patches.items()}
    return Mesh(m.nodes[order], inv[np.asarray(m.elements)], patches)


el = np.asarray(m.elements)
rows = np.repeat(el, el.shape[1], axis=1).ravel()
cols = np.tile(el, (1, el.shape[1])).ravel()
g = sp.csr_matrix((np.ones(rows.size, dtype=np.int8), (rows, cols)), shape=(nv, nv))
orders = {"native": np.arange(nv), "rcm": np.asarray(csg.reverse_cuthill_mckee(g, symmetric_mode=True)),
          "random": np.random.default_rng(0).permutation(nv)}
props = FluidProps(case.density, case.viscosity)
for tag, order in orders.items():
    q = promote_to_quadratic(renumber(order), case.geometry)
    op = SaddleOperator(q, props, 0)
    x = torch.randn((1, op.ld), dtype=torch.complex128, device=op.device)
    y = torch.zeros_like(x)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        op.spmv([6.28], x, jacobi=True, out=y)
    e0.record()
    for _ in range(reps):
        op.spmv([6.28], x, jacobi=True, out=y)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"{name} {tag:7s}: {ms:.3f} ms  {op.spmv_bytes(1) / (ms * 1e-3) / 1e9:.1f} GB/s  (n = {op.n})", flush=True)
    del op, x, y
    torch.cuda.empty_cache()
