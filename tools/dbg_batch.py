import sys; sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2009_06725_b200 import FluidProps, SolverSettings
from paper_2009_06725_b200.assembly import assemble_mode_systems, get_operator
from paper_2009_06725_b200.krylov import gmres_batched
from paper_2009_06725_b200.workloads import c1_case
case = c1_case(); props = FluidProps(case.density, case.viscosity); h = case.h_modes()
settings = SolverSettings(tolerance=1e-6, restart=30, max_iterations=300)
idx = [1, 4, 7]
full = assemble_mode_systems(case.qmesh, props, case.omegas[idx], None, [h[i] for i in idx])
X, rep = gmres_batched(full, settings)
for j, i in enumerate(idx):
    single = assemble_mode_systems(case.qmesh, props, case.omegas[[i]], None, [h[i]])
    print("rhs equal", torch.equal(single.rhs[0], full.rhs[j]))
    Xs, reps = gmres_batched(single, settings)
    ha, hb = np.array(rep[j].residual_history), np.array(reps[0].residual_history)
    n = min(len(ha), len(hb))
    d = np.nonzero(ha[:n] != hb[:n])[0]
    print(i, rep[j].iterations, reps[0].iterations, "first diff", d[:3], ha[d[:1]], hb[d[:1]], torch.equal(X[j], Xs[0]))
rev = assemble_mode_systems(case.qmesh, props, case.omegas[idx[::-1]], None, [h[i] for i in idx[::-1]])
Xr, repr_ = gmres_batched(rev, settings)
for j, i in enumerate(idx):
    jr = len(idx) - 1 - j
    ha, hb = np.array(rep[j].residual_history), np.array(repr_[jr].residual_history)
    n = min(len(ha), len(hb)); d = np.nonzero(ha[:n] != hb[:n])[0]
    print("rev", i, rep[j].iterations, repr_[jr].iterations, "first diff", d[:3], torch.equal(X[j], Xr[jr]))
