"""Solve config 1 (9 modes) and pipe3d (modes 1, 16) on a fixed budget with the library selected by
SS_B200_LIB and save solutions + histories to <out>.npz (bitwise A/B between library builds).

    SS_B200_LIB=tools/_variants/x.so python tools/lib_compare.py out_a
    python tools/lib_compare.py --compare out_a.npz out_b.npz
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

if sys.argv[1] == "--compare":
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    for k in a.files:
        print(f"{k:14s} bitwise {np.array_equal(a[k], b[k])}  max|d| {np.abs(a[k] - b[k]).max():.3e}")
    sys.exit(0)

from paper_2009_06725_b200 import FluidProps, SolverSettings, solve_mode_systems  # noqa: E402
from paper_2009_06725_b200.workloads import c1_case, pipe3d_case  # noqa: E402

out = {}
for name, case, idx in (("c1", c1_case(), list(range(9))), ("pipe3d", pipe3d_case(), [1, 16])):
    props = FluidProps(case.density, case.viscosity)
    st = SolverSettings(tolerance=1e-10, restart=200, max_iterations=1500)
    sols = solve_mode_systems(case.qmesh, props, idx, case.omegas[idx], case.g_modes() and [case.g_modes()[i] for i in idx],
                              case.h_modes() and [case.h_modes()[i] for i in idx], st)
    out[f"{name}_u"] = np.stack([s.velocity for s in sols])
    out[f"{name}_hist"] = np.concatenate([np.asarray(s.report.residual_history) for s in sols])
np.savez(sys.argv[1], **out)
print("saved", sys.argv[1])
