"""ORACLE — TEST INFRASTRUCTURE ONLY.

CPU restatement (numpy/scipy) of the reference's hot path, arXiv 2009.06725's spectral Stokes
solver as implemented in `/root/reference/pkg/src/spectralstokes` (assembly.py, krylov.py,
spectral.py).  It is the checker for the CUDA path: only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s CPU-baseline / ``--impl reference`` legs may import it.  The product package
``paper_2009_06725_b200`` never imports it and has no CPU fallback.

Parity pin: every function below is checked against vectors produced by the reference itself
(``tests/golden/make_golden.py`` imports the reference read-only in the build container and
writes ``tests/golden/*.npz``; ``tests/test_oracle_golden.py`` compares).
"""

from .scvs import (  # noqa: F401
    OracleSystem,
    assemble_divergence,
    assemble_mass_scalar,
    assemble_mode_system,
    assemble_stiffness_scalar,
    gmres,
    gmres_cycle_end_cost,
    gmres_inner_step_cost,
    gmres_solve,
    jacobi_scale,
    l2_norm,
    mode_coefficients,
    reconstruct,
    reference_tables,
    sampled_rows,
    solve_mode,
    surface_load,
)
