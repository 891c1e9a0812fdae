"""B200-native hot path of arXiv 2009.06725's spectral Stokes solver (SCVS).

Drop-in for the reference package's hot-path API (`pkg/src/spectralstokes/__init__.py:10-46`):
the assembly, Krylov and spectral names below keep the reference's signatures; the work runs in
hand-written sm_100a CUDA (libss_b200.so) behind a C ABI (include/spectralstokes_b200.h).
"""

from .assembly import (  # noqa: F401
    ComplexSaddleSystem,
    FluidProps,
    ModeSystemBatch,
    SaddleOperator,
    ShapeSet,
    assemble_mode_system,
    assemble_mode_systems,
    boundary_traction_load,
    get_operator,
    reference_shapes,
)
from .errors import ConfigError, ConvergenceError, DeviceError, MeshError  # noqa: F401
from .krylov import SolveReport, SolverSettings, gmres, gmres_batched, gmres_solve, jacobi_precondition  # noqa: F401
from .mesh import (  # noqa: F401
    BoundaryGeometry,
    BoundaryPatch,
    CircleBoundary,
    CylinderBoundary,
    Mesh,
    QuadraticMesh,
    promote_to_quadratic,
)
from .metrics import (  # noqa: F401
    field_error,
    fit_loglog_slope,
    flow_rate,
    interpolate_at_quadrature,
    l2_norm,
    l2_norms,
    patch_area,
)
from .spectral import (  # noqa: F401
    BoundaryWaveform,
    adaptive_mode_refinement,
    mode_energies,
    ModeSet,
    ModeSolution,
    fourier_transform_bcs,
    reconstruct,
    reconstruct_series,
    reconstruct_signal,
    solve_mode_systems,
    solve_modes,
    truncation_error,
)
from .structured import channel_grid, pipe_grid  # noqa: F401

__version__ = "0.1.0"
