"""Seeded synthetic workloads for the BASELINE configs (`BASELINE.json` "configs", `SURVEY.md` §8d).

The paper's own benchmark geometries are not available (no dataset, no network), so these seeded
meshes and waveforms stand in for them with the shapes, sizes and value distributions the
BASELINE names.  Seeds are fixed here and recorded in every bench line:

* waveform coefficients: ``np.random.default_rng(config_index)``; mode 0 real ``N(0,1)``, modes
  n>=1 complex ``(N(0,1) + i N(0,1)) / decay(n)``;
* mesh jitter: ``np.random.default_rng(100 + config_index)``.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .mesh import Mesh, promote_to_quadratic, with_patch_kinds
from .structured import channel_grid, jittered_pipe, parabolic_inlet_profile, pipe_grid
from .vessels import bent_pipe, y_junction

C1_TOL = 1e-10


@dataclass
class Case:
    name: str
    mesh: Mesh
    geometry: object
    density: float
    viscosity: float
    period: float
    n_modes: int
    coefficients: np.ndarray          # one-sided coefficients, modes 0..n_modes
    patch: str                        # driven patch
    kind: str                         # "neumann" (traction) or "dirichlet" (nodal profile)
    radius: float = 0.0
    _qmesh: object = field(default=None, repr=False)
    _profile: object = field(default=None, repr=False)

    @property
    def omegas(self):
        return 2.0 * np.pi * np.arange(self.n_modes + 1) / self.period

    @property
    def qmesh(self):
        if self._qmesh is None:
            self._qmesh = promote_to_quadratic(self.mesh, self.geometry)
        return self._qmesh

    @property
    def profile(self):
        """Nodal Dirichlet profile (unit flow rate) for "dirichlet" cases."""
        if self._profile is None and self.kind == "dirichlet":
            self._profile = parabolic_inlet_profile(self.qmesh, self.patch, self.radius)
        return self._profile

    def g_modes(self):
        """Per-mode nodal Dirichlet arrays (complex), or None for traction-driven cases."""
        if self.kind != "dirichlet":
            return None
        return [c * self.profile for c in self.coefficients]

    def h_modes(self):
        """Per-mode ``{patch: traction vector}`` dicts, or None for Dirichlet-driven cases."""
        if self.kind != "neumann":
            return None
        e = np.zeros(self.mesh.dim)
        e[0] = 1.0
        return [{self.patch: c * e.astype(complex)} for c in self.coefficients]


def _coefficients(seed: int, n_modes: int, decay) -> np.ndarray:
    rng = np.random.default_rng(seed)
    c = np.zeros(n_modes + 1, dtype=complex)
    c[0] = rng.normal()
    n = np.arange(1, n_modes + 1)
    c[1:] = (rng.normal(size=n_modes) + 1j * rng.normal(size=n_modes)) / decay(n)
    return c


def c1_case() -> Case:
    """Config 1: 2D Womersley channel [0,4]x[0,1], 64x16 cells split in 2, 9 modes, traction inlet."""
    base = channel_grid(64, 16, length=4.0, half_height=0.5)
    mesh = Mesh(base.nodes + np.array([0.0, 0.5]), base.elements, base.boundary_patches)
    return Case("c1_channel_64x16", mesh, None, 1.0, 0.01, 1.0, 8,
                _coefficients(1, 8, lambda n: 1.0 + n ** 2), "inlet", "neumann")


def c2_case() -> Case:
    """Config 2: straight pipe R=0.5, L=5, 199 800 jittered tets, parabolic inlet, 17 modes."""
    mesh, geom = jittered_pipe(10, 111, 0.5, 5.0, seed=102)
    return Case("c2_pipe_199800tets", mesh, geom, 1.06, 0.04, 1.0, 16,
                _coefficients(2, 16, lambda n: 1.0 + n ** 1.5), "inlet", "dirichlet", radius=0.5)


def pipe3d_case() -> Case:
    """Down-scaled config-2 stand-in that the CPU converges in seconds: pipe_grid(3,15)."""
    m, geom = pipe_grid(3, 15, 0.5, 5.0)
    mesh = with_patch_kinds(m, {"inlet": "dirichlet"})
    return Case("pipe3d_3x15", mesh, geom, 1.06, 0.04, 1.0, 16,
                _coefficients(2, 16, lambda n: 1.0 + n ** 1.5), "inlet", "dirichlet", radius=0.5)


def c3_case(n_rings: int = 20) -> Case:
    """Config 3: 90-degree bend (bend radius 2, R = 0.5), ~2.06 M tets at n_rings = 20, 64 modes ~ 1/n^2."""
    mesh = bent_pipe(n_rings, 0.5, 2.0, 2.0)
    return Case(f"c3_bend_{mesh.n_elements}tets", mesh, None, 1.06, 0.04, 1.0, 63,
                _coefficients(3, 63, lambda n: n.astype(float) ** 2), "inlet", "dirichlet", radius=0.5)


def c4_case(n_rings: int = 27) -> Case:
    """Config 4: seeded Y-junction, ~4.96 M tets at n_rings = 27, 32 modes, two zero-traction outlets."""
    mesh, _ = y_junction(n_rings, seed=104)
    return Case(f"c4_yjunction_{mesh.n_elements}tets", mesh, None, 1.06, 0.04, 1.0, 31,
                _coefficients(4, 31, lambda n: 1.0 + n ** 1.5), "inlet", "dirichlet", radius=0.5)


def c5_case(n_rings: int = 35, n_layers: int = 363) -> Case:
    """Config 5: jittered straight pipe, ~8.0 M tets at (35, 363), 128 modes ~ N(0,1)/(1+n^2)."""
    mesh, geom = jittered_pipe(n_rings, n_layers, 0.5, 5.0, seed=105)
    return Case(f"c5_pipe_{mesh.n_elements}tets", mesh, geom, 1.06, 0.04, 1.0, 127,
                _coefficients(5, 127, lambda n: 1.0 + n ** 2), "inlet", "dirichlet", radius=0.5)


def c5_slab(n_layers: int = 9) -> Case:
    """A slab of config 5: the same 35-ring cross-section, layer spacing (5/363), jitter amplitude and
    fluid, ``n_layers`` layers long.  Per-DOF work of a GMRES iteration is the same as config 5's
    (identical element shapes and row lengths); the CPU baseline times the oracle on it and scales
    by n_c5 / n_slab (SpMV ~ nnz, CGS2 ~ n k: both linear in n)."""
    mesh, geom = jittered_pipe(35, n_layers, 0.5, 5.0 * n_layers / 363, seed=105)
    return Case(f"c5_slab_{mesh.n_elements}tets", mesh, geom, 1.06, 0.04, 1.0, 127,
                _coefficients(5, 127, lambda n: 1.0 + n ** 2), "inlet", "dirichlet", radius=0.5)


# Down-scaled instances of the SAME generators (CPU-convergeable; parity at 1e-10 vs the reference)
def c3_small() -> Case:
    return c3_case(2)


def c4_small() -> Case:
    return c4_case(2)


def c5_small() -> Case:
    return c5_case(3, 12)
