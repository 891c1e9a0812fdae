"""Consistent traction loads on Neumann patches (boundary_traction_load, assembly.py:249-262; host
routine ss_surface_load) -- the reference's pkg/tests/test_assembly.py:175-210 behaviours,
restated (no GPU needed)."""

import numpy as np
import pytest

from paper_2009_06725_b200 import BoundaryPatch, Mesh, boundary_traction_load, promote_to_quadratic
from paper_2009_06725_b200.errors import MeshError


def test_uniform_traction_integrates_to_patch_length(small_channel_qmesh):
    load = boundary_traction_load(small_channel_qmesh, "inlet", np.array([1.0 + 0j, 0.0]))
    assert load[:, 0].sum() == pytest.approx(2.0, rel=1e-12)   # inlet spans y in [-1, 1]
    assert np.max(np.abs(load[:, 1])) == 0.0


def test_zero_traction_gives_zero_load(small_channel_qmesh):
    assert np.max(np.abs(boundary_traction_load(small_channel_qmesh, "inlet", np.zeros(2, complex)))) == 0.0


def test_traction_only_on_neumann_patches(small_channel_qmesh):
    with pytest.raises(MeshError, match="neumann"):
        boundary_traction_load(small_channel_qmesh, "walls", np.array([1.0, 0.0]))


def test_linear_nodal_traction_is_integrated_exactly():
    mesh = Mesh(np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0]]), np.array([[0, 1, 2]]),
                {"bottom": BoundaryPatch(kind="neumann", faces=np.array([[0, 1]])),
                 "rest": BoundaryPatch(kind="wall", faces=np.array([[1, 2], [2, 0]]))})
    q = promote_to_quadratic(mesh)
    h = np.zeros((q.n_velocity_nodes, 2), dtype=complex)
    h[:, 0] = q.nodes[:, 0]                          # h_x = x on the edge y = 0: integral 1/2
    assert boundary_traction_load(q, "bottom", h)[:, 0].sum() == pytest.approx(0.5, abs=1e-12)
