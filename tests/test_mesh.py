"""Mesh numbering contract: promotion reproduces the reference numbering bit for bit
(mesh.py:241-315) on meshes built by the reference itself (tests/golden/meshes.npz)."""

import numpy as np
import pytest

from paper_2009_06725_b200.errors import MeshError
from paper_2009_06725_b200.mesh import BoundaryGeometry, BoundaryPatch, CylinderBoundary, Mesh, promote_to_quadratic
from paper_2009_06725_b200.structured import channel_grid, jittered_pipe, pipe_grid
from golden_util import golden


def _compare(prefix, q, g):
    assert np.array_equal(q.nodes, g[f"{prefix}_nodes"])
    assert np.array_equal(q.elements, g[f"{prefix}_elements"])
    assert np.array_equal(q.vel_conn, g[f"{prefix}_vel_conn"])
    assert np.array_equal(q.edges, g[f"{prefix}_edges"])
    assert q.n_vertices == int(g[f"{prefix}_nvert"])
    names = [str(n) for n in g[f"{prefix}_patch_names"]]
    assert sorted(q.boundary_patches) == names
    for n in names:
        p = q.boundary_patches[n]
        assert p.kind == str(g[f"{prefix}_patch_{n}_kind"])
        assert np.array_equal(p.faces, g[f"{prefix}_patch_{n}_faces"])
        assert np.array_equal(p.face_conn, g[f"{prefix}_patch_{n}_face_conn"])


@pytest.mark.parametrize("prefix,args", [("chan10x4", (10, 4, 4.0, 1.0)), ("chan3x2", (3, 2, 2.0, 1.0))])
def test_channel_numbering_matches_reference(prefix, args):
    _compare(prefix, promote_to_quadratic(channel_grid(*args)), golden("meshes.npz"))


@pytest.mark.parametrize("prefix,args", [("pipe2x3", (2, 3)), ("pipe3x4", (3, 4))])
def test_pipe_numbering_matches_reference(prefix, args):
    m, geom = pipe_grid(*args, 0.5, 5.0)
    _compare(prefix, promote_to_quadratic(m, geom), golden("meshes.npz"))


def test_curved_wall_midpoints_on_cylinder():
    m, geom = pipe_grid(3, 2, 0.5, 1.0)
    q = promote_to_quadratic(m, geom)
    wall = np.unique(q.boundary_patches["wall"].face_conn)
    r = np.hypot(q.nodes[wall, 0], q.nodes[wall, 1])
    assert np.allclose(r, 0.5, atol=1e-14)


def test_jittered_pipe_valid_and_seeded():
    m1, _ = jittered_pipe(3, 6, 0.5, 2.0, seed=5)
    m2, _ = jittered_pipe(3, 6, 0.5, 2.0, seed=5)
    m0, _ = pipe_grid(3, 6, 0.5, 2.0)
    assert np.array_equal(m1.nodes, m2.nodes)
    assert not np.array_equal(m1.nodes, m0.nodes)
    assert np.array_equal(m1.elements, m0.elements)


def test_mesh_validation_errors():
    nodes = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0]])
    with pytest.raises(MeshError):
        Mesh(nodes, np.array([[0, 2, 1]]))                   # negative orientation
    with pytest.raises(MeshError):
        Mesh(nodes, np.array([[0, 1, 5]]))                   # dangling index
    with pytest.raises(MeshError):
        Mesh(nodes, np.array([[0, 1, 2]]), {"x": BoundaryPatch("wall", np.array([[0, 5]]))})
    with pytest.raises(MeshError):
        BoundaryPatch("slip", np.zeros((0, 2), int))
