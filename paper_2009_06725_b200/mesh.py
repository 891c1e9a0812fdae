"""Simplex meshes and P2/P1 promotion — the input contract of the hot path.

The node numbering produced here is a *parity contract*: the reduced-system sparsity pattern is
bit-compared with the reference, so this module reproduces the reference numbering exactly
(`pkg/src/spectralstokes/mesh.py:195-315`):

* velocity nodes are the mesh vertices followed by one mid-edge node per unique edge;
* unique edges are the sorted vertex pairs in lexicographic order (`mesh.py:241-248`);
* ``vel_conn`` is ``[element vertices, n_vertices + local edge ids]`` in VTK local-edge order
  (`mesh.py:23-24,282`), ``pres_conn`` is the vertex connectivity (`mesh.py:230-231`);
* patch ``face_conn`` lists face vertices then the face's mid-edge nodes (`mesh.py:303-315`).

Everything here is vectorised numpy (the reference's Python dict loops take seconds at 200k
tets, `SURVEY.md` §8f row 1).  It runs once per mesh on the host, before the device pattern
builder (`csrc/pattern.cpp`).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import MeshError

PATCH_KINDS = ("dirichlet", "neumann", "wall")

TRI_EDGES = ((0, 1), (1, 2), (2, 0))
TET_EDGES = ((0, 1), (1, 2), (0, 2), (0, 3), (1, 3), (2, 3))
TRI_FACES = ((0, 1), (1, 2), (2, 0))
TET_FACES = ((0, 2, 1), (0, 1, 3), (1, 2, 3), (0, 3, 2))


def _row_keys(rows: np.ndarray, n: int):
    """Map sorted integer rows to scalar keys whose order is lexicographic row order."""
    rows = np.asarray(rows, dtype=np.int64)
    width = rows.shape[1]
    if n ** width < 2 ** 62:
        key = np.zeros(rows.shape[0], dtype=np.int64)
        for c in range(width):
            key = key * n + rows[:, c]
        return key
    # Wide rows on huge meshes: fall back to a structured view (same lexicographic order).
    rows = np.ascontiguousarray(rows)
    return rows.view([("", np.int64)] * width).ravel()


@dataclass
class BoundaryPatch:
    """Named set of boundary faces with a boundary-condition kind (`mesh.py:31-41`)."""

    kind: str
    faces: np.ndarray

    def __post_init__(self):
        if self.kind not in PATCH_KINDS:
            raise MeshError(f"unknown patch kind '{self.kind}' (expected one of {PATCH_KINDS})")
        self.faces = np.asarray(self.faces, dtype=np.int64)


def signed_volumes(nodes, elements):
    """Signed area (2D) / volume (3D) per simplex (`mesh.py:113-123`)."""
    p = nodes[elements]
    e1 = p[:, 1] - p[:, 0]
    e2 = p[:, 2] - p[:, 0]
    if nodes.shape[1] == 2:
        return 0.5 * (e1[:, 0] * e2[:, 1] - e1[:, 1] * e2[:, 0])
    e3 = p[:, 3] - p[:, 0]
    return np.einsum("ij,ij->i", np.cross(e1, e2), e3) / 6.0


class Mesh:
    """Linear simplex mesh with named boundary patches (`mesh.py:44-110`).

    Validation matches the reference: index range, strictly positive orientation, and every
    patch face must be a boundary face (a face of exactly one element).
    """

    def __init__(self, nodes, elements, boundary_patches=None):
        self.nodes = np.ascontiguousarray(nodes, dtype=float)
        self.elements = np.ascontiguousarray(elements, dtype=np.int64)
        self.boundary_patches = dict(boundary_patches or {})
        self._validate()
        self.nodes.flags.writeable = False
        self.elements.flags.writeable = False

    @property
    def dim(self):
        return self.nodes.shape[1]

    @property
    def n_nodes(self):
        return self.nodes.shape[0]

    @property
    def n_elements(self):
        return self.elements.shape[0]

    def _validate(self):
        if self.nodes.ndim != 2 or self.nodes.shape[1] not in (2, 3):
            raise MeshError(f"nodes must be (n, 2) or (n, 3), got {self.nodes.shape}")
        dim = self.dim
        if self.elements.ndim != 2 or self.elements.shape[1] != dim + 1:
            raise MeshError(
                f"elements must be (n, {dim + 1}) for a {dim}D mesh, got {self.elements.shape}"
            )
        bad = np.nonzero(((self.elements < 0) | (self.elements >= self.n_nodes)).any(axis=1))[0]
        if bad.size:
            raise MeshError(
                f"element {bad[0]} references node {self.elements[bad[0]].max()} "
                f"outside the {self.n_nodes}-node table"
            )
        vol = signed_volumes(self.nodes, self.elements)
        bad = np.nonzero(vol <= 0.0)[0]
        if bad.size:
            ids = ", ".join(str(i) for i in bad[:8])
            raise MeshError(f"non-positive element volume for element(s) {ids}")
        if not self.boundary_patches:
            return
        bkeys = self._boundary_face_keys()
        for name, patch in self.boundary_patches.items():
            if patch.faces.ndim != 2 or patch.faces.shape[1] != dim:
                raise MeshError(f"patch '{name}' faces must be (n, {dim}) vertex tuples")
            if patch.faces.shape[0] == 0:
                continue
            if patch.faces.min() < 0 or patch.faces.max() >= self.n_nodes:
                raise MeshError(f"patch '{name}' references a node outside the {self.n_nodes}-node table")
            keys = _row_keys(np.sort(patch.faces, axis=1), self.n_nodes)
            pos = np.searchsorted(bkeys, keys)
            pos = np.minimum(pos, bkeys.size - 1)
            ok = bkeys[pos] == keys if bkeys.size else np.zeros(keys.size, bool)
            if not np.all(ok):
                f = patch.faces[np.nonzero(~ok)[0][0]]
                raise MeshError(
                    f"patch '{name}' face {tuple(int(v) for v in f)} is not a boundary face of "
                    "exactly one element"
                )

    def _boundary_face_keys(self):
        local = np.array(TRI_FACES if self.dim == 2 else TET_FACES)
        faces = np.sort(self.elements[:, local].reshape(-1, local.shape[1]), axis=1)
        keys = _row_keys(faces, self.n_nodes)
        uniq, counts = np.unique(keys, return_counts=True)
        return uniq[counts == 1]

    def boundary_faces(self):
        """Sorted vertex tuples of faces that belong to exactly one element."""
        local = np.array(TRI_FACES if self.dim == 2 else TET_FACES)
        faces = np.sort(self.elements[:, local].reshape(-1, local.shape[1]), axis=1)
        keys = _row_keys(faces, self.n_nodes)
        uniq, first, counts = np.unique(keys, return_index=True, return_counts=True)
        return faces[first[counts == 1]]


@dataclass
class CircleBoundary:
    """Circular arc boundary (2D) with closest-point projection (`mesh.py:126-142`)."""

    center: np.ndarray
    radius: float

    def __post_init__(self):
        self.center = np.asarray(self.center, dtype=float)

    def project(self, points):
        points = np.atleast_2d(points)
        rel = points - self.center
        dist = np.linalg.norm(rel, axis=1)
        if np.any(dist < 1e-14 * self.radius):
            raise MeshError("cannot project point coincident with circle center")
        return self.center + rel * (self.radius / dist)[:, None]


@dataclass
class CylinderBoundary:
    """Cylindrical surface (3D): axis point, direction, radius (`mesh.py:145-166`)."""

    point: np.ndarray
    axis: np.ndarray
    radius: float

    def __post_init__(self):
        self.point = np.asarray(self.point, dtype=float)
        axis = np.asarray(self.axis, dtype=float)
        self.axis = axis / np.linalg.norm(axis)

    def project(self, points):
        points = np.atleast_2d(points)
        rel = points - self.point
        axial = rel @ self.axis
        radial = rel - axial[:, None] * self.axis
        dist = np.linalg.norm(radial, axis=1)
        if np.any(dist < 1e-14 * self.radius):
            raise MeshError("cannot project point on the cylinder axis")
        return self.point + axial[:, None] * self.axis + radial * (self.radius / dist)[:, None]


@dataclass
class BoundaryGeometry:
    """Analytic surface descriptors for curved patches (`mesh.py:169-185`)."""

    surfaces: dict = field(default_factory=dict)

    def project(self, patch: str, points):
        surf = self.surfaces.get(patch)
        if surf is None:
            return np.atleast_2d(points)
        return surf.project(points)

    def is_curved(self, patch: str) -> bool:
        return patch in self.surfaces


@dataclass
class QuadraticPatch:
    kind: str
    faces: np.ndarray
    face_conn: np.ndarray


class QuadraticMesh:
    """P2 velocity nodes over P1 pressure vertices (`mesh.py:195-238`)."""

    def __init__(self, nodes, n_vertices, elements, vel_conn, edges, boundary_patches):
        self.nodes = np.ascontiguousarray(nodes, dtype=float)
        self.n_vertices = int(n_vertices)
        self.elements = np.ascontiguousarray(elements, dtype=np.int64)
        self.vel_conn = np.ascontiguousarray(vel_conn, dtype=np.int64)
        self.edges = np.ascontiguousarray(edges, dtype=np.int64)
        self.boundary_patches = dict(boundary_patches)
        for arr in (self.nodes, self.elements, self.vel_conn, self.edges):
            arr.flags.writeable = False
        self._device_cache = {}

    @property
    def dim(self):
        return self.nodes.shape[1]

    @property
    def n_velocity_nodes(self):
        return self.nodes.shape[0]

    @property
    def n_edges(self):
        return self.edges.shape[0]

    @property
    def n_elements(self):
        return self.elements.shape[0]

    @property
    def pres_conn(self):
        return self.elements

    def vertex_nodes(self):
        return self.nodes[: self.n_vertices]


def unique_edges(elements, dim):
    """Lexicographically sorted unique vertex pairs and per-element edge ids (`mesh.py:241-248`)."""
    local = np.array(TRI_EDGES if dim == 2 else TET_EDGES)
    elements = np.asarray(elements, dtype=np.int64)
    raw = np.sort(elements[:, local].reshape(-1, 2), axis=1)
    n = int(elements.max()) + 1 if elements.size else 1
    keys = raw[:, 0] * n + raw[:, 1]
    ukeys, first, inverse = np.unique(keys, return_index=True, return_inverse=True)
    edges = raw[first]
    return edges, inverse.reshape(elements.shape[0], local.shape[0])


def _edge_lookup(edges, n):
    keys = edges[:, 0] * n + edges[:, 1]

    def find(a, b):
        lo = np.minimum(a, b)
        hi = np.maximum(a, b)
        k = lo * n + hi
        pos = np.searchsorted(keys, k)
        pos = np.minimum(pos, keys.size - 1)
        if not np.all(keys[pos] == k):
            raise MeshError("patch face edge is not an edge of the mesh")
        return pos

    return find


def _face_edge_pairs(faces, dim):
    if dim == 2:
        return [(faces[:, 0], faces[:, 1])]
    return [(faces[:, 0], faces[:, 1]), (faces[:, 1], faces[:, 2]), (faces[:, 2], faces[:, 0])]


def promote_to_quadratic(mesh: Mesh, geom: BoundaryGeometry | None = None) -> QuadraticMesh:
    """Insert mid-edge nodes, projecting curved-patch midpoints (`mesh.py:251-289`)."""
    geom = geom or BoundaryGeometry()
    dim = mesh.dim
    n_vert = mesh.n_nodes
    edges, per_elem = unique_edges(mesh.elements, dim)
    midpoints = 0.5 * (mesh.nodes[edges[:, 0]] + mesh.nodes[edges[:, 1]])
    find = _edge_lookup(edges, max(n_vert, 1))

    for name, patch in mesh.boundary_patches.items():
        if not geom.is_curved(name) or patch.faces.shape[0] == 0:
            continue
        ids = np.unique(np.concatenate([find(a, b) for a, b in _face_edge_pairs(patch.faces, dim)]))
        target = geom.project(name, midpoints[ids])
        length = np.linalg.norm(mesh.nodes[edges[ids, 1]] - mesh.nodes[edges[ids, 0]], axis=1)
        moved = np.linalg.norm(target - midpoints[ids], axis=1)
        bad = np.nonzero(moved > 0.5 * length)[0]
        if bad.size:
            e = edges[ids[bad[0]]]
            raise MeshError(
                f"projection of edge {(int(e[0]), int(e[1]))} midpoint onto patch '{name}' "
                "moved it by more than half the edge length"
            )
        midpoints[ids] = target

    nodes = np.vstack([mesh.nodes, midpoints])
    vel_conn = np.hstack([mesh.elements, n_vert + per_elem])
    patches = {}
    for name, patch in mesh.boundary_patches.items():
        f = patch.faces
        if f.shape[0] == 0:
            face_conn = np.zeros((0, 3 if dim == 2 else 6), dtype=np.int64)
        else:
            mids = [n_vert + find(a, b) for a, b in _face_edge_pairs(f, dim)]
            face_conn = np.column_stack([f] + mids).astype(np.int64)
        patches[name] = QuadraticPatch(kind=patch.kind, faces=f.copy(), face_conn=face_conn)
    return QuadraticMesh(nodes, n_vert, mesh.elements, vel_conn, edges, patches)


def with_patch_kinds(mesh: Mesh, kinds: dict) -> Mesh:
    """Copy of ``mesh`` with some patches re-typed (e.g. a Dirichlet inlet)."""
    patches = {
        name: BoundaryPatch(kind=kinds.get(name, p.kind), faces=p.faces)
        for name, p in mesh.boundary_patches.items()
    }
    return Mesh(mesh.nodes, mesh.elements, patches)
