"""Benchmark mesh builders for the BASELINE configs.

``channel_grid`` and ``pipe_grid`` build the same meshes as the reference's builders
(`pkg/src/spectralstokes/structured.py:15-53,137-201`) — same vertex order, element order,
prism diagonals and patch faces — so that meshes, and therefore sparsity patterns, can be
compared bit for bit.  They are vectorised restatements of those constructions.
``jittered_pipe`` adds the seeded interior-vertex jitter that turns the structured pipe into the
"unstructured" ~200k-tet mesh of BASELINE config 2 (`SURVEY.md` §8d).
"""

from __future__ import annotations

import math

import numpy as np

from .mesh import BoundaryGeometry, BoundaryPatch, CylinderBoundary, Mesh, signed_volumes


def channel_grid(nx: int, ny: int, length: float = 10.0, half_height: float = 1.0) -> Mesh:
    """Structured triangles on [0,L] x [-H,H]; patches inlet/outlet (neumann), walls (wall)."""
    if nx < 1 or ny < 1:
        raise ValueError("need at least one cell per direction")
    x = np.linspace(0.0, length, nx + 1)
    y = np.linspace(-half_height, half_height, ny + 1)
    xx, yy = np.meshgrid(x, y, indexing="ij")
    nodes = np.column_stack([xx.ravel(), yy.ravel()])
    i, j = np.meshgrid(np.arange(nx), np.arange(ny), indexing="ij")
    i, j = i.ravel(), j.ravel()
    a = i * (ny + 1) + j
    b = (i + 1) * (ny + 1) + j
    c = (i + 1) * (ny + 1) + j + 1
    d = i * (ny + 1) + j + 1
    elements = np.stack([np.column_stack([a, b, c]), np.column_stack([a, c, d])], axis=1)
    elements = elements.reshape(-1, 3)
    jj = np.arange(ny)
    ii = np.arange(nx)
    inlet = np.column_stack([jj + 1, jj])
    outlet = np.column_stack([nx * (ny + 1) + jj, nx * (ny + 1) + jj + 1])
    bottom = np.column_stack([ii * (ny + 1), (ii + 1) * (ny + 1)])
    top = np.column_stack([(ii + 1) * (ny + 1) + ny, ii * (ny + 1) + ny])
    patches = {
        "inlet": BoundaryPatch(kind="neumann", faces=inlet),
        "outlet": BoundaryPatch(kind="neumann", faces=outlet),
        "walls": BoundaryPatch(kind="wall", faces=np.vstack([bottom, top])),
    }
    return Mesh(nodes, elements, patches)


def _disk_points(n_rings: int, radius: float) -> np.ndarray:
    """Centre point then ring k of 6k equally spaced points (scalar libm, like the reference)."""
    pts = [(0.0, 0.0)]
    for k in range(1, n_rings + 1):
        r = radius * k / n_rings
        for m in range(6 * k):
            ang = 2.0 * np.pi * m / (6 * k)
            pts.append((r * np.cos(ang), r * np.sin(ang)))
    return np.asarray(pts, dtype=float)


def _ring_start(k: int) -> int:
    return 1 + 3 * k * (k - 1) if k >= 1 else 0


def _disk_triangles(n_rings: int) -> np.ndarray:
    """Fan triangulation between consecutive rings.

    Per sector the k outer and k-1 inner intervals are merged by interval midpoint
    ((o+1/2)/k vs (i+1/2)/(k-1), outer first on ties); each outer step emits
    (inner, outer, next outer), each inner step (inner, outer, next inner).
    """
    tris = [np.column_stack([np.zeros(6, int), 1 + np.arange(6), 1 + (np.arange(6) + 1) % 6])]
    for k in range(2, n_rings + 1):
        outer, inner = _ring_start(k), _ring_start(k - 1)
        n_out, n_in = 6 * k, 6 * (k - 1)
        keys = np.concatenate([(np.arange(k) + 0.5) / k, (np.arange(k - 1) + 0.5) / (k - 1)])
        is_outer = np.concatenate([np.ones(k, bool), np.zeros(k - 1, bool)])
        order = np.argsort(keys, kind="stable")
        step_outer = is_outer[order]
        oi = np.concatenate([[0], np.cumsum(step_outer)[:-1]])       # outer steps before
        ii = np.concatenate([[0], np.cumsum(~step_outer)[:-1]])      # inner steps before
        for s in range(6):
            o0, i0 = s * k, s * (k - 1)
            i_a = inner + (i0 + ii) % n_in
            o_a = outer + (o0 + oi) % n_out
            third = np.where(step_outer, outer + (o0 + oi + 1) % n_out, inner + (i0 + ii + 1) % n_in)
            tris.append(np.column_stack([i_a, o_a, third]))
    return np.vstack(tris).astype(np.int64)


def _split_prisms(bottom: np.ndarray, top: np.ndarray) -> np.ndarray:
    """Vectorised 3-tet prism split; each quad takes the diagonal through its smallest vertex."""
    v = np.hstack([bottom, top])
    imin = np.argmin(v, axis=1)
    flip = imin >= 3
    bot = np.where(flip[:, None], v[:, [3, 5, 4]], v[:, [0, 1, 2]])
    tp = np.where(flip[:, None], v[:, [0, 2, 1]], v[:, [3, 4, 5]])
    imin = np.argmin(np.hstack([bot, tp]), axis=1)
    rot = (imin[:, None] + np.arange(3)[None, :]) % 3
    b = np.take_along_axis(bot, rot, axis=1)
    t = np.take_along_axis(tp, rot, axis=1)
    first = np.minimum(b[:, 1], t[:, 2]) < np.minimum(b[:, 2], t[:, 1])
    tet_a = np.stack([
        np.column_stack([b[:, 0], b[:, 1], b[:, 2], t[:, 2]]),
        np.column_stack([b[:, 0], b[:, 1], t[:, 2], t[:, 1]]),
        np.column_stack([b[:, 0], t[:, 1], t[:, 2], t[:, 0]]),
    ], axis=1)
    tet_b = np.stack([
        np.column_stack([b[:, 0], b[:, 1], b[:, 2], t[:, 1]]),
        np.column_stack([b[:, 0], t[:, 1], b[:, 2], t[:, 2]]),
        np.column_stack([b[:, 0], t[:, 1], t[:, 2], t[:, 0]]),
    ], axis=1)
    return np.where(first[:, None, None], tet_a, tet_b).reshape(-1, 4)


def _pipe_arrays(n_rings: int, n_layers: int, radius: float, length: float):
    disk = _disk_points(n_rings, radius)
    tris = _disk_triangles(n_rings)
    n_disk = disk.shape[0]
    z = np.linspace(0.0, length, n_layers + 1)
    nodes = np.vstack([np.column_stack([disk[:, 0], disk[:, 1], np.full(n_disk, zz)]) for zz in z])
    layers = np.arange(n_layers)
    bottom = (layers[:, None, None] * n_disk + tris[None, :, :]).reshape(-1, 3)
    top = bottom + n_disk
    tets = _split_prisms(bottom, top)
    p = nodes[tets]
    vol = np.einsum("ij,ij->i", np.cross(p[:, 1] - p[:, 0], p[:, 2] - p[:, 0]), p[:, 3] - p[:, 0])
    neg = vol < 0
    tets[neg, 0], tets[neg, 1] = tets[neg, 1].copy(), tets[neg, 0].copy()

    inlet = tris[:, ::-1].copy()
    outlet = tris + n_layers * n_disk
    ring0 = _ring_start(n_rings)
    n_out = 6 * n_rings
    m = np.arange(n_out)
    a = ring0 + m
    b = ring0 + (m + 1) % n_out
    off_b = (layers * n_disk)[:, None]
    off_t = ((layers + 1) * n_disk)[:, None]
    q0, q1, q2, q3 = off_b + a, off_b + b, off_t + b, off_t + a
    diag02 = np.minimum(q0, q2) < np.minimum(q1, q3)
    t1 = np.where(diag02[..., None], np.stack([q0, q1, q2], -1), np.stack([q0, q1, q3], -1))
    t2 = np.where(diag02[..., None], np.stack([q0, q2, q3], -1), np.stack([q1, q2, q3], -1))
    wall = np.stack([t1, t2], axis=2).reshape(-1, 3)
    return nodes, tets, inlet, outlet, wall


def pipe_grid(n_rings: int, n_layers: int, radius: float = 1.0, length: float = 3.0):
    """Tetrahedral pipe along +z; returns ``(mesh, geometry)`` with a cylindrical wall."""
    if n_rings < 1 or n_layers < 1:
        raise ValueError("need at least one ring and one layer")
    nodes, tets, inlet, outlet, wall = _pipe_arrays(n_rings, n_layers, radius, length)
    patches = {
        "inlet": BoundaryPatch(kind="neumann", faces=inlet),
        "outlet": BoundaryPatch(kind="neumann", faces=outlet),
        "wall": BoundaryPatch(kind="wall", faces=wall),
    }
    geom = BoundaryGeometry(
        surfaces={"wall": CylinderBoundary(point=(0.0, 0.0, 0.0), axis=(0.0, 0.0, 1.0), radius=radius)}
    )
    return Mesh(nodes, tets, patches), geom


def jittered_pipe(n_rings: int, n_layers: int, radius: float, length: float, seed: int,
                  amplitude: float = 0.2, inlet_kind: str = "dirichlet"):
    """Pipe with seeded interior-vertex jitter (BASELINE config 2's "unstructured" pipe).

    Interior vertices move by ``amplitude * h * U(-1,1)^3`` with ``h`` the smaller of the radial
    and axial spacings; moves that would invert an element are halved until none do.
    The inlet is re-typed ``inlet_kind`` (Dirichlet for the parabolic-inflow configs).
    """
    nodes, tets, inlet, outlet, wall = _pipe_arrays(n_rings, n_layers, radius, length)
    boundary = np.zeros(nodes.shape[0], bool)
    for f in (inlet, outlet, wall):
        boundary[f.ravel()] = True
    h = min(radius / n_rings, length / n_layers)
    rng = np.random.default_rng(seed)
    disp = amplitude * h * rng.uniform(-1.0, 1.0, size=nodes.shape)
    disp[boundary] = 0.0
    for _ in range(30):
        trial = nodes + disp
        vol = signed_volumes(trial, tets)
        bad = vol <= 1e-3 * np.abs(signed_volumes(nodes, tets))
        if not bad.any():
            break
        verts = np.unique(tets[bad].ravel())
        disp[verts] *= 0.5
    else:
        disp[:] = 0.0
    nodes = nodes + disp
    patches = {
        "inlet": BoundaryPatch(kind=inlet_kind, faces=inlet),
        "outlet": BoundaryPatch(kind="neumann", faces=outlet),
        "wall": BoundaryPatch(kind="wall", faces=wall),
    }
    geom = BoundaryGeometry(
        surfaces={"wall": CylinderBoundary(point=(0.0, 0.0, 0.0), axis=(0.0, 0.0, 1.0), radius=radius)}
    )
    return Mesh(nodes, tets, patches), geom


def parabolic_inlet_profile(qmesh, patch: str, radius: float, axis: int = 2) -> np.ndarray:
    """Flow-rate-normalised Poiseuille profile ``(2/(pi R^2)) (1 - r^2/R^2) e_axis`` on ``patch``.

    Returns a real nodal array ``(n_velocity_nodes, dim)``, zero off the patch; multiplying by
    ``Q_n`` gives the Dirichlet data of mode ``n`` (BASELINE config 2, `SURVEY.md` §8d).
    """
    g = np.zeros((qmesh.n_velocity_nodes, qmesh.dim))
    nodes = np.unique(qmesh.boundary_patches[patch].face_conn)
    xy = qmesh.nodes[nodes][:, [c for c in range(qmesh.dim) if c != axis]]
    r2 = np.einsum("ij,ij->i", xy, xy)
    g[nodes, axis] = (2.0 / (math.pi * radius * radius)) * np.maximum(0.0, 1.0 - r2 / (radius * radius))
    return g
