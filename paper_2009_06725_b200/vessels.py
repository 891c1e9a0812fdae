"""Seeded swept-tube meshes for BASELINE configs 3 and 4 (the reference has no generator for them).

* :func:`bent_pipe` — config 3: circular pipe (R = 0.5) with a 90° bend of centreline radius 2
  between two straight legs, built by sweeping the reference's ring-fan disk triangulation
  (`structured._disk_triangles`, the same construction as reference `structured.py:56-134`)
  along the centreline and splitting every prism into 3 tets with the min-index diagonal rule.
* :func:`y_junction` — config 4: bifurcating tube.  The parent disk is split along a diameter
  (a chain of mesh edges in the ring-fan triangulation); each half-disk is swept along a daughter
  centreline whose tilt ramps smoothly from 0 to a seeded branch angle (30-60°), while the
  cross-section grows to a seeded radius ratio (0.7-0.85, area-matched D-shaped section) and
  the wall carries a seeded axisymmetric undulation of amplitude 0.05 r.  The two daughters
  share only the diameter nodes of the split layer.

Element orientation is decided on a straight extrusion of the same topology and then every
element of the real geometry is required to be positive (so geometric inversions raise instead
of being silently flipped).  Mid-edge nodes are straight (no projection descriptor), identically
for the GPU path and the oracle.
"""

from __future__ import annotations

import numpy as np

from .errors import MeshError
from .mesh import BoundaryPatch, Mesh
from .structured import _disk_points, _disk_triangles, _ring_start, _split_prisms


def _orient(tets, ref_nodes, nodes):
    """Orientation fixed on a straight reference extrusion, then checked on the real nodes."""
    def vol(pts):
        p = pts[tets]
        return np.einsum("ij,ij->i", np.cross(p[:, 1] - p[:, 0], p[:, 2] - p[:, 0]), p[:, 3] - p[:, 0])

    neg = vol(ref_nodes) < 0
    tets = tets.copy()
    tets[neg, 0], tets[neg, 1] = tets[neg, 1].copy(), tets[neg, 0].copy()
    v = vol(nodes)
    if np.any(v <= 0):
        raise MeshError(f"swept mesh has {int((v <= 0).sum())} inverted elements")
    return tets


def _wall_quads(edges_b, edges_t):
    """Split lateral quads (b0, b1, t1, t0) with the prism rule (diagonal through the min index)."""
    q0, q1, q2, q3 = edges_b[:, 0], edges_b[:, 1], edges_t[:, 1], edges_t[:, 0]
    diag02 = np.minimum(q0, q2) < np.minimum(q1, q3)
    t1 = np.where(diag02[:, None], np.stack([q0, q1, q2], -1), np.stack([q0, q1, q3], -1))
    t2 = np.where(diag02[:, None], np.stack([q0, q2, q3], -1), np.stack([q1, q2, q3], -1))
    return np.stack([t1, t2], axis=1).reshape(-1, 3)


def _boundary_edges(tris):
    e = np.sort(np.vstack([tris[:, [0, 1]], tris[:, [1, 2]], tris[:, [2, 0]]]), axis=1)
    u, c = np.unique(e, axis=0, return_counts=True)
    return u[c == 1]


def _smoothstep(x):
    x = np.clip(x, 0.0, 1.0)
    return x * x * (3.0 - 2.0 * x)


def bent_pipe(n_rings: int, radius: float = 0.5, bend_radius: float = 2.0, leg: float = 2.0,
              n_layers: int | None = None, inlet_kind: str = "dirichlet"):
    """90° bend: straight leg along +z, quarter circle in the x-z plane, straight leg along +x.

    ``n_layers`` defaults to layer spacing = radial spacing (~2.06 M tets at n_rings = 20).
    Patches: ``inlet`` (``inlet_kind``), ``outlet`` (neumann), ``wall`` (wall).
    """
    disk = _disk_points(n_rings, radius)
    tris = _disk_triangles(n_rings)
    nd = disk.shape[0]
    arc = 0.5 * np.pi * bend_radius
    total = 2 * leg + arc
    if n_layers is None:
        n_layers = int(round(total / (radius / n_rings)))
    s = np.linspace(0.0, total, n_layers + 1)
    c = np.zeros((s.size, 3))
    n1 = np.zeros((s.size, 3))
    for i, si in enumerate(s):
        if si <= leg:
            c[i] = (0.0, 0.0, si)
            n1[i] = (1.0, 0.0, 0.0)
        elif si <= leg + arc:
            phi = (si - leg) / bend_radius
            c[i] = (bend_radius - bend_radius * np.cos(phi), 0.0, leg + bend_radius * np.sin(phi))
            n1[i] = (np.cos(phi), 0.0, -np.sin(phi))
        else:
            c[i] = (bend_radius + (si - leg - arc), 0.0, leg + bend_radius)
            n1[i] = (0.0, 0.0, -1.0)
    n2 = np.array([0.0, 1.0, 0.0])
    nodes = (c[:, None, :] + disk[None, :, 0:1] * n1[:, None, :] + disk[None, :, 1:2] * n2).reshape(-1, 3)
    ref = np.vstack([np.column_stack([disk, np.full(nd, float(i))]) for i in range(s.size)])
    layers = np.arange(n_layers)
    bottom = (layers[:, None, None] * nd + tris[None]).reshape(-1, 3)
    tets = _orient(_split_prisms(bottom, bottom + nd), ref, nodes)
    ring0 = _ring_start(n_rings)
    m = np.arange(6 * n_rings)
    ring_edges = np.column_stack([ring0 + m, ring0 + (m + 1) % (6 * n_rings)])
    wall = np.vstack([_wall_quads(ring_edges + l * nd, ring_edges + (l + 1) * nd) for l in range(n_layers)])
    patches = {
        "inlet": BoundaryPatch(kind=inlet_kind, faces=tris[:, ::-1].copy()),
        "outlet": BoundaryPatch(kind="neumann", faces=tris + n_layers * nd),
        "wall": BoundaryPatch(kind="wall", faces=wall),
    }
    return Mesh(nodes, tets, patches)


def y_junction(n_rings: int, seed: int, radius: float = 0.5, parent_length: float = 3.0,
               daughter_length: float = 4.0, transition: float = 1.0, inlet_kind: str = "dirichlet"):
    """Bifurcating tube (BASELINE config 4 at n_rings = 24: ~5 M tets).

    Returns ``(mesh, params)``; ``params`` records the seeded branch angles, radius ratios and
    undulation phases.  Patches: ``inlet`` (``inlet_kind``), ``outlet1``/``outlet2`` (neumann),
    ``wall``.
    """
    rng = np.random.default_rng(seed)
    angles = np.radians(rng.uniform(30.0, 60.0, size=2))
    ratios = rng.uniform(0.7, 0.85, size=2)
    phases = rng.uniform(0.0, 2.0 * np.pi, size=(3, 3))
    amp = 0.05
    h = radius / n_rings
    disk = _disk_points(n_rings, radius)
    tris = _disk_triangles(n_rings)
    nd = disk.shape[0]
    ang = np.mod(np.arctan2(disk[:, 1], disk[:, 0]), 2.0 * np.pi)
    # sectors 0-2 (angles 0..pi) and 3-5 (pi..2pi): the sector of a triangle is that of its centroid
    cen = disk[tris].mean(axis=1)
    upper = cen[:, 1] > 0
    half_tris = [tris[upper], tris[~upper]]

    def undulation(s, length, ph):
        k = np.arange(1, 4)
        w = np.sin(2.0 * np.pi * np.outer(s, k) / length + ph[None, :]).sum(axis=1) / 3.0
        return amp * w

    # parent: full disk along +z, undulation ramped to 0 at both ends of the parent
    n_par = int(round(parent_length / h))
    sp = np.linspace(0.0, parent_length, n_par + 1)
    ramp_p = _smoothstep(sp / transition) * _smoothstep((parent_length - sp) / transition)
    scale_p = 1.0 + ramp_p * undulation(sp, parent_length, phases[0])
    par = np.concatenate([np.column_stack([disk * scale_p[i], np.full(nd, sp[i])]) for i in range(sp.size)])
    ref = [np.column_stack([disk, np.full(nd, float(i))]) for i in range(sp.size)]
    nodes = [par]
    tets = [_split_prisms((np.arange(n_par)[:, None, None] * nd + tris[None]).reshape(-1, 3),
                          (np.arange(n_par)[:, None, None] * nd + tris[None]).reshape(-1, 3) + nd)]
    ring0 = _ring_start(n_rings)
    m = np.arange(6 * n_rings)
    ring_edges = np.column_stack([ring0 + m, ring0 + (m + 1) % (6 * n_rings)])
    wall = [_wall_quads(ring_edges + l * nd, ring_edges + (l + 1) * nd) for l in range(n_par)]
    offset = (n_par + 1) * nd
    split_layer = n_par * nd
    outlets = []
    y0 = 4.0 * radius / (3.0 * np.pi)
    n_d = int(round(daughter_length / h))
    for d, sigma in enumerate((1.0, -1.0)):
        ht = half_tris[d]
        pts = np.unique(ht)
        loc = -np.ones(nd, dtype=np.int64)
        loc[pts] = np.arange(pts.size)
        u = disk[pts, 0]
        v = disk[pts, 1] - sigma * y0
        sd = np.linspace(0.0, daughter_length, n_d + 1)
        blend = _smoothstep(sd / transition)
        alpha = angles[d] * blend
        scale = 1.0 + blend * (np.sqrt(2.0) * ratios[d] - 1.0)
        scale = scale * (1.0 + blend * undulation(sd, daughter_length, phases[1 + d]))
        # centreline by integrating the tangent (0, sigma sin a, cos a) from the half-disk centroid
        ds = np.diff(sd)
        ty = sigma * np.sin(alpha)
        tz = np.cos(alpha)
        cy = sigma * y0 + np.concatenate([[0.0], np.cumsum(0.5 * (ty[1:] + ty[:-1]) * ds)])
        cz = parent_length + np.concatenate([[0.0], np.cumsum(0.5 * (tz[1:] + tz[:-1]) * ds)])
        layers = []
        for i in range(1, n_d + 1):
            ev = np.array([0.0, np.cos(alpha[i]), -sigma * np.sin(alpha[i])])
            layers.append(np.column_stack([
                scale[i] * u,
                cy[i] + scale[i] * v * ev[1],
                cz[i] + scale[i] * v * ev[2],
            ]))
            ref.append(np.column_stack([disk[pts], np.full(pts.size, float(n_par + i))]))
        nodes.append(np.vstack(layers))
        npd = pts.size

        def gid(layer, local_or_global, is_global=False):
            # layer 0 = parent split layer (global disk ids), layer >= 1 = daughter copies
            if layer == 0:
                return split_layer + local_or_global
            return offset + (layer - 1) * npd + loc[local_or_global]

        bot = np.vstack([gid(0, ht)[None]] + [gid(l, ht)[None] for l in range(1, n_d)]).reshape(-1, 3)
        top = np.vstack([gid(l, ht)[None] for l in range(1, n_d + 1)]).reshape(-1, 3)
        tets.append(_split_prisms(bot, top))
        bedges = _boundary_edges(ht)
        wall += [_wall_quads(gid(l, bedges), gid(l + 1, bedges)) for l in range(n_d)]
        outlets.append(gid(n_d, ht))
        offset += n_d * npd
    nodes = np.vstack(nodes)
    ref = np.vstack(ref)
    tets = _orient(np.vstack(tets), ref, nodes)
    patches = {
        "inlet": BoundaryPatch(kind=inlet_kind, faces=tris[:, ::-1].copy()),
        "outlet1": BoundaryPatch(kind="neumann", faces=outlets[0]),
        "outlet2": BoundaryPatch(kind="neumann", faces=outlets[1]),
        "wall": BoundaryPatch(kind="wall", faces=np.vstack(wall)),
    }
    params = {"branch_angles_deg": np.degrees(angles).tolist(), "radius_ratios": ratios.tolist(),
              "undulation_amplitude": amp, "seed": seed}
    return Mesh(nodes, tets, patches), params
