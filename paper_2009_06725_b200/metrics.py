"""Post-processing: the step after reconstruction that also drives adaptive
refinement.  Element-quadrature work runs on the device -- L2 norms / mode energies (reference
`metrics.py:12-18`, `spectral.py:320-330`), `interpolate_at_quadrature` (`assembly.py:497-511`) and
the interpolation behind `field_error` (`metrics.py:21-39`; the user's point oracle is Python and
is evaluated on the host).  Boundary-patch work (`flow_rate`, `patch_area`, `metrics.py:42-101`) is
O(boundary faces) and stays host-side, vectorised; `fit_loglog_slope` is a 4-point host fit."""

from __future__ import annotations

import numpy as np
from ctypes import byref, c_int as C_int

from . import _lib
from .assembly import FluidProps, _OP_CACHE, get_operator
from .errors import MeshError

__all__ = ["l2_norm", "l2_norms", "mode_energies", "interpolate_at_quadrature", "field_error", "flow_rate",
           "patch_area", "fit_loglog_slope"]


def _mesh_operator(qmesh):
    """Any device operator of this mesh (only its geometry is used here)."""
    try:
        cached = _OP_CACHE.get(qmesh)
    except TypeError:
        cached = None
    if cached:
        return next(iter(cached.values()))
    return get_operator(qmesh, FluidProps(1.0, 1.0))


def l2_norms(fields, qmesh) -> np.ndarray:
    """L2(Omega) norms of a batch of nodal fields ``(nb, n_velocity_nodes[, ncomp])`` (device kernel)."""
    torch = _lib.torch_mod()
    op = _mesh_operator(qmesh)
    if isinstance(fields, torch.Tensor):
        f = fields.to(op.device, torch.complex128)
    else:
        f = torch.from_numpy(np.ascontiguousarray(np.asarray(fields, dtype=complex))).to(op.device)
    if f.dim() == 2:
        f = f.unsqueeze(-1)
    if f.shape[1] != qmesh.n_velocity_nodes:
        raise ValueError("fields must be (nb, n_velocity_nodes[, ncomp])")
    f = f.contiguous()
    out = np.zeros(f.shape[0])
    _lib.call("ss_l2_norms", op.handle, f.shape[0], f.shape[2], _lib.dptr(f), _lib.ptr(out),
              _lib.stream_ptr(op.device))
    return out


def l2_norm(nodal, qmesh) -> float:
    """L2(Omega) norm of a nodal velocity-space field, vector or scalar (metrics.py:12-18)."""
    return float(l2_norms(np.asarray(nodal)[None], qmesh)[0])


def mode_energies(solutions, qmesh, period: float) -> np.ndarray:
    """Per-mode contribution to ||u||^2 over Omega x [0,T] (spectral.py:320-330), one batched launch."""
    norms = l2_norms(np.stack([s.velocity for s in solutions]), qmesh)
    w = np.array([period if s.index == 0 else 0.5 * period for s in solutions])
    return w * norms ** 2


def interpolate_at_quadrature(qmesh, nodal):
    """Velocity nodal values -> ``(coords, values, weights)`` at the element quadrature points
    (assembly.py:497-511); ``weights`` include |det J|, so ``sum(weights * f(coords))`` integrates
    over the mesh.  ``nodal`` is ``(n_velocity_nodes, ...)``; real input gives real values."""
    torch = _lib.torch_mod()
    op = _mesh_operator(qmesh)
    arr = np.asarray(nodal)
    if arr.shape[0] != qmesh.n_velocity_nodes:
        raise ValueError("nodal must be (n_velocity_nodes, ...)")
    trail = arr.shape[1:]
    ncomp = int(np.prod(trail)) if trail else 1
    f = torch.from_numpy(np.ascontiguousarray(arr.reshape(arr.shape[0], ncomp), dtype=complex)).to(op.device)
    nq = C_int()
    _lib.call("ss_quadrature_points", qmesh.dim, byref(nq))
    ne, nq = len(qmesh.elements), nq.value
    coords = torch.empty((ne, nq, qmesh.dim), dtype=torch.float64, device=op.device)
    vals = torch.empty((ne, nq, ncomp), dtype=torch.complex128, device=op.device)
    w = torch.empty((ne, nq), dtype=torch.float64, device=op.device)
    _lib.call("ss_interp_quadrature", op.handle, ncomp, _lib.dptr(f), _lib.dptr(coords), _lib.dptr(vals),
              _lib.dptr(w), _lib.stream_ptr(op.device))
    vals = vals.cpu().numpy().reshape((ne, nq) + trail)
    if not np.iscomplexobj(arr):
        vals = vals.real.copy()
    return coords.cpu().numpy(), vals, w.cpu().numpy()


def field_error(nodal, oracle, qmesh) -> float:
    """Relative L2(Omega) difference between a nodal field and a point oracle evaluated at the
    quadrature points (metrics.py:21-39)."""
    coords, vals, w = interpolate_at_quadrature(qmesh, nodal)
    flat = coords.reshape(-1, coords.shape[-1])
    exact = np.asarray(oracle(flat)).reshape(vals.shape)
    diff = np.abs(vals - exact) ** 2
    ref = np.abs(exact) ** 2
    if diff.ndim == 3:
        diff = diff.sum(axis=2)
        ref = ref.sum(axis=2)
    denom = np.sum(w * ref)
    if denom <= 0.0:
        raise ZeroDivisionError("field_error: reference field has zero norm")
    return float(np.sqrt(np.sum(w * diff) / denom))


def _edge_shapes():
    """P2 shapes on a straight edge, 3-point Gauss (assembly.py:131-137)."""
    g = np.sqrt(3.0 / 5.0)
    t = 0.5 * np.array([1 - g, 1.0, 1 + g])
    wq = np.array([5.0, 8.0, 5.0]) / 18.0
    vals = np.column_stack([(1 - t) * (1 - 2 * t), t * (2 * t - 1), 4 * t * (1 - t)])
    return t, wq, vals


def _face_tri_shapes():
    """P2 shapes on a triangular face at the degree-4 triangle rule (assembly.py:140-144)."""
    a1, w1 = 0.445948490915965, 0.223381589678011
    a2, w2 = 0.091576213509771, 0.109951743655322
    bary = np.array([(1 - 2 * a1, a1, a1), (a1, 1 - 2 * a1, a1), (a1, a1, 1 - 2 * a1),
                     (1 - 2 * a2, a2, a2), (a2, 1 - 2 * a2, a2), (a2, a2, 1 - 2 * a2)])
    wq = 0.5 * np.array([w1, w1, w1, w2, w2, w2])
    lam = np.column_stack([1.0 - bary[:, 1:].sum(axis=1), bary[:, 1], bary[:, 2]])
    vals = np.empty((6, 6))
    for i in range(3):
        vals[:, i] = lam[:, i] * (2.0 * lam[:, i] - 1.0)
    for k, (i, j) in enumerate(((0, 1), (1, 2), (2, 0))):
        vals[:, 3 + k] = 4.0 * lam[:, i] * lam[:, j]
    return bary[:, 1:], wq, vals


def _patch_face_frames(qmesh, patch: str):
    """Outward unit normal and surface Jacobian per face of a patch (metrics.py:42-78), vectorised:
    each face finds its owner element by matching sorted vertex keys against all element faces."""
    try:
        pdata = qmesh.boundary_patches[patch]
    except KeyError:
        raise MeshError(f"unknown boundary patch '{patch}'") from None
    faces = np.asarray(pdata.faces, dtype=np.int64)
    dim = qmesh.dim
    elems = np.asarray(qmesh.elements, dtype=np.int64)
    local = ((0, 1), (1, 2), (2, 0)) if dim == 2 else ((0, 2, 1), (0, 1, 3), (1, 2, 3), (0, 3, 2))
    ekeys = np.sort(np.concatenate([elems[:, list(loc)] for loc in local]), axis=1)
    eown = np.tile(np.arange(len(elems)), len(local))
    fkeys = np.sort(faces, axis=1)
    nv = np.int64(qmesh.n_vertices)
    if qmesh.n_vertices >= 1 << 21:
        raise MeshError("patch frames: too many vertices for packed face keys")

    def pack(k):
        out = k[:, 0].astype(np.int64)
        for c in range(1, k.shape[1]):
            out = out * nv + k[:, c]
        return out

    ek, fk = pack(ekeys), pack(fkeys)
    order = np.argsort(ek, kind="stable")
    pos = np.searchsorted(ek[order], fk)
    if len(faces) and (np.any(pos >= len(ek)) or np.any(ek[order][np.minimum(pos, len(ek) - 1)] != fk)):
        raise MeshError(f"patch '{patch}' has a face that is not an element face")
    owner = eown[order][pos]   # a boundary face belongs to exactly one element
    verts = np.asarray(qmesh.nodes)[: qmesh.n_vertices]
    p = verts[faces]
    if dim == 2:
        t = p[:, 1] - p[:, 0]
        n = np.stack([t[:, 1], -t[:, 0]], axis=1)
        jac = np.linalg.norm(t, axis=1)
    else:
        n = np.cross(p[:, 1] - p[:, 0], p[:, 2] - p[:, 0])
        jac = np.linalg.norm(n, axis=1)
    n = n / np.linalg.norm(n, axis=1)[:, None]
    centroid = verts[elems[owner]].mean(axis=1)
    flip = np.einsum("fd,fd->f", n, p.mean(axis=1) - centroid) < 0
    n[flip] = -n[flip]
    return pdata, n, jac


def flow_rate(nodal, qmesh, patch: str):
    """Flux integral(u . n) of a nodal velocity field through a boundary patch (metrics.py:81-93)."""
    pdata, normals, jac = _patch_face_frames(qmesh, patch)
    nodal = np.asarray(nodal)
    _, wq, vals = _edge_shapes() if qmesh.dim == 2 else _face_tri_shapes()
    face_vals = nodal[np.asarray(pdata.face_conn)]
    uq = np.einsum("qa,fad->fqd", vals, face_vals)
    un = np.einsum("fqd,fd->fq", uq, normals)
    total = np.einsum("fq,q,f->", un, wq, jac)
    return complex(total) if np.iscomplexobj(nodal) else float(total)


def patch_area(qmesh, patch: str) -> float:
    """Measure of a boundary patch: length in 2D, area in 3D (metrics.py:96-101)."""
    _, _, jac = _patch_face_frames(qmesh, patch)
    return float(jac.sum()) if qmesh.dim == 2 else float(0.5 * jac.sum())


def fit_loglog_slope(x, y) -> float:
    """Least-squares slope of log(y) against log(x) (metrics.py:104-110)."""
    x = np.asarray(x, dtype=float)
    y = np.asarray(y, dtype=float)
    if np.any(x <= 0) or np.any(y <= 0):
        raise ValueError("log-log fit requires positive data")
    return float(np.polyfit(np.log(x), np.log(y), 1)[0])
