"""Post-processing on the device: L2 norms / mode energies (reference `metrics.py:12-18`,
`spectral.py:320-330`) — the step after reconstruction that also drives adaptive refinement
(SURVEY.md §8f rank 2)."""

from __future__ import annotations

import numpy as np

from . import _lib
from .assembly import FluidProps, _OP_CACHE, get_operator

__all__ = ["l2_norm", "l2_norms", "mode_energies"]


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
