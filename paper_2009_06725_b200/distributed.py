"""Multi-GPU mode sharding: one process per GPU, modes partitioned, one collective at the end.

Modes are independent boundary-value problems (reference spectral.py:287-305; PAPER §1): there
is no exchange during the solves.  The only data movement is gathering the solved modal fields
to the reconstructing rank, done here with one ``all_gather`` over torch.distributed (NCCL over
NVLink on the GPU box, gloo in the CPU tests).

* :func:`lpt_shard` — longest-processing-time-first assignment by expected GMRES iterations
  (SURVEY.md §8e); deterministic for a given cost vector.
* :func:`expected_iterations` — cost model: flat in 2D, growing ~linearly with the mode index in
  3D (measured on the reference: 9 687 iterations for mode 1 vs 20 603 for mode 16 on the small
  pipe, tests/golden/pipe3d.npz).
* :func:`gather_mode_fields` — padded all_gather of per-rank modal fields to every rank / dst.
* :func:`solve_mode_systems_distributed` — shard, solve the local batch on the local GPU, gather.
"""

from __future__ import annotations

import numpy as np

__all__ = ["lpt_shard", "expected_iterations", "gather_mode_fields", "solve_mode_systems_distributed"]


def expected_iterations(indices, dim: int) -> np.ndarray:
    idx = np.asarray(indices, dtype=float)
    if dim == 2:
        return np.ones_like(idx)
    return 1.0 + 0.075 * idx


def lpt_shard(costs, world: int):
    """Assign items to ``world`` bins, largest cost first, each to the least-loaded bin.

    Ties are broken by item index and then by rank, so every rank computes the same plan.
    Returns per-rank sorted index lists.
    """
    costs = np.asarray(costs, dtype=float)
    order = sorted(range(costs.size), key=lambda i: (-costs[i], i))
    load = np.zeros(world)
    bins = [[] for _ in range(world)]
    for i in order:
        r = int(np.argmin(load))
        bins[r].append(i)
        load[r] += costs[i]
    return [sorted(b) for b in bins]


def gather_mode_fields(local, plan, rank: int, world: int, group=None):
    """All-gather per-rank (m_r, N) field blocks into the global (sum m_r, N) order of ``plan``.

    ``local`` is a real or complex torch tensor on the backend's device; complex data travels as
    float64 pairs.  Returns the global tensor (every rank receives it).
    """
    import torch
    import torch.distributed as dist

    counts = [len(p) for p in plan]
    m = max(counts) if counts else 0
    is_complex = local.is_complex()
    payload = torch.view_as_real(local) if is_complex else local
    tail = tuple(payload.shape[1:])
    pad = torch.zeros((m,) + tail, dtype=payload.dtype, device=payload.device)
    pad[: payload.shape[0]] = payload
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    total = sum(counts)
    out = torch.empty((total,) + tail, dtype=payload.dtype, device=payload.device)
    for r, idxs in enumerate(plan):
        if idxs:
            out[torch.as_tensor(idxs, device=payload.device)] = bufs[r][: len(idxs)]
    return torch.view_as_complex(out) if is_complex else out


def solve_mode_systems_distributed(qmesh, props, indices, omegas, g_modes, h_modes, settings, rank: int,
                                   world: int, group=None):
    """Shard modes over ranks (LPT), solve the local batch on this rank's GPU, gather fields.

    Returns ``(U, P, reports_local, plan)`` with U (n_modes, n_vn, dim) and P (n_modes, n_vert)
    complex device tensors on every rank.
    """
    import torch

    from .spectral import solve_mode_systems

    plan = lpt_shard(expected_iterations(indices, qmesh.dim), world)
    mine = plan[rank]
    sols = solve_mode_systems(qmesh, props, [indices[i] for i in mine], np.asarray(omegas)[mine],
                              None if g_modes is None else [g_modes[i] for i in mine],
                              None if h_modes is None else [h_modes[i] for i in mine], settings, keep_device=True)
    dev = torch.device("cuda", torch.cuda.current_device())
    nu = qmesh.n_velocity_nodes * qmesh.dim
    local = torch.zeros((len(mine), nu + qmesh.n_vertices), dtype=torch.complex128, device=dev)
    for j, s in enumerate(sols):
        local[j, :nu] = s._device[0].reshape(-1)
        local[j, nu:] = s._device[1]
    full = gather_mode_fields(local, plan, rank, world, group)
    U = full[:, :nu].reshape(-1, qmesh.n_velocity_nodes, qmesh.dim)
    P = full[:, nu:]
    return U, P, [s.report for s in sols], plan
