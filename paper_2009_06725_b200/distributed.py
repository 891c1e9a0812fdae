"""Multi-GPU mode sharding: one process per GPU, modes partitioned, one gather at the end.

Modes are independent boundary-value problems (reference spectral.py:287-305; PAPER §1): there is
no exchange during the solves.  The only data movement is gathering the solved modal fields to the
reconstructing rank:

* on GPUs, through the library's NCCL communicator (:class:`~.comm.ModeComm`,
  ``ss_comm_gather_modes``: one grouped ncclSend/ncclRecv round over NVLink, fields land in their
  global slot on the root);
* without GPUs (the CPU tests), through torch.distributed ``gather`` on the gloo backend.

Pieces:

* :func:`expected_iterations` -- the LPT cost model: flat in 2D, linear in the mode index in 3D,
  fitted to converged iteration counts measured at BASELINE config 2 (modes 1 and 16);
  :func:`calibrate_iterations` refits it from any measured counts and
  :func:`iterations_from_first_cycle` predicts counts from a first restart cycle's estimates.
* :func:`lpt_shard` -- longest-processing-time-first assignment.
* :func:`gather_mode_fields` -- the gather to one destination rank.
* :func:`solve_mode_systems_distributed` -- shard, solve the local batch on this rank's GPU, free
  the Krylov workspace, gather.
"""

from __future__ import annotations

import numpy as np

__all__ = ["lpt_shard", "expected_iterations", "calibrate_iterations", "iterations_from_first_cycle",
           "gather_mode_fields", "solve_mode_systems_distributed", "reconstruct_distributed", "DEFAULT_3D_MODEL"]

# Iterations to 1e-10 (restart 200) measured on the GPU at BASELINE config 2 (n = 796 978;
# profiles/r2_c2_converge.json, tools/c2_converge.py): mode 1 336 974, mode 16 886 922 -> per mode-1
# cost a + b*idx with a + b = 1, a + 16 b = 2.632.  (The reference's own counts on the down-scaled
# pipe, tests/golden/pipe3d.npz: 9 687 and 20 603, ratio 2.13 -- the growth with the mode index
# steepens with n.)
C2_MEASURED_ITERATIONS = {1: 336_974, 16: 886_922}
DEFAULT_3D_MODEL = (1.0 - (886_922 / 336_974 - 1.0) / 15.0, (886_922 / 336_974 - 1.0) / 15.0)


def calibrate_iterations(indices, iterations):
    """Least-squares fit ``iters ~ a + b * idx`` to measured counts; returns (a, b) scaled so a + b = 1
    at mode 1 (only ratios matter for load balance)."""
    idx = np.asarray(indices, dtype=float)
    it = np.asarray(iterations, dtype=float)
    if idx.size < 2 or np.ptp(idx) == 0:
        return 1.0, 0.0
    b, a = np.polyfit(idx, it, 1)
    s = a + b
    if s <= 0:
        return 1.0, 0.0
    return float(a / s), float(b / s)


def iterations_from_first_cycle(histories, tol, restart):
    """Predicted total iterations per mode from the first restart cycle's residual estimates.

    Restarted GMRES reduces the estimate by roughly the same factor every cycle, so
    ``cycles ~ log(tol / est_0) / log(est_end / est_0)`` for each mode's first-cycle history.
    """
    out = []
    for h in histories:
        h = np.asarray(h, dtype=float)
        if h.size == 0 or h[0] <= 0:
            out.append(0.0)
            continue
        if h[-1] <= tol * h[0] or h.size < restart:
            out.append(float(h.size))
            continue
        rate = np.log(max(h[-1], 1e-300) / h[0])
        cycles = np.log(tol) / rate if rate < 0 else 1e6
        out.append(float(cycles * restart))
    return np.asarray(out)


def expected_iterations(indices, dim: int, model=None) -> np.ndarray:
    idx = np.asarray(indices, dtype=float)
    if dim == 2:
        return np.ones_like(idx)
    a, b = DEFAULT_3D_MODEL if model is None else model
    return a + b * idx


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


def gather_mode_fields(local, plan, rank: int, world: int, group=None, comm=None, dst: int = 0):
    """Gather per-rank (m_r, N) field blocks to rank ``dst`` in the global order of ``plan``.

    With a :class:`~.comm.ModeComm` the library's NCCL gather runs on the device; otherwise
    torch.distributed ``gather`` (gloo in the CPU tests; CUDA tensors are staged through host
    memory).  Returns the (sum m_r, N) tensor on ``dst`` and None elsewhere.
    """
    import torch

    if comm is not None:
        return comm.gather_modes(local, plan, root=dst)
    import torch.distributed as dist

    counts = [len(p) for p in plan]
    m = max(counts) if counts else 0
    is_complex = local.is_complex()
    payload = torch.view_as_real(local) if is_complex else local
    staged = dist.get_backend(group) == "gloo" and payload.is_cuda
    dev = payload.device
    if staged:
        payload = payload.cpu()
    tail = tuple(payload.shape[1:])
    pad = torch.zeros((m,) + tail, dtype=payload.dtype, device=payload.device)
    pad[: payload.shape[0]] = payload
    bufs = [torch.empty_like(pad) for _ in range(world)] if rank == dst else None
    dist.gather(pad, bufs, dst=dst, group=group)
    if rank != dst:
        return None
    total = sum(counts)
    out = torch.empty((total,) + tail, dtype=payload.dtype, device=payload.device)
    for r, idxs in enumerate(plan):
        if idxs:
            out[torch.as_tensor(idxs)] = bufs[r][: len(idxs)]
    if staged:
        out = out.to(dev)
    return torch.view_as_complex(out) if is_complex else out


def solve_mode_systems_distributed(qmesh, props, indices, omegas, g_modes, h_modes, settings, rank: int,
                                   world: int, group=None, comm=None, dst: int = 0, model=None):
    """Shard modes over ranks (LPT), solve the local batch on this rank's GPU, gather fields to ``dst``.

    Returns ``(U, P, reports_local, plan)``: U (n_modes, n_vn, dim) and P (n_modes, n_vert) complex
    device tensors on ``dst`` (None elsewhere).
    """
    import torch

    from .assembly import get_operator
    from .spectral import solve_mode_systems

    plan = lpt_shard(expected_iterations(indices, qmesh.dim, model), world)
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
        s._device = None
    get_operator(qmesh, props).release_workspaces()   # the basis is dead weight during the gather
    full = gather_mode_fields(local, plan, rank, world, group, comm=comm, dst=dst)
    if full is None:
        return None, None, [s.report for s in sols], plan
    U = full[:, :nu].reshape(-1, qmesh.n_velocity_nodes, qmesh.dim)
    P = full[:, nu:]
    return U, P, [s.report for s in sols], plan


def reconstruct_distributed(local_solutions, times, rank: int, world: int, group=None, comm=None, dst: int = 0):
    """u(x, t_j), p(x, t_j) on rank ``dst`` from modes sharded over ranks, without gathering them:
    each rank reconstructs its own modes for all samples (``reconstruct_series``, one fused launch)
    and the partial sums are added over ranks (``ss_comm_reduce_sum``: ncclReduce; gloo ``reduce``
    in the CPU tests).  Cheaper than gathering the modal fields when the number of samples T is
    below twice the modes per rank.  Returns ``(U, P)`` (T, n_vn, dim) / (T, n_vert)
    host arrays on ``dst`` and None elsewhere; a rank with no modes contributes zeros.
    """
    import torch

    from .spectral import reconstruct_series

    times = np.atleast_1d(np.asarray(times, dtype=float))
    if local_solutions:
        u, p = reconstruct_series(local_solutions, times)
        shape_u = u.shape[1:]
        flat = np.concatenate([u.reshape(times.size, -1), p], axis=1)
    else:
        flat = None
    # every rank needs the field sizes: take them from the first rank that has modes
    if comm is not None:
        dev = torch.device("cuda", comm.device)
        buf = torch.from_numpy(flat).to(dev) if flat is not None else None
        if buf is None:
            raise ValueError("every rank needs at least one mode for the NCCL reduction (plan with world <= modes)")
        comm.reduce_sum(buf, root=dst)
        out = buf.cpu().numpy() if rank == dst else None
    else:
        import torch.distributed as dist

        t = torch.from_numpy(flat) if flat is not None else None
        if t is None:
            raise ValueError("every rank needs at least one mode (plan with world <= modes)")
        dist.reduce(t, dst=dst, group=group)
        out = t.numpy() if rank == dst else None
    if out is None:
        return None, None
    nu = int(np.prod(shape_u))
    return out[:, :nu].reshape((times.size,) + tuple(shape_u)), out[:, nu:]
