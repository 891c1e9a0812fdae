"""GPU checks of the mode-sharded path.

* ``ss_comm_*`` (the library's NCCL communicator): a one-rank communicator on cuda:0 gathers
  fields into their global slots exactly (the send/recv pairs of N > 1 ranks need N GPUs; the
  posting logic for other ranks is the same loop).
* ``solve_mode_systems_distributed`` end to end with two processes (gloo, fields staged through
  host memory, both ranks on cuda:0 solving independent batches -- no kernel waits on another
  rank): the gathered fields equal a single-process ``solve_mode_systems`` bit for bit.
"""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def test_nccl_comm_single_rank_gather():
    from paper_2009_06725_b200 import _lib
    from paper_2009_06725_b200.comm import ModeComm

    assert _lib.load().ss_comm_nccl_version() >= 21800
    comm = ModeComm.single(0)
    plan = [[3, 0, 2, 1]]
    local = torch.randn((4, 1001), dtype=torch.complex128, device="cuda")
    full = comm.gather_modes(local, plan)
    torch.cuda.synchronize()
    for j, i in enumerate(plan[0]):
        assert torch.equal(full[i], local[j])
    t = torch.tensor([1.5, -2.0], dtype=torch.float64, device="cuda")
    comm.allreduce_max(t)
    assert t.tolist() == [1.5, -2.0]
    comm.close()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _c1_inputs():
    from paper_2009_06725_b200 import FluidProps, SolverSettings
    from paper_2009_06725_b200.workloads import c1_case

    case = c1_case()
    idx = [1, 2, 3, 5, 8]
    h = case.h_modes()
    return case, FluidProps(case.density, case.viscosity), idx, case.omegas[idx], [h[i] for i in idx], \
        SolverSettings(tolerance=1e-9, restart=60)


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2009_06725_b200.distributed import solve_mode_systems_distributed

        case, props, idx, om, h, settings = _c1_inputs()
        U, P, reps, plan = solve_mode_systems_distributed(case.qmesh, props, idx, om, None, h, settings, rank, world,
                                                          dst=0)
        out[rank] = (None if U is None else (U.cpu().numpy(), P.cpu().numpy()), [r.iterations for r in reps], plan)
    finally:
        dist.destroy_process_group()


def test_distributed_solve_world2_matches_single_process():
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    from paper_2009_06725_b200 import solve_mode_systems

    case, props, idx, om, h, settings = _c1_inputs()
    ref = solve_mode_systems(case.qmesh, props, idx, om, None, h, settings)
    (U, P), _, plan = out[0]
    assert out[1][0] is None
    assert sorted(i for p in plan for i in p) == list(range(len(idx)))
    for k, s in enumerate(ref):
        assert np.array_equal(U[k], s.velocity) and np.array_equal(P[k], s.pressure)
    iters = {plan[r][j]: it for r in (0, 1) for j, it in enumerate(out[r][1])}
    assert [iters[k] for k in range(len(idx))] == [s.report.iterations for s in ref]


def test_nccl_reduce_single_rank():
    from paper_2009_06725_b200.comm import ModeComm

    comm = ModeComm.single(0)
    t = torch.randn(1000, dtype=torch.float64, device="cuda")
    ref = t.clone()
    comm.reduce_sum(t)
    torch.cuda.synchronize()
    assert torch.equal(t, ref)
    comm.close()


def _recon_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2009_06725_b200 import solve_mode_systems
        from paper_2009_06725_b200.distributed import expected_iterations, lpt_shard, reconstruct_distributed

        case, props, idx, om, h, settings = _c1_inputs()
        plan = lpt_shard(expected_iterations(idx, 2), world)
        mine = plan[rank]
        sols = solve_mode_systems(case.qmesh, props, [idx[i] for i in mine], om[mine], None, [h[i] for i in mine],
                                  settings)
        U, P = reconstruct_distributed(sols, [0.0, 0.3, 0.7], rank, world)
        out[rank] = None if U is None else (U, P)
    finally:
        dist.destroy_process_group()


def test_reconstruct_distributed_world2_matches_single_process():
    """Per-rank partial reconstructions summed over ranks (gloo reduce here; ncclReduce through
    ss_comm_reduce_sum on GPUs) equal the single-process reconstruction to rounding."""
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_recon_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    from paper_2009_06725_b200 import reconstruct_series, solve_mode_systems

    case, props, idx, om, h, settings = _c1_inputs()
    sols = solve_mode_systems(case.qmesh, props, idx, om, None, h, settings)
    Ur, Pr = reconstruct_series(sols, [0.0, 0.3, 0.7])
    U, P = out[0]
    assert out[1] is None
    assert np.abs(U - Ur).max() <= 1e-13 * np.abs(Ur).max()
    assert np.abs(P - Pr).max() <= 1e-13 * np.abs(Pr).max()
