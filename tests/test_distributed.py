"""Multi-rank mode sharding on CPU (gloo, world size 2): LPT plan and the modal-field gather.

The GPU path is one process per GPU with the library's NCCL gather (ss_comm_gather_modes); the
host logic (sharding plan, gather to one destination rank, global ordering) is exercised here with
gloo so it runs without GPUs.  GPU end-to-end checks live in tests/test_gpu_distributed.py.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2009_06725_b200.distributed import (
    calibrate_iterations, expected_iterations, gather_mode_fields, iterations_from_first_cycle, lpt_shard,
)


def test_lpt_balances_and_covers():
    costs = expected_iterations(np.arange(128), 3)
    for world in (1, 2, 4, 8):
        plan = lpt_shard(costs, world)
        flat = sorted(i for p in plan for i in p)
        assert flat == list(range(128))
        loads = [costs[p].sum() for p in plan]
        assert max(loads) - min(loads) <= costs.max()
    assert lpt_shard(costs, 4) == lpt_shard(costs, 4)            # deterministic
    assert lpt_shard(np.ones(17), 8)[0] == [0, 8, 16]             # ties -> lowest rank, index order


def test_expected_iterations_model():
    assert np.all(expected_iterations(np.arange(9), 2) == 1.0)
    c = expected_iterations([1, 16], 3)
    assert c[1] / c[0] == pytest.approx(886_922 / 336_974)         # measured at config 2 (profiles/)


def test_calibration_from_reference_counts():
    from golden_util import golden

    g = golden("pipe3d.npz")
    a, b = calibrate_iterations([1, 16], [int(g["iters_1"]), int(g["iters_16"])])
    assert a + b == pytest.approx(1.0)
    assert (a + 16 * b) == pytest.approx(int(g["iters_16"]) / int(g["iters_1"]), rel=1e-12)
    assert calibrate_iterations([3], [100]) == (1.0, 0.0)


def test_first_cycle_prediction():
    h = list(0.5 ** np.arange(1, 201) ** 0 * np.geomspace(1.0, 1e-2, 200))   # 1e-2 per 200-iteration cycle
    pred = iterations_from_first_cycle([h, h[:50]], 1e-10, 200)
    assert pred[0] == pytest.approx(1000.0, rel=0.01)                   # 5 cycles of 200
    assert pred[1] == 50.0                                              # converged inside the first cycle


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n_modes, n_field, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        plan = lpt_shard(expected_iterations(np.arange(n_modes), 3), world)
        mine = plan[rank]
        # each rank "solves" its modes: field of mode i is a deterministic function of i
        local = torch.zeros((len(mine), n_field), dtype=torch.complex128)
        for j, i in enumerate(mine):
            local[j] = torch.arange(n_field, dtype=torch.float64) * (i + 1) + 1j * i
        full = gather_mode_fields(local, plan, rank, world, dst=world - 1)
        out[rank] = None if full is None else full.numpy().copy()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_modes", [17, 5])
def test_gather_mode_fields_gloo_world2(n_modes):
    world, n_field = 2, 37
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), n_modes, n_field, out), nprocs=world, join=True)
    ref = np.stack([np.arange(n_field) * (i + 1) + 1j * i for i in range(n_modes)])
    assert np.array_equal(out[world - 1], ref)        # only the destination rank receives
    assert all(out[r] is None for r in range(world - 1))
