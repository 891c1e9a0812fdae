"""Multi-rank mode sharding on CPU (gloo, world size 2): LPT plan and the modal-field gather.

The GPU path is one process per GPU with NCCL; the host logic (sharding plan, padded
all_gather, global ordering) is exercised here with gloo so it runs without GPUs.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2009_06725_b200.distributed import expected_iterations, gather_mode_fields, lpt_shard


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
    assert 1.9 < c[1] / c[0] < 2.3                                 # reference: 20 603 / 9 687 = 2.13


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
        full = gather_mode_fields(local, plan, rank, world)
        out[rank] = full.numpy().copy()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_modes", [17, 5])
def test_gather_mode_fields_gloo_world2(n_modes):
    world, n_field = 2, 37
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), n_modes, n_field, out), nprocs=world, join=True)
    ref = np.stack([np.arange(n_field) * (i + 1) + 1j * i for i in range(n_modes)])
    for r in range(world):
        assert np.array_equal(out[r], ref)
